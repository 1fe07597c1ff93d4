"""The C ABI from a plain-C host (examples/c_host.c): the header compiles as C99 with -Werror and
every entry point the program calls links against the in-tree library (CPU); on the GPU the
program's results through ps_eval_batch_host and ps_eval_batch_host_delta match the oracle."""

import shutil
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


def compile_host(tmp_path: Path) -> Path:
    from paper_2510_05186_b200 import build
    lib = build.build()
    if shutil.which("gcc") is None:
        pytest.skip("no gcc")
    exe = tmp_path / "c_host"
    subprocess.run(["gcc", "-std=c99", "-O2", "-Wall", "-Wextra", "-Werror", "-I", str(ROOT / "include"),
                    str(ROOT / "examples" / "c_host.c"), "-L", str(lib.parent), "-lpipesched_b200",
                    f"-Wl,-rpath,{lib.parent}", "-o", str(exe)], check=True)
    return exe


def test_c_host_compiles_and_links(tmp_path):
    exe = compile_host(tmp_path)
    r = subprocess.run([str(exe)], capture_output=True, text=True)
    assert r.returncode == 1 and "usage" in r.stderr


def write_input(path: Path, pk, orders, masks):
    with open(path, "wb") as f:
        np.array([pk.num_stages, pk.num_microbatches, pk.num_channels, int(pk.post_validation)],
                 np.int32).tofile(f)
        np.array([pk.comm_time, pk.offload_time], np.int64).tofile(f)
        for a in (pk.proc_time, pk.mem_delta, pk.act_size, pk.mem_limit):
            np.ascontiguousarray(a, np.int64).tofile(f)
        np.ascontiguousarray(pk.stage_channel, np.int32).tofile(f)
        np.array([orders.shape[0]], np.int64).tofile(f)
        np.ascontiguousarray(orders, np.uint16).tofile(f)
        np.ascontiguousarray(masks, np.uint32).tofile(f)


def read_output(path: Path, n: int, P: int):
    raw = path.read_bytes()
    out, off = {}, 0
    for name, dt, cnt in (("makespan", np.int64, n), ("bubble", np.float64, n), ("flags", np.uint32, n),
                          ("blocked", np.uint32, n), ("peak", np.int64, n * P), ("makespan_d", np.int64, n),
                          ("bubble_d", np.float64, n), ("flags_d", np.uint32, n)):
        out[name] = np.frombuffer(raw, dt, cnt, off)
        off += np.dtype(dt).itemsize * cnt
    assert off == len(raw)
    out["peak"] = out["peak"].reshape(n, P)
    return out


def neighbours(pk, orders0, mask0, n, rng):
    """Candidate 0 is the base; the rest are one adjacent swap, one offload toggle, or a few of
    each (which the delta entry point rebuilds in HBM instead of move-encoding)."""
    P, m = pk.num_stages, pk.num_microbatches
    offloadable = np.flatnonzero(pk.act_size.reshape(-1) > 0)
    orders = np.repeat(orders0[None], n, 0)
    masks = np.repeat(mask0[None], n, 0)
    for c in range(1, n):
        k = 1 if c % 3 else int(rng.integers(2, 5))
        for _ in range(k):
            if len(offloadable) and rng.random() < 0.3:
                b = int(rng.choice(offloadable))
                masks[c, b >> 5] ^= np.uint32(1 << (b & 31))
            else:
                i, a = int(rng.integers(P)), int(rng.integers(3 * m - 1))
                orders[c, i, a], orders[c, i, a + 1] = orders[c, i, a + 1], orders[c, i, a]
    return orders, masks


@pytest.mark.gpu
@pytest.mark.parametrize("cfg", ["config1", "config2", "config3"])
def test_c_host_matches_oracle(tmp_path, cuda_ok, cfg):
    from oracle.oracle import Oracle
    from paper_2510_05186_b200 import workloads
    from paper_2510_05186_b200.heuristics import generator_structures
    from paper_2510_05186_b200.packing import encode_candidate, pack_instance

    exe = compile_host(tmp_path)
    inst = getattr(workloads, cfg)()
    pk = pack_instance(inst)
    o, mk, _ = [encode_candidate(pk, o, f) for o, f in generator_structures(inst)][0]
    orders, masks = neighbours(pk, o, mk, 512, np.random.default_rng(7))
    write_input(tmp_path / "in.bin", pk, orders, masks)
    r = subprocess.run([str(exe), str(tmp_path / "in.bin"), str(tmp_path / "out.bin")],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    got = read_output(tmp_path / "out.bin", len(orders), pk.num_stages)
    want = Oracle(pk).eval_batch(orders, masks)
    assert (got["flags"] == want["flags"]).all()
    assert (got["makespan"] == want["makespan"]).all()
    ok = want["flags"] == 1
    assert ok.sum() > 10 and (~ok).any()
    assert (got["peak"][ok] == want["peak"][ok]).all()
    assert (got["bubble"][ok] == want["bubble"][ok]).all()
    dead = (want["flags"] & 2) != 0
    assert (got["blocked"][dead] == want["blocked"][dead]).all()
    # the delta-encoded batch: same outcomes
    assert (got["flags_d"] == want["flags"]).all()
    assert (got["makespan_d"] == want["makespan"]).all()
    assert (got["bubble_d"][ok] == want["bubble"][ok]).all()
