"""GPU local search vs its CPU restatement (oracle/ps_oracle.c): moves, rounds, whole searches."""

from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SEED, PERMILLE, MAXSHIFT = 11, 700, 4


def _setup(cfg=2):
    from paper_2510_05186_b200 import workloads
    from paper_2510_05186_b200.heuristics import best_feasible
    from paper_2510_05186_b200.listsched import stage_order_of
    from paper_2510_05186_b200.search import LocalSearch, SearchConfig
    inst = workloads.CONFIGS[cfg]()
    s, _ = best_feasible(inst)
    orders = {i: stage_order_of(s, i) for i in range(1, inst.num_stages + 1)}
    return inst, orders, s.offloaded, LocalSearch, SearchConfig


def test_move_decoding_matches_the_cpu_restatement(cuda_ok):
    from oracle.oracle import Oracle
    inst, orders, off, LocalSearch, SearchConfig = _setup()
    ls = LocalSearch(inst, orders, off, SearchConfig(seed=SEED, neighbours=512, shift_permille=PERMILLE,
                                                     max_shift=MAXSHIFT))
    orc = Oracle(ls.di.packed)
    inc_o = ls.inc_orders.cpu().numpy().view(np.uint16)
    inc_m = ls.inc_mask.cpu().numpy().view(np.uint32)
    for rnd in (0, 3):
        o, mk = ls.materialize(0, 512, rnd)
        o = o.cpu().numpy().view(np.uint16)
        mk = mk.cpu().numpy().view(np.uint32)
        kinds = set()
        for idx in range(512):
            t, oo, mm = orc.neighbour(inc_o, inc_m, SEED, PERMILLE, MAXSHIFT, rnd, idx)
            kinds.add(t)
            assert (oo == o[idx]).all(), idx
            assert (mm == mk[idx]).all(), idx
        assert kinds == {0, 1, 2}


def test_search_round_matches_cpu_round(cuda_ok):
    import torch
    import ctypes as C
    from oracle.oracle import Oracle
    from paper_2510_05186_b200 import _native as N
    inst, orders, off, LocalSearch, SearchConfig = _setup(3)
    n = 2048
    ls = LocalSearch(inst, orders, off, SearchConfig(seed=SEED, neighbours=n, shift_permille=PERMILLE,
                                                     max_shift=MAXSHIFT))
    ms = torch.empty(n, dtype=torch.int64, device="cuda")
    ls.launch_round(ms)
    torch.cuda.synchronize()
    orc = Oracle(ls.di.packed)
    best, want = orc.search_round(ls.inc_orders.cpu().numpy().view(np.uint16),
                                  ls.inc_mask.cpu().numpy().view(np.uint32), SEED, PERMILLE, MAXSHIFT,
                                  0, 0, n, want_makespans=True)
    assert (ms.cpu().numpy() == want).all()
    assert int(ls.best_key.item()) == best


@pytest.mark.parametrize("cfg,n", [(5, 24), (4, 256)])
def test_search_round_matches_cpu_round_large(cuda_ok, cfg, n):
    """Configs 5 (32 x 256) and 4 (16 x 128), whose search rounds keep per-candidate state in
    global scratch (16-warp blocks sharing the incumbent): a round's neighbours with prefix/suffix
    sharing against the recorded incumbent vs the CPU restatement."""
    import torch
    from oracle.oracle import Oracle
    inst, orders, off, LocalSearch, SearchConfig = _setup(cfg)
    ls = LocalSearch(inst, orders, off, SearchConfig(seed=SEED, neighbours=n, shift_permille=PERMILLE,
                                                     max_shift=MAXSHIFT))
    ms = torch.empty(n, dtype=torch.int64, device="cuda")
    ls.launch_round(ms)
    torch.cuda.synchronize()
    orc = Oracle(ls.di.packed)
    best, want = orc.search_round(ls.inc_orders.cpu().numpy().view(np.uint16),
                                  ls.inc_mask.cpu().numpy().view(np.uint32), SEED, PERMILLE, MAXSHIFT,
                                  0, 0, n, want_makespans=True)
    assert (ms.cpu().numpy() == want).all()
    assert int(ls.best_key.item()) == best


def test_identical_best_schedule_for_equal_budgets(cuda_ok):
    """A whole search: the GPU and the CPU restatement adopt the same moves and end identical."""
    from oracle.oracle import Oracle
    inst, orders, off, LocalSearch, SearchConfig = _setup(2)
    n, rounds = 1024, 6
    ls = LocalSearch(inst, orders, off, SearchConfig(seed=SEED, neighbours=n, shift_permille=PERMILLE,
                                                     max_shift=MAXSHIFT))
    orc = Oracle(ls.di.packed)
    inc_o = ls.inc_orders.cpu().numpy().view(np.uint16)
    inc_m = ls.inc_mask.cpu().numpy().view(np.uint32)
    span = ls.makespan
    cpu_trail = []
    for rnd in range(rounds):
        best, _ = orc.search_round(inc_o, inc_m, SEED, PERMILLE, MAXSHIFT, rnd, 0, n)
        if best != (1 << 63) - 1 and (best >> 32) < span:
            span = best >> 32
            _, inc_o, inc_m = orc.neighbour(inc_o, inc_m, SEED, PERMILLE, MAXSHIFT, rnd, best & 0xFFFFFFFF)
            cpu_trail.append((rnd, span))
    res = ls.run(rounds=rounds)
    assert [(imp.round, imp.makespan) for imp in res.improvements] == cpu_trail
    assert res.makespan == span
    assert (ls.inc_orders.cpu().numpy().view(np.uint16) == inc_o).all()
    assert (ls.inc_mask.cpu().numpy().view(np.uint32) == inc_m).all()
    from paper_2510_05186_b200 import makespan, validate
    assert validate(res.schedule, inst).ok and makespan(res.schedule, inst) == span


def test_generators_match_reference_outputs(cuda_ok):
    """Batched warm-start generation vs the reference generators (tests/golden/generators.json.gz)."""
    import gzip
    import json
    from pathlib import Path
    from paper_2510_05186_b200 import instance_from_dict, makespan, memory_trace
    from paper_2510_05186_b200.heuristics import best_feasible, generate_all, ada_fill_counts
    from paper_2510_05186_b200.listsched import stage_order_of
    g = json.load(gzip.open(Path(__file__).parent / "golden" / "generators.json.gz", "rt"))
    for row in g["generators"]:
        inst = instance_from_dict(row["instance"])
        assert [ada_fill_counts(inst)[i] for i in range(1, inst.num_stages + 1)] == row["ada_fills"]
        out = generate_all(inst)
        for name, want in row["generators"].items():
            got = out[name]
            if "infeasible" in want:
                assert isinstance(got, Exception), name
                continue
            assert makespan(got, inst) == want["makespan"], name
            enc = [[((op.microbatch - 1) << 2) | int(op.kind) for op in stage_order_of(got, i)]
                   for i in range(1, inst.num_stages + 1)]
            assert enc == want["orders"], name
            assert sorted([op.stage, op.microbatch] for op in got.offloaded) == want["offloaded"]
            assert [memory_trace(got, inst).peak[i] for i in range(1, inst.num_stages + 1)] == want["peak"]
        if row["best_feasible"] is None:
            continue
        s, name = best_feasible(inst)
        assert name == row["best_feasible"]["name"]
        assert makespan(s, inst) == row["best_feasible"]["makespan"]


def _eval_both(di, orders, masks, base):
    r0 = di.evaluate(orders, masks, peak=True)
    r1 = di.evaluate(orders, masks, peak=True, base=base)
    # without the blocked-stage output, deadlocks may be concluded early (cyclic waits)
    r2 = di.evaluate(orders, masks, base=base, out=di.alloc_results(int(orders.shape[0]), peak=True, blocked=False))
    import torch
    torch.cuda.synchronize()
    for f in ("flags", "makespan", "peak", "blocked"):
        a, b = getattr(r0, f).cpu().numpy(), getattr(r1, f).cpu().numpy()
        assert (a == b).all(), f
    for f in ("flags", "makespan", "peak"):
        assert (getattr(r0, f).cpu().numpy() == getattr(r2, f).cpu().numpy()).all(), f + " (no blocked output)"
    ok = (r0.flags.cpu().numpy() & 1) == 1
    assert (r0.bubble.cpu().numpy()[ok] == r1.bubble.cpu().numpy()[ok]).all()
    return r0


@pytest.mark.parametrize("cfg", [2, 3, 4])
def test_prefix_sharing_is_exact(cuda_ok, cfg):
    """Evaluations resumed from the recorded incumbent's checkpoints equal full simulations."""
    import ctypes as C
    import torch
    from paper_2510_05186_b200 import _native as N
    from paper_2510_05186_b200.engine import Base
    inst, orders, off, LocalSearch, SearchConfig = _setup(cfg)
    n = 1024
    ls = LocalSearch(inst, orders, off, SearchConfig(seed=SEED, neighbours=n, shift_permille=PERMILLE,
                                                     max_shift=MAXSHIFT, share_prefix=True))
    # materialised neighbours, with and without the base
    o, mk = ls.materialize(0, n, 0)
    r = _eval_both(ls.di, o, mk, ls.base)
    # search-round makespans, with and without the base
    ms = []
    for base in (None, ls.base):
        out = torch.empty(n, dtype=torch.int64, device="cuda")
        ls.best_key.fill_(N.BEST_NONE)
        desc = N.SearchDesc(ls.inc_orders.data_ptr(), ls.inc_mask.data_ptr(), 0, 0, n, ls.moves, None,
                            base.handle if base is not None else None)
        N.check(ls.lib.ps_search_round(ls.di.handle, C.byref(desc), C.c_void_p(ls.best_key.data_ptr()),
                                       C.c_void_p(out.data_ptr()), ls._stream()))
        torch.cuda.synchronize()
        ms.append((out.cpu().numpy(), int(ls.best_key.item())))
    assert (ms[0][0] == ms[1][0]).all() and ms[0][1] == ms[1][1]
    assert (ms[0][0] == r.makespan.cpu().numpy()).all()
    # an unrelated (deadlocking) base: still exact
    bad = Base(ls.di)
    o2 = o[1:2].clone()
    row = o2[0, 0].clone()
    o2[0, 0, :2] = torch.flip(row[:2], [0])
    bad.record(o2[0], mk[1])
    _eval_both(ls.di, o, mk, bad)


@pytest.mark.parametrize("cfg,n", [(4, 16384), (5, 4096)])
def test_global_state_row_bands_are_exact(cuda_ok, cfg, n):
    """Configs 4 and 5 keep each warp's candidate state in global scratch and restore / compare only
    the end-time rows' bands.  With several neighbours per warp (so each slot goes
    through resumes from different checkpoints, fresh starts and convergences in turn), a search
    round with the recorded base gives every neighbour the makespan of its full simulation."""
    import ctypes as C
    import torch
    from paper_2510_05186_b200 import _native as N
    inst, orders, off, LocalSearch, SearchConfig = _setup(cfg)
    ls = LocalSearch(inst, orders, off, SearchConfig(seed=SEED, neighbours=n, shift_permille=PERMILLE,
                                                     max_shift=MAXSHIFT))
    got = []
    for rnd in (0, 1):
        for base in (ls.base, None):
            out = torch.empty(n, dtype=torch.int64, device="cuda")
            ls.best_key.fill_(N.BEST_NONE)
            desc = N.SearchDesc(ls.inc_orders.data_ptr(), ls.inc_mask.data_ptr(), rnd, 0, n, ls.moves, None,
                                base.handle if base is not None else None)
            N.check(ls.lib.ps_search_round(ls.di.handle, C.byref(desc), C.c_void_p(ls.best_key.data_ptr()),
                                           C.c_void_p(out.data_ptr()), ls._stream()))
            torch.cuda.synchronize()
            got.append((out.cpu().numpy(), int(ls.best_key.item())))
        (a, ka), (b, kb) = got[-2], got[-1]
        assert (a == b).all(), (rnd, int((a != b).sum()))
        assert ka == kb
        assert (a >= 0).any()


@pytest.mark.parametrize("cfg", [2, 3])
def test_rerecorded_base_is_exact(cuda_ok, cfg):
    """A base re-recorded over a previous one (it resumes from the previous checkpoints up to their
    first difference) shares exactly: feasible and deadlocking bases in turn."""
    from paper_2510_05186_b200.engine import Base
    inst, orders, off, LocalSearch, SearchConfig = _setup(cfg)
    n = 1024
    ls = LocalSearch(inst, orders, off, SearchConfig(seed=SEED, neighbours=n, shift_permille=PERMILLE,
                                                     max_shift=MAXSHIFT, share_prefix=True))
    o, mk = ls.materialize(0, n, 1)
    flags = ls.di.evaluate(o, mk, peak=False).flags.cpu().numpy()
    feas = [int(x) for x in np.nonzero(flags & 1)[0][:3]]
    dead = [int(x) for x in np.nonzero(flags & 2)[0][:2]]
    assert len(feas) == 3 and len(dead) == 2
    rb = Base(ls.di)
    rb.record(ls.inc_orders, ls.inc_mask)
    for idx in (feas[0], dead[0], feas[1], dead[1], feas[2]):
        rb.record(o[idx], mk[idx])
        _eval_both(ls.di, o, mk, rb)


def _base_tables(base, P, m, MW, vw=1):
    """A recorded base's tables with only what readers use: checkpoints up to the count, each
    with its state words, the live window slots and every lane's saved scalars (all but word 9,
    the widest window so far, a sizing hint).  `vw`: 32-bit words per ledger usage value."""
    from paper_2510_05186_b200 import _native as N
    info = np.frombuffer(base.read(N.BASE_INFO), np.int32).copy()
    res = np.frombuffer(base.read(N.BASE_RESULT), np.int64).copy()
    cstep = np.frombuffer(base.read(N.BASE_CSTEP), np.uint32).copy()
    fstep = np.frombuffer(base.read(N.BASE_FSTEP), np.uint32).copy()
    raw = np.frombuffer(base.read(N.BASE_CHECKPOINTS), np.uint32)
    ckw, ck_max, _, kc, ck_t, ck_u, ck_r, regw = np.frombuffer(base.read(N.BASE_LAYOUT), np.int32).tolist()
    nz = 2 * P * m + 3 * P * MW
    cks = []
    for c in range(max(info[0], 0)):
        w = raw[c * ckw:(c + 1) * ckw]
        regs = w[ck_r:ck_r + regw * P].reshape(P, regw).copy()
        # an idle exclusive link's free time at or below the stage's is dead (the same_state
        # relaxation): a re-recording that converged under it keeps its predecessor's shifted value
        dead = (regs[:, 5] == 0) & (regs[:, 6] == 0) & (regs[:, 2] <= regs[:, 1])
        regs[dead, 2] = 0xFFFFFFFF
        win = [(w[ck_t + s * kc: ck_t + s * kc + regs[s, 4]].tolist(),
                w[ck_u + vw * s * kc: ck_u + vw * (s * kc + regs[s, 4])].tolist()) for s in range(P)]
        # word 20 (the event step) is warp-wide: every lane's copy, not just the stage lanes'
        steps = w[ck_r:ck_r + regw * 32].reshape(32, regw)[:, 20].tolist()
        cks.append((w[:nz].tolist(), regs[:, list(range(9)) + list(range(10, 21))].tolist(), win, steps))
    return info[[0, 1, 2, 3]].tolist(), res.tolist(), cstep.tolist(), fstep.tolist(), cks


@pytest.mark.parametrize("cfg", [2, 3])
def test_rerecording_equals_fresh_recording(cuda_ok, cfg):
    """A base re-recorded over its predecessor — resumed from the predecessor's checkpoints and,
    where it converges onto it, finished by shifting the predecessor's later checkpoints — leaves
    exactly the tables a fresh recording does."""
    import torch
    from paper_2510_05186_b200.engine import Base
    inst, orders, off, LocalSearch, SearchConfig = _setup(cfg)
    n = 512
    ls = LocalSearch(inst, orders, off, SearchConfig(seed=SEED, neighbours=n, shift_permille=PERMILLE,
                                                     max_shift=MAXSHIFT, share_prefix=True))
    pk = ls.di.packed
    P, m, MW = pk.num_stages, pk.num_microbatches, (pk.num_microbatches + 31) // 32
    o, mk = ls.materialize(0, n, 2)
    r = ls.di.evaluate(o, mk, peak=False)
    torch.cuda.synchronize()
    flags, spans = r.flags.cpu().numpy(), r.makespan.cpu().numpy()
    feas = np.nonzero(flags & 1)[0]
    order = feas[np.argsort(spans[feas], kind="stable")]
    picks = [int(x) for x in list(order[:4]) + list(order[-2:])] + [int(np.nonzero(flags & 2)[0][0])]
    for idx in picks:
        fresh, again = Base(ls.di), Base(ls.di)
        fresh.record(o[idx], mk[idx])
        again.record(ls.inc_orders, ls.inc_mask)
        again.record(o[idx], mk[idx])
        assert _base_tables(fresh, P, m, MW) == _base_tables(again, P, m, MW), idx


@pytest.mark.timeout(300)
def test_long_search_with_converging_rerecordings(cuda_ok):
    """Forty rounds on config 3: every improvement re-records the base, most by converging onto
    the previous one and shifting its checkpoints; candidates then resume from shifted ones.  The
    search must run through and end on a valid schedule with the makespan it reports."""
    from paper_2510_05186_b200 import makespan, validate
    inst, orders, off, LocalSearch, SearchConfig = _setup(3)
    ls = LocalSearch(inst, orders, off, SearchConfig(seed=SEED, neighbours=8192, shift_permille=PERMILLE,
                                                     max_shift=MAXSHIFT))
    res = ls.run(rounds=40)
    assert len(res.improvements) >= 10
    assert validate(res.schedule, inst).ok and makespan(res.schedule, inst) == res.makespan


def test_host_buffer_path_matches_device_path(cuda_ok):
    """ps_eval_batch_host (chunked, copies overlapped) == ps_eval_batch on the same candidates."""
    import torch
    inst, orders, off, LocalSearch, SearchConfig = _setup(3)
    n = 20000                      # several pipeline chunks
    ls = LocalSearch(inst, orders, off, SearchConfig(seed=SEED, neighbours=n))
    o, mk = ls.materialize(0, n, 0)
    dev = ls.di.evaluate(o, mk, peak=True)
    torch.cuda.synchronize()
    h_o = o.cpu().numpy()
    h_m = mk.cpu().numpy()
    h_o8 = h_o.astype(np.uint8)                      # m = 64: op codes fit in one byte
    assert (h_o8.astype(np.int16) == h_o).all()
    for base, ho in ((None, h_o), (ls.base, h_o), (None, h_o8), (ls.base, h_o8)):
        host = ls.di.evaluate_host(ho, h_m, peak=True, base=base)
        assert (host.flags == dev.flags.cpu().numpy()).all()
        assert (host.makespan == dev.makespan.cpu().numpy()).all()
        assert (host.peak == dev.peak.cpu().numpy()).all()


def test_search_resumes_from_a_checkpoint(cuda_ok):
    """state_dict / load_state_dict: a search stopped after 3 rounds and resumed in a new
    LocalSearch follows the uninterrupted one exactly."""
    inst, orders, off, LocalSearch, SearchConfig = _setup(2)
    cfg = SearchConfig(seed=SEED, neighbours=2048, shift_permille=PERMILLE, max_shift=MAXSHIFT)
    full = LocalSearch(inst, orders, off, cfg)
    full.run(rounds=6)
    part = LocalSearch(inst, orders, off, cfg)
    part.run(rounds=3)
    state = part.state_dict()
    resumed = LocalSearch(inst, orders, off, cfg)
    resumed.load_state_dict(state)
    resumed.run(rounds=6)
    assert resumed.makespan == full.makespan
    assert [(i.round, i.makespan, i.index) for i in resumed.improvements] == \
        [(i.round, i.makespan, i.index) for i in full.improvements]
    assert (resumed.inc_orders.cpu() == full.inc_orders.cpu()).all()


SANITIZER_SCRIPT = (
    "import sys; sys.path.insert(0, %r)\n"
    "import numpy as np, torch\n"
    "from paper_2510_05186_b200 import workloads\n"
    "from paper_2510_05186_b200.heuristics import best_feasible\n"
    "from paper_2510_05186_b200.listsched import stage_order_of\n"
    "from paper_2510_05186_b200.search import LocalSearch, SearchConfig\n"
    "from paper_2510_05186_b200.bound import lower_bounds\n"
    "inst = workloads.CONFIGS[2]()\n"
    "s, _ = best_feasible(inst)\n"
    "o = {i: stage_order_of(s, i) for i in range(1, inst.num_stages + 1)}\n"
    "ls = LocalSearch(inst, o, s.offloaded, SearchConfig(seed=1, neighbours=512, kick_moves=2))\n"
    "ls.run(rounds=3)\n"
    "ls.kick()\n"
    "ls.run(rounds=5)\n"
    "od, md = ls.materialize(0, 256)\n"
    "ho = od.cpu().numpy().view(np.uint16).copy()\n"
    "ho[1, 0, 1] = ho[1, 0, 0]\n"                 # a repeated op: the literal replay pass
    "ls.di.evaluate_host(ho.astype(np.uint8), md.cpu().numpy(), base=ls.base)\n"
    "ls.di.evaluate_host(ho.astype(np.uint8), md.cpu().numpy(), base=None)\n"      # full-simulation build
    "from paper_2510_05186_b200.packing import delta_encode\n"                     # delta batch: moves + general
    "ro, rm = ls.inc_orders.cpu().numpy().view(np.uint16), ls.inc_mask.cpu().numpy().view(np.uint32)\n"
    "ls.di.evaluate_host_delta(ro, rm, *delta_encode(ro, rm, ho, md.cpu().numpy()), base=ls.base)\n"
    "print(lower_bounds(inst, [(0, {i: 0 for i in range(1, inst.num_stages + 1)}, {})]))\n"
    "for c, n in ((4, 64), (5, 32)):\n"                                              # global-state kernels
    "    i2 = workloads.CONFIGS[c]()\n"
    "    s2, _ = best_feasible(i2)\n"
    "    l2 = LocalSearch(i2, {i: stage_order_of(s2, i) for i in range(1, i2.num_stages + 1)}, s2.offloaded,\n"
    "                     SearchConfig(seed=1, neighbours=n))\n"
    "    l2.run(rounds=2)\n"
    "from paper_2510_05186_b200 import make_uniform_instance\n"                    # 64-bit completion
    "best_feasible(make_uniform_instance(4, 8, 20000000, 20000000, 20000000, 5, 1000, 2, 4))\n"
)


@pytest.mark.timeout(1200)
@pytest.mark.parametrize("tool", ["memcheck", "synccheck"])
def test_kernels_are_sanitizer_clean(cuda_ok, tool):
    """compute-sanitizer memcheck / synccheck over a recording, bounded search rounds, an ILS kick,
    a host-buffer batch with a malformed row (the literal replay kernel) and the node bounds
    (sanitizers on the GPU box)."""
    import os
    import shutil
    import subprocess
    import sys
    san = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not os.path.exists(san):
        pytest.skip("compute-sanitizer not installed")
    script = SANITIZER_SCRIPT % str(Path(__file__).resolve().parents[1])
    r = subprocess.run([san, "--tool", tool, "--error-exitcode", "3", "--print-limit", "5",
                        sys.executable, "-c", script], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]


def test_iterated_local_search_follows_the_cpu_restatement(cuda_ok):
    """ILS: descents, kicks from the best, the same improvement trail and the same
    best structure as the CPU restatement (tests/_search_cpu.py)."""
    from _search_cpu import cpu_search
    from oracle.oracle import Oracle
    inst, orders, off, LocalSearch, SearchConfig = _setup(2)
    n, kicks, km = 1024, 3, 4
    ls = LocalSearch(inst, orders, off, SearchConfig(seed=SEED, neighbours=n, shift_permille=PERMILLE,
                                                     max_shift=MAXSHIFT, kick_moves=km))
    orc = Oracle(ls.di.packed)
    want = cpu_search(orc, ls.inc_orders.cpu().numpy().view(np.uint16), ls.inc_mask.cpu().numpy().view(np.uint32),
                      SEED, PERMILLE, MAXSHIFT, n, kick_moves=km, kicks=kicks)
    res = ls.run(kicks=kicks)
    assert [(i.round, i.makespan, i.index) for i in res.improvements] == want["trail"]
    assert (ls.round, ls.kicks) == (want["rounds"], want["kicks"])
    assert res.makespan == want["best_span"] < ls.initial_makespan
    assert (ls.best_orders.cpu().numpy().view(np.uint16) == want["best_orders"]).all()
    assert (ls.best_mask.cpu().numpy().view(np.uint32) == want["best_mask"]).all()
    from paper_2510_05186_b200 import makespan, validate
    assert validate(res.schedule, inst).ok and makespan(res.schedule, inst) == res.makespan


def _channel_search(n=512):
    from paper_2510_05186_b200 import workloads
    from paper_2510_05186_b200.heuristics import best_feasible
    from paper_2510_05186_b200.search import ChannelSearch, SearchConfig
    inst = workloads.config2()
    s, _ = best_feasible(inst)
    cs = ChannelSearch.from_schedule(inst, s, SearchConfig(seed=SEED, neighbours=n, shift_permille=400,
                                                           max_shift=MAXSHIFT))
    return inst, s, cs


def test_channel_search_moves_match_the_cpu_restatement(cuda_ok):
    """Channel-order neighbours (stage-op shifts and transfer shifts within a channel, DESIGN.md
    §4.2) decoded on the device equal or_neighbour_explicit's, and the explicit replay of the warm
    schedule's channel orders reproduces its makespan."""
    from oracle.oracle import Oracle, neighbour_explicit
    from paper_2510_05186_b200 import makespan
    inst, s, cs = _channel_search()
    assert cs.makespan == makespan(s, inst)
    orc = Oracle(cs.di.packed)
    inc_o = cs.inc_orders.cpu().numpy().view(np.uint16)
    inc_m = cs.inc_mask.cpu().numpy().view(np.uint32)
    inc_c = cs.inc_chan.cpu().numpy().view(np.uint32)
    kinds = set()
    for rnd in (0, 7):
        o, mk, ch = cs.materialize(0, 512, rnd)
        o, mk, ch = (t.cpu().numpy().view(dt) for t, dt in ((o, np.uint16), (mk, np.uint32), (ch, np.uint32)))
        for idx in range(512):
            t, oo, mm, cc = neighbour_explicit(orc, inc_o, inc_m, inc_c, SEED, 400, MAXSHIFT, rnd, idx)
            kinds.add(t)
            assert (oo == o[idx]).all() and (mm == mk[idx]).all() and (cc == ch[idx]).all(), (rnd, idx, t)
    assert kinds == {0, 1, 3}


def test_channel_search_rounds_and_trail_match_the_cpu_restatement(cuda_ok):
    import torch
    from oracle.oracle import Oracle, search_round_explicit
    inst, s, cs = _channel_search(n=1024)
    orc = Oracle(cs.di.packed)
    inc_o = cs.inc_orders.cpu().numpy().view(np.uint16)
    inc_m = cs.inc_mask.cpu().numpy().view(np.uint32)
    inc_c = cs.inc_chan.cpu().numpy().view(np.uint32)
    ms = torch.empty(1024, dtype=torch.int64, device="cuda")
    cs.launch_round(ms)
    best, want = search_round_explicit(orc, inc_o, inc_m, inc_c, SEED, 400, MAXSHIFT, 0, 0, 1024, want_makespans=True)
    assert (ms.cpu().numpy() == want).all()
    assert int(cs.best_key.item()) == best
    # a whole search: same adopted moves as the CPU restatement
    from oracle.oracle import neighbour_explicit
    span, trail = cs.makespan, []
    for rnd in range(6):
        b, _ = search_round_explicit(orc, inc_o, inc_m, inc_c, SEED, 400, MAXSHIFT, rnd, 0, 1024)
        if b != (1 << 63) - 1 and (b >> 32) < span:
            span = b >> 32
            _, inc_o, inc_m, inc_c = neighbour_explicit(orc, inc_o, inc_m, inc_c, SEED, 400, MAXSHIFT, rnd,
                                                        b & 0xFFFFFFFF)
            trail.append((rnd, span))
    res = cs.run(rounds=6)
    assert [(i.round, i.makespan) for i in res.improvements] == trail and len(trail) > 0
    assert (cs.inc_chan.cpu().numpy().view(np.uint32) == inc_c).all()
    from paper_2510_05186_b200 import makespan, validate
    assert validate(res.schedule, inst).ok and makespan(res.schedule, inst) == span


@pytest.mark.parametrize("cfg", [2, 3, 4])
def test_channel_search_prefix_sharing_is_exact(cuda_ok, cfg):
    """Channel-order search with the incumbent recorded in explicit channel mode (checkpoints with
    channel cursors, per-position commit steps) against the same search with every
    neighbour simulated in full: equal makespans for every neighbour of every round, the same
    adopted moves, the same final channel orders — across re-recordings of the incumbent."""
    import torch
    from paper_2510_05186_b200 import workloads
    from paper_2510_05186_b200.heuristics import best_feasible
    from paper_2510_05186_b200.search import ChannelSearch, SearchConfig
    inst = workloads.CONFIGS[cfg]()
    s, _ = best_feasible(inst)
    n = 8192 if cfg != 4 else 2048
    runs = []
    for share in (True, False):
        cs = ChannelSearch.from_schedule(inst, s, SearchConfig(seed=SEED, neighbours=n, shift_permille=400,
                                                               max_shift=MAXSHIFT, share_prefix=share))
        spans = []
        for _ in range(8):
            ms = torch.empty(n, dtype=torch.int64, device="cuda")
            cs.launch_round(ms)
            spans.append(ms.cpu().numpy())
            cs.step()            # (runs the round again, then adopts its winner and re-records)
        runs.append((spans, [(i.round, i.makespan) for i in cs.improvements], cs.inc_chan.cpu().numpy().copy()))
    (a, ta, ca), (b, tb, cb) = runs
    for r, (x, y) in enumerate(zip(a, b)):
        assert (x == y).all(), (cfg, r, int((x != y).sum()))
    assert ta == tb and len(ta) >= 1
    assert (ca == cb).all()


@pytest.mark.parametrize("late", [False, True])
def test_bound_pruning_keeps_every_round_decision(cuda_ok, late):
    """Search rounds with the incumbent's makespan as cutoff abandon neighbours
    whose bound reaches it; a round's adopted move (a strict improvement) is the same as with every
    neighbour simulated — config 3, from the warm start and from the late incumbent."""
    import ctypes as C
    import torch
    from paper_2510_05186_b200 import _native as N
    from paper_2510_05186_b200.search import improves
    inst, orders, off, LocalSearch, SearchConfig = _setup(3)
    ls = LocalSearch(inst, orders, off, SearchConfig(seed=SEED, neighbours=65536))
    if late:
        z = np.load(Path(__file__).parent / "golden" / "inc320_config3.npz")
        ls.inc_orders.copy_(torch.from_numpy(z["orders"].view(np.int16)))
        ls.inc_mask.copy_(torch.from_numpy(z["mask"].view(np.int32)))
        ls.base.record(ls.inc_orders, ls.inc_mask)
        r = ls.di.evaluate(ls.inc_orders.view(1, *ls.inc_orders.shape), ls.inc_mask.view(1, -1), peak=False)
        ls.makespan = int(r.makespan[0].item())
    stream = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    adopted = 0
    for rnd in range(6):
        keys = []
        for cutoff in (0, ls.makespan):
            k = torch.full((1,), N.BEST_NONE, dtype=torch.int64, device="cuda")
            desc = N.SearchDesc(ls.inc_orders.data_ptr(), ls.inc_mask.data_ptr(), rnd, 0, 65536, ls.moves, None,
                                ls.base.handle, 1, cutoff)
            N.check(ls.lib.ps_search_round(ls.di.handle, C.byref(desc), C.c_void_p(k.data_ptr()), None, stream))
            keys.append(int(k.item()))
        full, pruned = keys
        assert improves(full, ls.makespan) == improves(pruned, ls.makespan), rnd
        if improves(full, ls.makespan):
            assert full == pruned
            adopted += 1
            ls.best_key.fill_(full)
            ls.round = rnd
            ls.finish_round()
    assert adopted >= 1 or late


@pytest.mark.parametrize("cfg", [2, 3])
def test_pruned_descent_follows_the_full_trail(cuda_ok, cfg):
    """SearchConfig(prune=True) against the default: the whole descent to convergence adopts the
    same moves (same improvement trail and final structure)."""
    inst, orders, off, LocalSearch, SearchConfig = _setup(cfg)
    runs = []
    for prune in (False, True):
        ls = LocalSearch(inst, orders, off, SearchConfig(seed=SEED, neighbours=65536, prune=prune))
        while ls.stale < 16 and ls.round < 3000:
            ls.step()
        o, m = ls.incumbent_structure()
        runs.append(([(i.round, i.makespan, i.index) for i in ls.improvements], ls.round, o, m))
    assert runs[0] == runs[1]
    assert len(runs[0][0]) > 3


@pytest.mark.parametrize("late", [False, True])
def test_suffix_sharing_equals_full_simulation(cuda_ok, late):
    """Every neighbour of config-3 search rounds (65,536 each, from the warm start and from the late
    incumbent, where the convergence rules for finished stages and idle links matter most): its
    makespan with prefix/suffix sharing against the recorded incumbent equals its full simulation,
    and so does the peak of every stage on a materialised sample."""
    import ctypes as C
    import torch
    from paper_2510_05186_b200 import _native as N
    inst, orders, off, LocalSearch, SearchConfig = _setup(3)
    n = 65536
    ls = LocalSearch(inst, orders, off, SearchConfig(seed=SEED, neighbours=n, shift_permille=PERMILLE,
                                                     max_shift=MAXSHIFT))
    if late:
        z = np.load(Path(__file__).parent / "golden" / "inc320_config3.npz")
        ls.inc_orders.copy_(torch.from_numpy(z["orders"].view(np.int16)))
        ls.inc_mask.copy_(torch.from_numpy(z["mask"].view(np.int32)))
        ls.base.record(ls.inc_orders, ls.inc_mask)
    stream = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    for rnd in (0, 1):
        got = []
        for base in (ls.base, None):
            out = torch.empty(n, dtype=torch.int64, device="cuda")
            ls.best_key.fill_(N.BEST_NONE)
            desc = N.SearchDesc(ls.inc_orders.data_ptr(), ls.inc_mask.data_ptr(), rnd, 0, n, ls.moves, None,
                                base.handle if base is not None else None)
            N.check(ls.lib.ps_search_round(ls.di.handle, C.byref(desc), C.c_void_p(ls.best_key.data_ptr()),
                                           C.c_void_p(out.data_ptr()), stream))
            torch.cuda.synchronize()
            got.append((out.cpu().numpy(), int(ls.best_key.item())))
        (a, ka), (b, kb) = got
        assert (a == b).all(), (rnd, int((a != b).sum()))
        assert ka == kb
    # peaks and bubbles: materialised neighbours with and without the base
    o, mk = ls.materialize(0, 4096, 0)
    _eval_both(ls.di, o, mk, ls.base)


@pytest.mark.parametrize("cfg", [2, 3])
def test_materialised_search_rounds_equal_the_move_encoded_ones(cuda_ok, cfg, monkeypatch):
    """An incumbent too large for shared memory (P = 32, m above ~1,100) is searched by
    materialising the neighbours in chunks (search_round_rows in ps_abi.cu); forced here with
    PS_SEARCH_ROWS=1 on configs 2/3: every neighbour's makespan of a round, and a whole descent's
    trail and final structure, equal the move-encoded search's."""
    import torch
    inst, orders, off, LocalSearch, SearchConfig = _setup(cfg)
    n = 4096
    runs = []
    for rows in ("0", "1"):
        monkeypatch.setenv("PS_SEARCH_ROWS", rows)
        ls = LocalSearch(inst, orders, off, SearchConfig(seed=SEED, neighbours=n))
        ms = torch.empty(n, dtype=torch.int64, device="cuda")
        ls.launch_round(ms)
        torch.cuda.synchronize()
        first = ms.cpu().numpy().copy()
        ls.finish_round()
        while ls.stale < 8 and ls.round < 60:
            ls.step()
        o, mk = ls.incumbent_structure()
        runs.append((first, [(i.round, i.makespan, i.index) for i in ls.improvements], ls.round, o, mk))
    assert (runs[0][0] == runs[1][0]).all()
    assert runs[0][1:] == runs[1][1:] and len(runs[0][1]) > 3
