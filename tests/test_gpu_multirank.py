"""The sharded bench path with two ranks (torchrun), both on the one GPU of a test box over gloo
(PS_SHARE_GPU=1): sharding, the all-reduce(MIN) of each round's key, max-over-ranks timing and the
rank-0 JSON line.  On a multi-GPU node the same path runs one rank per GPU over NCCL."""

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.timeout(600)
def test_two_rank_bench_line(cuda_ok):
    env = dict(os.environ, PS_SHARE_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29541", str(ROOT / "bench.py"), "--gpus", "2",
           "--steps", "3", "--warmup", "3", "--no-cpu", "--no-ttb", "--no-e2e"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=540, env=env, cwd=str(ROOT))
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{\"metric\"")]
    assert len(lines) == 1                       # rank 0 alone prints
    d = lines[0]
    assert d["n_gpus"] == 2 and d["config"]["candidates_per_round"] == 2 * d["config"]["candidates_per_gpu"]
    assert d["value"] > 0 and d["search"]["final_makespan"] < d["search"]["initial_makespan"]


def _run_world(tmp_path, world, cfg, n, rounds, kick_moves=0, kicks=0, port=29543):
    env = dict(os.environ, PS_SHARE_GPU="1")
    out = str(tmp_path / f"w{world}")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(world),
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(ROOT / "tests" / "_multirank_worker.py"),
           str(cfg), str(n), str(rounds), str(kick_moves), str(kicks), out]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env, cwd=str(ROOT))
    assert r.returncode == 0, r.stderr[-3000:]
    return [json.load(open(f"{out}.rank{k}.json")) for k in range(world)]


@pytest.mark.timeout(1200)
@pytest.mark.parametrize("kick_moves", [0, 4])
def test_one_and_two_ranks_follow_the_same_trajectory(cuda_ok, tmp_path, kick_moves):
    """Config 3, 8,192 neighbours per round in total: one rank, and two ranks owning half the
    indices each (gloo, both on cuda:0), adopt the same move every round (descent: 24 rounds;
    ILS: 2 kicks), end with the same best structure, and every rank agrees."""
    rounds, kicks = 24, 2
    one = _run_world(tmp_path, 1, 3, 8192, rounds, kick_moves, kicks, port=29543 + kick_moves)
    two = _run_world(tmp_path, 2, 3, 8192, rounds, kick_moves, kicks, port=29553 + kick_moves)
    assert [(d["first"], d["count"]) for d in two] == [(0, 4096), (4096, 4096)]
    ref = one[0]
    assert len(ref["trail"]) >= 5
    for d in two:
        for key in ("trail", "best", "rounds", "kicks", "orders", "mask"):
            assert d[key] == ref[key], (key, d["rank"])


@pytest.mark.timeout(1500)
def test_identical_best_schedule_at_1_2_4_8_ranks(cuda_ok, tmp_path):
    """BASELINE's "identical best schedule for equal search budgets" at 1, 2, 4 and 8 ranks
    (gloo, all on cuda:0): config 3, 8,192 neighbours per round in total, 16 descent rounds —
    every rank of every world size holds the same improvement trail and best structure."""
    runs = {w: _run_world(tmp_path, w, 3, 8192, 16, port=29571 + w) for w in (1, 2, 4, 8)}
    ref = runs[1][0]
    assert len(ref["trail"]) >= 5
    for w, docs in runs.items():
        assert [(d["first"], d["count"]) for d in docs] == [(k * 8192 // w, 8192 // w) for k in range(w)]
        for d in docs:
            for key in ("trail", "best", "rounds", "orders", "mask"):
                assert d[key] == ref[key], (w, key, d["rank"])


def test_sharded_round_through_the_c_abi_with_an_nccl_communicator(cuda_ok):
    """ps_search_round_sharded with the ncclComm_t of a one-rank NCCL group: the all-reduce(MIN)
    inside the C ABI call leaves the round's key as ps_search_round computes it."""
    import ctypes as C
    import socket
    import torch
    import torch.distributed as dist
    from paper_2510_05186_b200 import _native as N, workloads
    from paper_2510_05186_b200.heuristics import best_feasible
    from paper_2510_05186_b200.listsched import stage_order_of
    from paper_2510_05186_b200.search import LocalSearch, SearchConfig, nccl_comm_ptr
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        comm = nccl_comm_ptr(None, 0)
        assert comm
        inst = workloads.config2()
        s0, _ = best_feasible(inst, device=0)
        orders = {i: stage_order_of(s0, i) for i in range(1, inst.num_stages + 1)}
        ls = LocalSearch(inst, orders, s0.offloaded, SearchConfig(seed=3, neighbours=4096), device=0)
        stream = C.c_void_p(torch.cuda.current_stream().cuda_stream)
        keys = []
        for fn, extra in ((ls.lib.ps_search_round, ()), (ls.lib.ps_search_round_sharded, (C.c_void_p(comm),))):
            k = torch.full((1,), N.BEST_NONE, dtype=torch.int64, device="cuda")
            desc = N.SearchDesc(ls.inc_orders.data_ptr(), ls.inc_mask.data_ptr(), 0, 0, 4096, ls.moves, None,
                                ls.base.handle, 0)
            N.check(fn(ls.di.handle, C.byref(desc), C.c_void_p(k.data_ptr()), None, *extra, stream))
            keys.append(int(k.item()))
        assert keys[0] == keys[1] != N.BEST_NONE
    finally:
        dist.destroy_process_group()
