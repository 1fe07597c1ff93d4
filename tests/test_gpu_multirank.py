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
