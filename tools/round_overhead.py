"""Where a search round's wall time goes beyond its kernels (host phases of LocalSearch.step)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2510_05186_b200 import workloads  # noqa: E402
from paper_2510_05186_b200.heuristics import best_feasible  # noqa: E402
from paper_2510_05186_b200.listsched import stage_order_of  # noqa: E402
from paper_2510_05186_b200.search import LocalSearch, SearchConfig  # noqa: E402

inst = workloads.config3()
s0, _ = best_feasible(inst)
ls = LocalSearch(inst, {i: stage_order_of(s0, i) for i in range(1, 9)}, s0.offloaded,
                 SearchConfig(seed=20251005, neighbours=65536, shift_permille=700, max_shift=4))
ls.run(rounds=5)
torch.cuda.synchronize()
T = {"launch": 0.0, "item": 0.0, "finish": 0.0}
ev = []
t_all = time.perf_counter()
R = 100
for _ in range(R):
    a = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ls.launch_round()
    e1.record()
    b = time.perf_counter()
    ls.best_key.item()
    c = time.perf_counter()
    ls.finish_round()
    d = time.perf_counter()
    T["launch"] += b - a
    T["item"] += c - b
    T["finish"] += d - c
    ev.append((e0, e1))
torch.cuda.synchronize()
wall = time.perf_counter() - t_all
gpu = sum(e0.elapsed_time(e1) for e0, e1 in ev) / 1e3
print({k: round(1000 * v / R, 3) for k, v in T.items()}, "wall ms/round", round(1000 * wall / R, 3),
      "gpu ms/round", round(1000 * gpu / R, 3))
