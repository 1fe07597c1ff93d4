"""Evaluate one round's 65,536 neighbours (config 3) as a generic materialised batch with no base:
the path of e2e_no_base, for ncu.   python tools/nobase_batch.py [config] [n]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2510_05186_b200 import workloads  # noqa: E402
from paper_2510_05186_b200.heuristics import best_feasible  # noqa: E402
from paper_2510_05186_b200.listsched import stage_order_of  # noqa: E402
from paper_2510_05186_b200.search import LocalSearch, SearchConfig  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
n = int(sys.argv[2]) if len(sys.argv) > 2 else 65536
inst = workloads.CONFIGS[cfg]()
s0, _ = best_feasible(inst)
orders = {i: stage_order_of(s0, i) for i in range(1, inst.num_stages + 1)}
ls = LocalSearch(inst, orders, s0.offloaded, SearchConfig(seed=20251005, neighbours=n))
o, mk = ls.materialize(0, n, 5)
for _ in range(3):
    r = ls.di.evaluate(o, mk, peak=True)
torch.cuda.synchronize()
print("feasible", int((r.flags & 1).sum().item()), "of", n)
