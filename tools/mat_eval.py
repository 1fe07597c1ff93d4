"""Diagnostic: one materialised batch (65,536 config-3 neighbours, uint8 codes, base attached)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2510_05186_b200 import workloads  # noqa: E402
from paper_2510_05186_b200.heuristics import best_feasible  # noqa: E402
from paper_2510_05186_b200.listsched import stage_order_of  # noqa: E402
from paper_2510_05186_b200.search import LocalSearch, SearchConfig  # noqa: E402

inst = workloads.CONFIGS[3]()
s0, _ = best_feasible(inst)
orders = {i: stage_order_of(s0, i) for i in range(1, inst.num_stages + 1)}
n = 65536
ls = LocalSearch(inst, orders, s0.offloaded, SearchConfig(seed=20251005, neighbours=n, shift_permille=700, max_shift=4))
od, md = ls.materialize(0, n)
od8 = od.to(torch.uint8)
out = ls.di.alloc_results(n, peak=True, blocked=False)
for _ in range(3):
    ls.di.evaluate(od8, md, base=ls.base, out=out)
torch.cuda.synchronize()
