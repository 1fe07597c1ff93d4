"""Diagnostic: shared vs unshared evaluation of config-N neighbours; print the disagreements."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from paper_2510_05186_b200 import workloads  # noqa: E402
from paper_2510_05186_b200.heuristics import best_feasible  # noqa: E402
from paper_2510_05186_b200.listsched import stage_order_of  # noqa: E402
from paper_2510_05186_b200.search import LocalSearch, SearchConfig  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
inst = workloads.CONFIGS[cfg]()
s0, _ = best_feasible(inst)
orders = {i: stage_order_of(s0, i) for i in range(1, inst.num_stages + 1)}
n = int(os.environ.get("NCAND", "1024"))
ls = LocalSearch(inst, orders, s0.offloaded, SearchConfig(seed=11, neighbours=n, shift_permille=700, max_shift=4))
o, mk = ls.materialize(0, n, 0)
for rep in range(int(os.environ.get("REPS", "3"))):
    r0 = ls.di.evaluate(o, mk, peak=True)
    r1 = ls.di.evaluate(o, mk, peak=True, base=ls.base)
    torch.cuda.synchronize()
    f0, f1 = r0.flags.cpu().numpy(), r1.flags.cpu().numpy()
    m0, m1 = r0.makespan.cpu().numpy(), r1.makespan.cpu().numpy()
    bad = np.nonzero((f0 != f1) | (m0 != m1))[0]
    print("rep", rep, "mismatches", len(bad), [(int(k), int(f0[k]), int(f1[k]), int(m0[k]), int(m1[k])) for k in bad[:8]])
