"""Diagnostic (PS_LIBRARY=<-DPS_DEBUG_EVENTS build>): simulated events per neighbour by outcome."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from oracle.oracle import Oracle  # noqa: E402
from paper_2510_05186_b200 import workloads  # noqa: E402
from paper_2510_05186_b200.heuristics import best_feasible  # noqa: E402
from paper_2510_05186_b200.listsched import stage_order_of  # noqa: E402
from paper_2510_05186_b200.search import LocalSearch, SearchConfig  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
inst = workloads.CONFIGS[cfg]()
s0, _ = best_feasible(inst)
orders = {i: stage_order_of(s0, i) for i in range(1, inst.num_stages + 1)}
n = 8192
ls = LocalSearch(inst, orders, s0.offloaded, SearchConfig(seed=20251005, neighbours=n, shift_permille=700, max_shift=4))
if os.environ.get("KVAR_INCUMBENT"):
    z = np.load(os.environ["KVAR_INCUMBENT"])
    ls.inc_orders.copy_(torch.from_numpy(z["orders"].view(np.int16)))
    ls.inc_mask.copy_(torch.from_numpy(z["mask"].view(np.int32)))
    ls.base.record(ls.inc_orders, ls.inc_mask)
o, mk = ls.materialize(0, n, 0)
r = ls.di.evaluate(o, mk, base=ls.base, out=ls.di.alloc_results(n, peak=False, blocked=False))
torch.cuda.synchronize()
bl = r.bubble.cpu().numpy().astype(np.uint32)
ev, e0 = bl & 0xFFFF, bl >> 16
fl = r.flags.cpu().numpy()
orc = Oracle(ls.di.packed)
inc_o = ls.inc_orders.cpu().numpy().view(np.uint16)
inc_m = ls.inc_mask.cpu().numpy().view(np.uint32)
mt = np.array([orc.neighbour(inc_o, inc_m, 20251005, 700, 4, 0, k)[0] for k in range(n)])
base_events = 3 * inst.num_stages * inst.num_microbatches
print("mean simulated events", ev.mean(), "median", np.median(ev))
for name, sel in [("feasible", (fl & 1) == 1), ("deadlock", (fl & 2) == 2), ("shift", mt == 1), ("toggle", mt == 2), ("noop", mt == 0)]:
    if sel.any():
        print(f"{name:9s} n={sel.sum():5d} share={sel.mean():.3f} mean_ev={ev[sel].mean():7.1f} p50={np.median(ev[sel]):6.0f} p90={np.percentile(ev[sel], 90):6.0f} max={ev[sel].max():5d} restored_at_mean={e0[sel].mean():7.1f}")
h = np.histogram(ev, bins=[0, 1, 16, 32, 64, 128, 256, 512, 1024, 4096, 65536])
print("histogram", list(zip(h[1][:-1].tolist(), h[0].tolist())))
print("share of all simulated events by bucket:", [round(float(ev[(ev >= a) & (ev < b)].sum() / ev.sum()), 3) for a, b in zip(h[1][:-1], h[1][1:])])
