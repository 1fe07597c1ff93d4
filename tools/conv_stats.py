"""Diagnostic (PS_LIBRARY=<-DPS_DEBUG_CONV build>): why suffix-sharing compares fail."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2510_05186_b200 import _native as N, workloads  # noqa: E402
from paper_2510_05186_b200.heuristics import best_feasible  # noqa: E402
from paper_2510_05186_b200.listsched import stage_order_of  # noqa: E402
from paper_2510_05186_b200.search import LocalSearch, SearchConfig  # noqa: E402

inst = workloads.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 3]()
s0, _ = best_feasible(inst)
orders = {i: stage_order_of(s0, i) for i in range(1, inst.num_stages + 1)}
n = 65536
ls = LocalSearch(inst, orders, s0.offloaded, SearchConfig(seed=20251005, neighbours=n, shift_permille=700, max_shift=4))
if os.environ.get("KVAR_INCUMBENT"):
    import numpy as np
    z = np.load(os.environ["KVAR_INCUMBENT"])
    ls.inc_orders.copy_(torch.from_numpy(z["orders"].view(np.int16)))
    ls.inc_mask.copy_(torch.from_numpy(z["mask"].view(np.int32)))
    ls.base.record(ls.inc_orders, ls.inc_mask)
ev = torch.zeros(16, dtype=torch.int64, device="cuda")
ls.best_key.fill_(N.BEST_NONE)
desc = N.SearchDesc(ls.inc_orders.data_ptr(), ls.inc_mask.data_ptr(), 0, 0, n, ls.moves, ev.data_ptr(), ls.base.handle)
N.check(ls.lib.ps_search_round(ls.di.handle, C.byref(desc), C.c_void_p(ls.best_key.data_ptr()), None,
                               C.c_void_p(torch.cuda.current_stream().cuda_stream)))
torch.cuda.synchronize()
names = ["pos", "sfree shift", "cfree", "window count", "pending counts", "first_start", "base/top",
         "end-time words", "pending bitsets", "window contents", "ok if finished stages exempt", "converged"]
v = ev.cpu().tolist()
print("simulated", v[0], "algorithmic", v[1])
for k, nm in enumerate(names):
    if v[2 + k]:
        print(f"{nm:16s} {v[2 + k]}")
