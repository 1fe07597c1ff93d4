"""Diagnostic: simulated events and time, materialised batch vs search round on the same neighbours."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2510_05186_b200 import _native as N, workloads  # noqa: E402
from paper_2510_05186_b200.heuristics import best_feasible  # noqa: E402
from paper_2510_05186_b200.listsched import stage_order_of  # noqa: E402
from paper_2510_05186_b200.search import LocalSearch, SearchConfig  # noqa: E402

inst = workloads.CONFIGS[3]()
s0, _ = best_feasible(inst)
orders = {i: stage_order_of(s0, i) for i in range(1, inst.num_stages + 1)}
n = 65536
ls = LocalSearch(inst, orders, s0.offloaded, SearchConfig(seed=20251005, neighbours=n, shift_permille=700, max_shift=4))
od, md = ls.materialize(0, n, 0)
od8 = od.to(torch.uint8)
for mode in ("mat", "moves"):
    ev = torch.zeros(2, dtype=torch.int64, device="cuda")
    ts = []
    for rep in range(4):
        ev.zero_()
        torch.cuda.synchronize()
        t = time.perf_counter()
        if mode == "mat":
            out = ls.di.alloc_results(n, peak=True, blocked=False)
            cb = N.CandBatch(n, od8.data_ptr(), md.data_ptr(), None, 0, ls.base.handle, 1)
            rb = N.ResultBatch(out.makespan.data_ptr(), out.bubble.data_ptr(), out.peak.data_ptr(), out.flags.data_ptr(),
                               None, None, None, 0, ev.data_ptr())
            N.check(ls.lib.ps_eval_batch(ls.di.handle, C.byref(cb), C.byref(rb), C.c_void_p(torch.cuda.current_stream().cuda_stream)))
        else:
            ms = torch.empty(n, dtype=torch.int64, device="cuda")
            ls.best_key.fill_(N.BEST_NONE)
            d = N.SearchDesc(ls.inc_orders.data_ptr(), ls.inc_mask.data_ptr(), 0, 0, n, ls.moves, ev.data_ptr(), ls.base.handle)
            N.check(ls.lib.ps_search_round(ls.di.handle, C.byref(d), C.c_void_p(ls.best_key.data_ptr()), C.c_void_p(ms.data_ptr()),
                                           C.c_void_p(torch.cuda.current_stream().cuda_stream)))
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t)
    print(mode, "ms", round(1000 * sorted(ts)[1], 3), "simulated events", int(ev[0]), "algorithmic", int(ev[1]))
