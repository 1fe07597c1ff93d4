"""Diagnostic: where the host-buffer evaluation's time goes (H2D alone, device eval alone, total)."""
import os
import sys
import time

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
h8 = torch.empty(od8.shape, dtype=torch.uint8, pin_memory=True)
h8.copy_(od8)
hm = torch.empty(md.shape, dtype=torch.int32, pin_memory=True)
hm.copy_(md)
dev8 = torch.empty_like(od8)


def t(fn, reps=5):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        a = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - a)
    return 1000 * sorted(ts)[len(ts) // 2]


print("h2d 8-bit orders  ms", t(lambda: dev8.copy_(h8, non_blocking=True)), "bytes", h8.numel())
print("eval device u8    ms", t(lambda: ls.di.evaluate(od8, md, peak=True, base=ls.base)))
print("eval device u16   ms", t(lambda: ls.di.evaluate(od, md, peak=True, base=ls.base)))
nb = ls.di.alloc_results(n, peak=True, blocked=False)
print("eval device u8 no blocked ms", t(lambda: ls.di.evaluate(od8, md, base=ls.base, out=nb)))
import ctypes as _C
from paper_2510_05186_b200 import _native as _N
bk = torch.empty(1, dtype=torch.int64, device="cuda")
def _search():
    bk.fill_(_N.BEST_NONE)
    d = _N.SearchDesc(ls.inc_orders.data_ptr(), ls.inc_mask.data_ptr(), 0, 0, n, ls.moves, None, ls.base.handle)
    ms = torch.empty(n, dtype=torch.int64, device="cuda")
    _N.check(ls.lib.ps_search_round(ls.di.handle, _C.byref(d), _C.c_void_p(bk.data_ptr()), _C.c_void_p(ms.data_ptr()),
                                    _C.c_void_p(torch.cuda.current_stream().cuda_stream)))
print("search round (same neighbours, makespans out) ms", t(_search))
print("eval device nobase ms", t(lambda: ls.di.evaluate(od8, md, peak=True)))
import numpy as np
ho, hmm = h8.numpy(), hm.numpy()
print("eval host u8      ms", t(lambda: ls.di.evaluate_host(ho, hmm, peak=True, base=ls.base)))
import ctypes as C  # noqa: E402
from paper_2510_05186_b200 import _native as N  # noqa: E402
pk = ls.di.packed
for nn in (64, 4096, 65536):
    hs = ho[:nn].copy() if nn < n else ho
    out = dict(ms=np.empty(nn, np.int64), bb=np.empty(nn, np.float64), fl=np.empty(nn, np.int32), pk=np.empty((nn, pk.num_stages), np.int64))
    hmm2 = hmm[:nn].copy() if nn < n else hmm
    cb = N.CandBatch(nn, hs.ctypes.data, hmm2.ctypes.data, None, 0, ls.base.handle, 1)
    rb = N.ResultBatch(out["ms"].ctypes.data, out["bb"].ctypes.data, out["pk"].ctypes.data, out["fl"].ctypes.data, None, None, None, 0, None)
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    print("host call N=%d (numpy pageable, no blocked)" % nn, "ms", t(lambda: N.check(ls.lib.ps_eval_batch_host(ls.di.handle, C.byref(cb), C.byref(rb), st))))
