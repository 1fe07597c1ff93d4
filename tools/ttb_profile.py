"""Diagnostic: per-round cost along a whole search (config 3): kernel ms and simulated events."""
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

cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 3
rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 520
inst = workloads.CONFIGS[cfg_id]()
s0, _ = best_feasible(inst)
orders = {i: stage_order_of(s0, i) for i in range(1, inst.num_stages + 1)}
ls = LocalSearch(inst, orders, s0.offloaded, SearchConfig(seed=20251005, neighbours=65536, shift_permille=700, max_shift=4))
ev = torch.zeros(2, dtype=torch.int64, device="cuda")
stream = torch.cuda.current_stream()
rows = []
t0 = time.perf_counter()
for r in range(rounds):
    ev.zero_()
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    ls.best_key.fill_(N.BEST_NONE)
    desc = N.SearchDesc(ls.inc_orders.data_ptr(), ls.inc_mask.data_ptr(), ls.round, 0, ls.count, ls.moves,
                        ev.data_ptr(), ls.base.handle)
    e0.record()
    N.check(ls.lib.ps_search_round(ls.di.handle, C.byref(desc), C.c_void_p(ls.best_key.data_ptr()), None,
                                   C.c_void_p(stream.cuda_stream)))
    e1.record()
    imp = ls.finish_round(t0)
    e2.record()
    torch.cuda.synchronize()
    rows.append((r, e0.elapsed_time(e1), e1.elapsed_time(e2), int(ev[0]), ls.makespan, imp))
wall = time.perf_counter() - t0
for r in rows[::40] + rows[-3:]:
    print("round %4d kernel %7.2f ms  finish %6.2f ms  sim events/cand %6.1f  makespan %d  improved %s" %
          (r[0], r[1], r[2], r[3] / 65536, r[4], r[5]))
print("wall", wall, "sum kernel", sum(r[1] for r in rows) / 1e3, "sum finish", sum(r[2] for r in rows) / 1e3)
if len(sys.argv) > 3:
    import numpy as np
    np.savez(sys.argv[3], orders=ls.inc_orders.cpu().numpy().view(np.uint16), mask=ls.inc_mask.cpu().numpy().view(np.uint32))
