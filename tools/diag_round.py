import ctypes as C, os, sys, time, json
sys.path.insert(0, '/root/repo')
import torch
from paper_2510_05186_b200 import _native as N, workloads
from paper_2510_05186_b200.heuristics import best_feasible
from paper_2510_05186_b200.listsched import stage_order_of
from paper_2510_05186_b200.search import LocalSearch, SearchConfig
inst = workloads.config3()
s0, _ = best_feasible(inst)
orders = {i: stage_order_of(s0, i) for i in range(1, 9)}
ls = LocalSearch(inst, orders, s0.offloaded, SearchConfig(seed=20251005, neighbours=65536, shift_permille=700, max_shift=4))
st = torch.cuda.current_stream()
ev = torch.zeros(1, dtype=torch.int64, device='cuda')
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for variant in ("plain", "flush", "flush+nosync", "plain"):
    for rep in range(4):
        ls.best_key.fill_(N.BEST_NONE)
        desc = N.SearchDesc(ls.inc_orders.data_ptr(), ls.inc_mask.data_ptr(), ls.round, 0, 65536, ls.moves,
                            None, ls.base.handle)
        if 'flush' in variant:
            flush.fill_(rep & 0xFF)
        if 'nosync' not in variant:
            torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(st)
        N.check(ls.lib.ps_search_round(ls.di.handle, C.byref(desc), C.c_void_p(ls.best_key.data_ptr()), None, C.c_void_p(st.cuda_stream)))
        e1.record(st)
        th = time.perf_counter() - t0
        torch.cuda.synchronize()
        tw = time.perf_counter() - t0
        imp = False
        if variant == "events+advance":
            imp = ls.finish_round()
        print(json.dumps({"variant": variant, "gpu_ms": round(e0.elapsed_time(e1), 2), "host_call_ms": round(1e3*th, 2), "wall_ms": round(1e3*tw, 2), "improved": imp}), flush=True)
