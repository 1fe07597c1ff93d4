"""Kernel launch-plan experiments: time search rounds / materialised batches under env knobs."""
import ctypes as C
import itertools
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2510_05186_b200 import _native as N, workloads  # noqa: E402
from paper_2510_05186_b200.heuristics import best_feasible  # noqa: E402
from paper_2510_05186_b200.listsched import stage_order_of  # noqa: E402
from paper_2510_05186_b200.search import LocalSearch, SearchConfig  # noqa: E402


def main():
    cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 65536
    inst = workloads.CONFIGS[cfg_id]()
    s0, _ = best_feasible(inst)
    orders = {i: stage_order_of(s0, i) for i in range(1, inst.num_stages + 1)}
    ls = LocalSearch(inst, orders, s0.offloaded, SearchConfig(seed=1, neighbours=n))
    stream = torch.cuda.current_stream()
    od, md = ls.materialize(0, n)
    grid = [(1, win, warps) for win in [int(x) for x in os.environ.get('KEXP_WINDOWS', '16').split(',')] for warps in (4,)]
    for (segs, win, warps), share in [(g, sh) for g in grid for sh in (False, True)]:
        os.environ["PS_SEGS_PER_WARP"] = str(segs)
        os.environ["PS_WINDOW"] = str(win)
        os.environ["PS_WARPS_PER_BLOCK"] = str(warps)
        res = {}
        for mode in ("search", "materialized"):
            ts = []
            for rep in range(3):
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                if mode == "search":
                    ls.best_key.fill_(N.BEST_NONE)
                    desc = N.SearchDesc(ls.inc_orders.data_ptr(), ls.inc_mask.data_ptr(), 0, 0, n, ls.moves, None,
                                        ls.base.handle if (share and ls.base is not None) else None)
                    N.check(ls.lib.ps_search_round(ls.di.handle, C.byref(desc), C.c_void_p(ls.best_key.data_ptr()),
                                                   None, C.c_void_p(stream.cuda_stream)))
                else:
                    ls.di.evaluate(od, md, peak=True, base=ls.base if share else None)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            res[mode] = min(ts)
        print(json.dumps({"share": share, "lib": os.path.basename(os.environ.get("PS_LIBRARY", "default")), "config": cfg_id, "segs": segs, "window": win, "warps": warps,
                          "search_ms": round(res["search"], 3), "mat_ms": round(res["materialized"], 3),
                          "search_cps": round(n / res["search"] * 1e3), "mat_cps": round(n / res["materialized"] * 1e3)}),
              flush=True)


if __name__ == "__main__":
    main()
