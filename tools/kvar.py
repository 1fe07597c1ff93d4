"""Time one config's search round (65,536 neighbours, prefix/suffix sharing) per library variant.

  PS_LIBRARY=<variant .so> python tools/kvar.py [config] [n]   (prints one JSON line)
"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2510_05186_b200 import _native as N, workloads  # noqa: E402
from paper_2510_05186_b200.heuristics import best_feasible  # noqa: E402
from paper_2510_05186_b200.listsched import stage_order_of  # noqa: E402
from paper_2510_05186_b200.search import LocalSearch, SearchConfig  # noqa: E402

cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 3
n = int(sys.argv[2]) if len(sys.argv) > 2 else 65536
inst = workloads.CONFIGS[cfg_id]()
s0, _ = best_feasible(inst)
orders = {i: stage_order_of(s0, i) for i in range(1, inst.num_stages + 1)}
ls = LocalSearch(inst, orders, s0.offloaded, SearchConfig(seed=20251005, neighbours=n, shift_permille=int(os.environ.get("KVAR_SHIFT", 700)), max_shift=4))
if os.environ.get("KVAR_INCUMBENT"):
    # start from a saved incumbent (tools/ttb_profile.py ... <file.npz>) instead of the warm start
    import numpy as np
    z = np.load(os.environ["KVAR_INCUMBENT"])
    ls.inc_orders.copy_(torch.from_numpy(z["orders"].view(np.int16)))
    ls.inc_mask.copy_(torch.from_numpy(z["mask"].view(np.int32)))
    ls.base.record(ls.inc_orders, ls.inc_mask)
cutoff = 0
if os.environ.get("KVAR_PRUNE"):
    # the current point's makespan, as LocalSearch passes it
    r = ls.di.evaluate(ls.inc_orders[None], ls.inc_mask[None])
    cutoff = int(r.makespan[0].item())
dedup = int(os.environ.get("KVAR_DEDUP", "0"))
stream = torch.cuda.current_stream()
ev = torch.zeros(2, dtype=torch.int64, device="cuda")
ts = []
for rep in range(8):
    ev.zero_()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ls.best_key.fill_(N.BEST_NONE)
    desc = N.SearchDesc(ls.inc_orders.data_ptr(), ls.inc_mask.data_ptr(), rep, 0, n, ls.moves, ev.data_ptr(),
                        ls.base.handle if ls.base is not None else None, dedup, cutoff)
    e0.record()
    N.check(ls.lib.ps_search_round(ls.di.handle, C.byref(desc), C.c_void_p(ls.best_key.data_ptr()), None,
                                   C.c_void_p(stream.cuda_stream)))
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ts = sorted(ts[2:])
print(json.dumps({"lib": os.path.basename(os.environ.get("PS_LIBRARY", "default")),
                  "dynamic": os.environ.get("PS_DYNAMIC", "1"), "interval": os.environ.get("PS_CHECKPOINT_INTERVAL", "32"),
                  "config": cfg_id, "median_ms": round(ts[len(ts) // 2], 3), "min_ms": round(ts[0], 3),
                  "cand_per_s": round(n / ts[len(ts) // 2] * 1e3), "events_last": int(ev[0].item()), "events_full": int(ev[1].item()), "shift_permille": ls.moves.shift_permille, "cutoff": cutoff, "dedup": dedup}), flush=True)
