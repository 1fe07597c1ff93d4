"""Time materialised batches on the device (one round's neighbours as uint8/uint16 rows): with the
incumbent as recorded base and without a base, no blocked-stage output (the e2e configuration).
  PS_LIBRARY=<variant> python tools/mat_time.py [config] [n]      (one JSON line)"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2510_05186_b200 import workloads  # noqa: E402
from paper_2510_05186_b200.heuristics import best_feasible  # noqa: E402
from paper_2510_05186_b200.listsched import stage_order_of  # noqa: E402
from paper_2510_05186_b200.search import LocalSearch, SearchConfig  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
n = int(sys.argv[2]) if len(sys.argv) > 2 else 65536
inst = workloads.CONFIGS[cfg]()
s0, _ = best_feasible(inst)
ls = LocalSearch(inst, {i: stage_order_of(s0, i) for i in range(1, inst.num_stages + 1)}, s0.offloaded,
                 SearchConfig(seed=20251005, neighbours=n, shift_permille=700, max_shift=4))
o, mk = ls.materialize(0, n, 5)
if 4 * inst.num_microbatches <= 256:
    o = o.to(torch.uint8)
out = ls.di.alloc_results(n, peak=True, blocked=False)


def t(base, reps=5):
    ts = []
    for _ in range(reps + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ls.di.evaluate(o, mk, base=base, out=out)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return round(sorted(ts[1:])[reps // 2], 3)


print(json.dumps({"lib": os.path.basename(os.environ.get("PS_LIBRARY", "default")), "config": cfg,
                  "with_base_ms": t(ls.base), "no_base_ms": t(None, 3)}), flush=True)
