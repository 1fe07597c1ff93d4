"""Time base recordings: a fresh recording of the warm start, then the re-recordings of a search's
first rounds (each resumes from its predecessor's checkpoints and converges onto it).

  python tools/rec_time.py [config] [neighbours] [rounds]      (one JSON line)
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2510_05186_b200 import workloads  # noqa: E402
from paper_2510_05186_b200.engine import Base  # noqa: E402
from paper_2510_05186_b200.heuristics import best_feasible  # noqa: E402
from paper_2510_05186_b200.listsched import stage_order_of  # noqa: E402
from paper_2510_05186_b200.search import LocalSearch, SearchConfig  # noqa: E402

cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 5
n = int(sys.argv[2]) if len(sys.argv) > 2 else 131072
rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 12
inst = workloads.CONFIGS[cfg_id]()
s0, _ = best_feasible(inst)
orders = {i: stage_order_of(s0, i) for i in range(1, inst.num_stages + 1)}
ls = LocalSearch(inst, orders, s0.offloaded, SearchConfig(seed=20251005, neighbours=n, shift_permille=700, max_shift=4))


def timed(fn):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


fresh = [timed(lambda: Base(ls.di).record(ls.inc_orders, ls.inc_mask)) for _ in range(3)]
rec_ms = []
orig = ls.base.record
ls.base.record = lambda o, m, stream=None: rec_ms.append(timed(lambda: orig(o, m, stream)))
for _ in range(rounds):
    ls.launch_round()
    ls.finish_round()
print(json.dumps({"config": cfg_id, "fresh_ms": [round(x, 2) for x in fresh],
                  "rerecord_ms": [round(x, 3) for x in rec_ms],
                  "rerecord_mean_ms": round(sum(rec_ms) / max(1, len(rec_ms)), 3)}), flush=True)
