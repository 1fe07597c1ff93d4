"""Time channel-order search rounds (explicit channel mode) on a config."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2510_05186_b200 import workloads  # noqa: E402
from paper_2510_05186_b200.heuristics import best_feasible  # noqa: E402
from paper_2510_05186_b200.search import ChannelSearch, SearchConfig  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
n = int(sys.argv[2]) if len(sys.argv) > 2 else 65536
inst = workloads.CONFIGS[cfg]()
s0, _ = best_feasible(inst)
share = os.environ.get("CHAN_SHARE", "1") != "0"
cs = ChannelSearch.from_schedule(inst, s0, SearchConfig(seed=7, neighbours=n, shift_permille=500, max_shift=4,
                                                        share_prefix=share))
cs.run(rounds=1)
torch.cuda.synchronize()
t = time.perf_counter()
res = cs.run(rounds=5)
torch.cuda.synchronize()
dt = (time.perf_counter() - t) / 5
print(json.dumps({"lib": os.path.basename(os.environ.get("PS_LIBRARY", "default")), "share_prefix": share, "config": cfg,
                  "ms_per_round": round(1000 * dt, 2), "cand_per_s": round(n / dt), "makespan": res.makespan}))
