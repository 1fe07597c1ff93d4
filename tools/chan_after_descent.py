"""Does a channel-order descent improve on the derived-mode descent's local optimum?"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_05186_b200 import workloads  # noqa: E402
from paper_2510_05186_b200.heuristics import best_feasible  # noqa: E402
from paper_2510_05186_b200.listsched import stage_order_of  # noqa: E402
from paper_2510_05186_b200.search import ChannelSearch, LocalSearch, SearchConfig  # noqa: E402

for cfg in [int(x) for x in (sys.argv[1:] or ["2", "3"])]:
    inst = workloads.CONFIGS[cfg]()
    s0, _ = best_feasible(inst)
    n = 4096 if cfg == 2 else 65536
    t0 = time.perf_counter()
    ls = LocalSearch(inst, {i: stage_order_of(s0, i) for i in range(1, inst.num_stages + 1)}, s0.offloaded,
                     SearchConfig(seed=1, neighbours=n, shift_permille=700, max_shift=4))
    res = ls.run(patience=16)
    t1 = time.perf_counter()
    out = {"config": cfg, "descent": res.makespan, "descent_s": round(t1 - t0, 2)}
    for permille in (0, 300):
        cs = ChannelSearch.from_schedule(inst, res.schedule, SearchConfig(seed=2, neighbours=n, shift_permille=permille,
                                                                          max_shift=4))
        r2 = cs.run(patience=16)
        out[f"channel_{permille}"] = r2.makespan
        out[f"channel_{permille}_s"] = round(time.perf_counter() - t1, 2)
        out[f"channel_{permille}_rounds"] = cs.round
    print(json.dumps(out), flush=True)
