"""Time the drop-in generators per call (heuristics.best_feasible / ada_offload) per config."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_05186_b200 import workloads  # noqa: E402
from paper_2510_05186_b200.heuristics import best_feasible  # noqa: E402

for c in [int(x) for x in (sys.argv[1:] or ["3", "4", "5"])]:
    inst = workloads.CONFIGS[c]()
    best_feasible(inst)
    t = time.perf_counter()
    s, name = best_feasible(inst)
    print(json.dumps({"config": c, "best_feasible_ms": round(1000 * (time.perf_counter() - t), 1), "name": name}), flush=True)
