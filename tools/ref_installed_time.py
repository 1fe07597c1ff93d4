"""The reference's own best_feasible under integrate.install: run_order rebound only, vs the
batched generators (one launch for the AdaOffload back-off sequence).  Needs baseline/_ref."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
import pipesched  # noqa: E402

from paper_2510_05186_b200 import integrate, workloads  # noqa: E402
from paper_2510_05186_b200.instance import instance_to_dict  # noqa: E402

for cfg in [int(x) for x in (sys.argv[1:] or ["3", "4", "5"])]:
    inst = pipesched.instance_from_dict(instance_to_dict(workloads.CONFIGS[cfg]()))
    row = {"config": cfg}
    for gens in (False, True):
        integrate.install(pipesched, generators=gens)
        try:
            pipesched.best_feasible(inst)
            t = time.perf_counter()
            s, name = pipesched.best_feasible(inst)
            row["batched" if gens else "run_order_only"] = round(time.perf_counter() - t, 3)
            row["name"] = name
        finally:
            integrate.uninstall(pipesched)
    print(json.dumps(row), flush=True)
