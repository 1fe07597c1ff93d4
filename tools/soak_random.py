"""Exactness soak over many random instances (tests/test_gpu_soak_random.py's cases):
  python tools/soak_random.py <first seed> <count> [small|wide|big] [search|channel|batch|ils]
(one JSON line per instance, then a total)"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from test_gpu_soak_random import soak_batch_case, soak_case, soak_channel_case, soak_ils_case  # noqa: E402

first, count = int(sys.argv[1]), int(sys.argv[2])
kind = sys.argv[3] if len(sys.argv) > 3 else "small"
path = sys.argv[4] if len(sys.argv) > 4 else "search"
kw = {"small": {}, "wide": dict(stages=(12, 32), microbatches=(16, 96), n=1024),
      "big": dict(stages=(2, 16), microbatches=(4, 64), n=1024, big=True)}[kind]
if path == "ils":
    kw = {"small": {}, "wide": dict(stages=(10, 20), microbatches=(16, 48), n=256),
          "big": dict(stages=(2, 10), microbatches=(4, 24), big=True)}[kind]
elif path != "batch" and kind != "small":
    kw["rounds"] = 12 if kind == "wide" else 16
case = {"search": soak_case, "channel": soak_channel_case, "batch": soak_batch_case, "ils": soak_ils_case}[path]
total = 0
for seed in range(first, first + count):
    t0 = time.time()
    r = case(seed, **kw)
    if r is not None:
        total += r[2]
    print(json.dumps({"seed": seed, "kind": kind, "path": path, "P": r and r[0], "m": r and r[1], "checked": r and r[2],
                      "seconds": round(time.time() - t0, 2)}), flush=True)
print(json.dumps({"kind": kind, "path": path, "seeds": count, "checked": total, "mismatches": 0}), flush=True)
