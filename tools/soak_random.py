"""Exactness soak of the search over many random instances (tests/test_gpu_soak_random.py's case):
  python tools/soak_random.py <first seed> <count> [small|wide|big]   (one JSON line per instance)"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from test_gpu_soak_random import soak_case  # noqa: E402

first, count = int(sys.argv[1]), int(sys.argv[2])
kind = sys.argv[3] if len(sys.argv) > 3 else "small"
kw = {"small": {}, "wide": dict(stages=(12, 32), microbatches=(16, 96), n=1024, rounds=12),
      "big": dict(stages=(2, 16), microbatches=(4, 64), n=1024, rounds=16, big=True)}[kind]
total = 0
for seed in range(first, first + count):
    t0 = time.time()
    r = soak_case(seed, **kw)
    if r is not None:
        total += r[2]
    print(json.dumps({"seed": seed, "kind": kind, "P": r and r[0], "m": r and r[1], "checked": r and r[2],
                      "seconds": round(time.time() - t0, 2)}), flush=True)
print(json.dumps({"kind": kind, "seeds": count, "checked": total, "mismatches": 0}), flush=True)
