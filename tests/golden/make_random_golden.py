"""Reference answers on random non-uniform mid-size instances (the soak's instance family).

    python tests/golden/make_random_golden.py        (here: imports the unmodified reference)

The soaks in tests/test_gpu_soak_random.py check the GPU against the C restatement on instances
drawn by `random_tables` (independent per-(stage, microbatch) times and bytes, shared transfer
channels, post-validation, zero comm/offload times, 64-bit byte counts).  This script pins that
family to the reference itself: for instances drawn the same way, it records with
`pipesched.run_order` (make_golden.record) the generator structures, their explicit-channel
replays and perturbed structures, into random.json.gz, a corpus the oracle and GPU parity tests
read like the others (tests/_golden.py CORPORA).
"""

from __future__ import annotations

import random
import sys
import time
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))
sys.path.insert(0, str(HERE.parent))

import make_golden as mg  # noqa: E402  (imports the reference as `ps`)
from test_gpu_soak_random import random_tables  # noqa: E402


def main():
    rng = random.Random(20251018)
    t0 = time.time()
    insts = []
    shapes = [((2, 8), (4, 16), False)] * 28 + [((6, 12), (12, 24), False)] * 16 + \
             [((2, 8), (4, 16), True)] * 10 + [((10, 20), (16, 48), False)] * 6
    for stages, microbatches, big in shapes:
        P, m = rng.randint(*stages), rng.randint(*microbatches)
        insts.append(mg.ps.instance_from_dict(random_tables(rng, P, m, big)))
    out = mg.corpus_cases("random", insts, rng, 12)
    n = sum(len(e["cases"]) for e in out["instances"])
    mg.dump(out, "random.json.gz")
    print(f"{len(insts)} instances, {n} cases in {time.time() - t0:.1f} s")


if __name__ == "__main__":
    main()
