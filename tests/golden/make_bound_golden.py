"""Golden fixtures for the B&B node lower bound, by running the REFERENCE solver.

Run here (the reference is importable only in the build container):

    python tests/golden/make_bound_golden.py

It runs the unmodified reference branch-and-bound (`solver._Search`, solver.py:164-520) on a
corpus of small instances with a node budget and records, at every call of `_Search._bound`
(solver.py:352-383, which uses `_chain_ends`, solver.py:321-350), the node state the bound
reads — clock, stage free times, committed compute starts, post-validation flag — and the value
the reference returns.  Output: tests/golden/bounds.json.gz.
"""

from __future__ import annotations

import gzip
import json
import sys
from pathlib import Path

REF = "/root/reference/pkg/src"
HERE = Path(__file__).resolve().parent
sys.path.insert(0, REF)
sys.path.insert(0, str(HERE.parents[1]))

import pipesched as ps  # noqa: E402  (the reference)
from pipesched import solver as rs  # noqa: E402

from paper_2510_05186_b200.instance import instance_to_dict as our_to_dict  # noqa: E402
from paper_2510_05186_b200.instance import instance_from_dict as our_from_dict  # noqa: E402

sys.setrecursionlimit(50000)


def corpus():
    out = []
    for P, m in ((2, 2), (3, 3), (4, 4), (4, 8)):
        for post in (False, True):
            out.append(ps.make_uniform_instance(P, m, 2, 2, 1, 1, 1, 2, 4, post_validation=post))
    for seed in range(12):
        P, m = 2 + seed % 3, 2 + (seed // 3) % 3
        out.append(ps.random_instance(seed, P, m, mem_profile=("ample", "tight")[seed % 2],
                                      post_validation=bool(seed % 4 == 3)))
    out.append(ps.make_uniform_instance(8, 16, 3, 4, 2, 1, 2, 2, 5))
    return out


def main():
    rows = []
    for inst in corpus():
        # the reference instance, rebuilt from our JSON codec so both sides read the same tables
        ref = ps.instance_from_dict(our_to_dict(our_from_dict(json.loads(json.dumps(ps.instance_to_dict(inst))))))
        for symmetry in (True, False):
            nodes = []
            orig = rs._Search._bound

            def hooked(self, _orig=orig, _nodes=nodes):
                lb = _orig(self)
                if len(_nodes) < 160:
                    _nodes.append({"t": self.clock,
                                   "sfree": [self.stage_free[i] for i in self.stages],
                                   "comp": sorted([op.stage, op.microbatch, int(op.kind), s]
                                                  for op, s in self.comp_start.items()),
                                   "lb": lb})
                return lb

            rs._Search._bound = hooked
            try:
                rs.start_session(ref, rs.SolveBudget(wall_time_limit=10.0, node_limit=300), symmetry=symmetry)
            finally:
                rs._Search._bound = orig
            rows.append({"instance": our_to_dict(our_from_dict(json.loads(json.dumps(ps.instance_to_dict(inst))))),
                         "post": bool(ref.post_validation), "symmetry": symmetry, "nodes": nodes})
    path = HERE / "bounds.json.gz"
    with gzip.open(path, "wt") as f:
        json.dump({"generator": "tests/golden/make_bound_golden.py", "rows": rows}, f)
    print(path, sum(len(r["nodes"]) for r in rows), "nodes")


if __name__ == "__main__":
    main()
