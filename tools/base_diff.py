"""Diagnostic: a base recorded afresh vs the same base re-recorded over its predecessor."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_05186_b200 import _native as N, workloads  # noqa: E402
from paper_2510_05186_b200.engine import Base  # noqa: E402
from paper_2510_05186_b200.heuristics import best_feasible  # noqa: E402
from paper_2510_05186_b200.listsched import stage_order_of  # noqa: E402
from paper_2510_05186_b200.search import LocalSearch, SearchConfig  # noqa: E402

inst = workloads.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 3]()
s0, _ = best_feasible(inst)
orders = {i: stage_order_of(s0, i) for i in range(1, inst.num_stages + 1)}
ls = LocalSearch(inst, orders, s0.offloaded, SearchConfig(seed=20251005, neighbours=4096))
o, mk = ls.materialize(0, 4096, 0)
flags = ls.di.evaluate(o, mk, peak=False).flags.cpu().numpy()
idx = int(np.nonzero(flags & 1)[0][5])
fresh, resumed = Base(ls.di), Base(ls.di)
fresh.record(o[idx], mk[idx])
resumed.record(ls.inc_orders, ls.inc_mask)
resumed.record(o[idx], mk[idx])
for what, name in enumerate(["ck", "cstep", "fstep", "info", "res"]):
    a, b = fresh.read(what), resumed.read(what)
    dt = np.int64 if name == "res" else np.uint32
    a, b = np.frombuffer(a, dt), np.frombuffer(b, dt)
    if name == "info":
        print("info fresh", a, "resumed", b)
    d = np.nonzero(a != b)[0]
    print(name, len(a), "differ", len(d), d[:20])
    if name == "ck" and len(d):
        info = np.frombuffer(fresh.read(N.BASE_INFO), np.int32)
        nck = info[0]
        ckw = len(a) // (5 * inst.num_stages * inst.num_microbatches // 32 + 2)
        print("ck_words", ckw, "n_ck", nck, "differing checkpoints", sorted(set((d // ckw).tolist()))[:40])
        print("offsets within checkpoint", sorted(set((d % ckw).tolist()))[:60])
a = np.frombuffer(fresh.read(0), np.uint32).reshape(82, -1) if inst.num_microbatches == 64 else None
b = np.frombuffer(resumed.read(0), np.uint32).reshape(82, -1) if a is not None else None
if a is not None:
    for c in (41, 42, 43, 60):
        dd = np.nonzero(a[c] != b[c])[0]
        print("ck", c, "ndiff", len(dd), "first", [(int(x), int(a[c][x]), int(b[c][x])) for x in dd[:8]])
