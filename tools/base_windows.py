"""Diagnostic: per-checkpoint live window sizes of a recorded base (max over stages)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2510_05186_b200 import _native as N, workloads  # noqa: E402
from paper_2510_05186_b200.heuristics import best_feasible  # noqa: E402
from paper_2510_05186_b200.listsched import stage_order_of  # noqa: E402
from paper_2510_05186_b200.search import LocalSearch, SearchConfig  # noqa: E402

inst = workloads.CONFIGS[3]()
s0, _ = best_feasible(inst)
orders = {i: stage_order_of(s0, i) for i in range(1, inst.num_stages + 1)}
ls = LocalSearch(inst, orders, s0.offloaded, SearchConfig(seed=20251005, neighbours=1024))
for name in ("warm", "late"):
    if name == "late":
        z = np.load("tests/golden/inc320_config3.npz")
        ls.inc_orders.copy_(torch.from_numpy(z["orders"].view(np.int16)))
        ls.inc_mask.copy_(torch.from_numpy(z["mask"].view(np.int32)))
        ls.base.record(ls.inc_orders, ls.inc_mask)
    info = np.frombuffer(ls.base.read(N.BASE_INFO), np.int32)
    lay = np.frombuffer(ls.base.read(N.BASE_LAYOUT), np.int32)
    ckw, ckmax, iv, kc, ck_t, ck_u, ck_r, regw = lay.tolist()
    raw = np.frombuffer(ls.base.read(N.BASE_CHECKPOINTS), np.uint32)
    P = inst.num_stages
    counts = [int(raw[c * ckw + ck_r: c * ckw + ck_r + regw * P].reshape(P, regw)[:, 4].max()) for c in range(info[0])]
    print(name, "n_ck", info[0], "max_window", info[4], "counts by checkpoint (every 8th):", counts[::8])
