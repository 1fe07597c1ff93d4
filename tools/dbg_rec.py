import os, sys
import numpy as np
sys.path.insert(0, '/root/repo')
import torch
from paper_2510_05186_b200 import _native as N, workloads
from paper_2510_05186_b200.engine import Base
from paper_2510_05186_b200.heuristics import best_feasible
from paper_2510_05186_b200.listsched import stage_order_of
from paper_2510_05186_b200.search import LocalSearch, SearchConfig
for cfg in (2, 3, 4):
    inst = workloads.CONFIGS[cfg]()
    s0, _ = best_feasible(inst)
    orders = {i: stage_order_of(s0, i) for i in range(1, inst.num_stages + 1)}
    ls = LocalSearch(inst, orders, s0.offloaded, SearchConfig(seed=11, neighbours=64))
    r = ls.di.evaluate(ls.inc_orders.view(1, *ls.inc_orders.shape), ls.inc_mask.view(1, -1), peak=True, trace=True)
    torch.cuda.synchronize()
    info = np.frombuffer(ls.base.read(N.BASE_INFO), np.int32)
    res = np.frombuffer(ls.base.read(N.BASE_RESULT), np.int64)
    P = inst.num_stages
    print("cfg", cfg, "plain flags", int(r.flags[0]), "span", int(r.makespan[0]), "peak", r.peak[0].tolist()[:4])
    print("   base info", info.tolist(), "span", res[0], "peaks", res[2:2+4].tolist(), "sfree", res[2+P:2+P+4].tolist())
    ev = int((r.trace_code[0] != 0).sum())
    print("   plain events ~", ev)
