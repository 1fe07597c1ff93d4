"""Soak test of exactness along whole searches: every `every`-th round of a search, every
neighbour's makespan with prefix/suffix sharing (recorded incumbent) against its full simulation
(no base).   python tools/soak_exact.py [config] [neighbours] [rounds] [every] [seed]"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2510_05186_b200 import _native as N, workloads  # noqa: E402
from paper_2510_05186_b200.heuristics import best_feasible  # noqa: E402
from paper_2510_05186_b200.listsched import stage_order_of  # noqa: E402
from paper_2510_05186_b200.search import LocalSearch, SearchConfig  # noqa: E402

cfg, n, rounds, every, seed = (int(x) for x in (sys.argv[1:] + ["3", "16384", "200", "10", "1"][len(sys.argv) - 1:])[:5])
inst = workloads.CONFIGS[cfg]()
s0, _ = best_feasible(inst)
ls = LocalSearch(inst, {i: stage_order_of(s0, i) for i in range(1, inst.num_stages + 1)}, s0.offloaded,
                 SearchConfig(seed=seed, neighbours=n, shift_permille=700, max_shift=4, kick_moves=4))
stream = C.c_void_p(torch.cuda.current_stream().cuda_stream)
checked = mism = 0
for r in range(rounds):
    if r % every == 0:
        got = []
        for base in (ls.base, None):
            out = torch.empty(n, dtype=torch.int64, device="cuda")
            k = torch.full((1,), N.BEST_NONE, dtype=torch.int64, device="cuda")
            desc = N.SearchDesc(ls.inc_orders.data_ptr(), ls.inc_mask.data_ptr(), ls.round, 0, n, ls.moves, None,
                                base.handle if base is not None else None)
            N.check(ls.lib.ps_search_round(ls.di.handle, C.byref(desc), C.c_void_p(k.data_ptr()),
                                           C.c_void_p(out.data_ptr()), stream))
            torch.cuda.synchronize()
            got.append((out.cpu().numpy(), int(k.item())))
        bad = int((got[0][0] != got[1][0]).sum()) + int(got[0][1] != got[1][1])
        checked += n
        mism += bad
        if bad:
            print(json.dumps({"round": r, "mismatches": bad}), flush=True)
    if not ls.step():
        ls.stale = getattr(ls, "stale", 0)
        if ls.cfg.kick_moves:
            ls.kick()
print(json.dumps({"config": cfg, "rounds": rounds, "checked": checked, "mismatches": mism,
                  "final": ls.best_makespan}), flush=True)
