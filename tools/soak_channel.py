"""Soak test of explicit-channel prefix/suffix sharing: a channel-order search with the incumbent
recorded in explicit mode, every `every`-th round compared neighbour by neighbour with the same
round evaluated without a base.   python tools/soak_channel.py [config] [neighbours] [rounds] [every]"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2510_05186_b200 import _native as N, workloads  # noqa: E402
from paper_2510_05186_b200.heuristics import best_feasible  # noqa: E402
from paper_2510_05186_b200.search import ChannelSearch, SearchConfig  # noqa: E402

cfg, n, rounds, every = (int(x) for x in (sys.argv[1:] + ["3", "8192", "120", "5"][len(sys.argv) - 1:])[:4])
inst = workloads.CONFIGS[cfg]()
s0, _ = best_feasible(inst)
cs = ChannelSearch.from_schedule(inst, s0, SearchConfig(seed=9, neighbours=n, shift_permille=400, max_shift=4))
stream = C.c_void_p(torch.cuda.current_stream().cuda_stream)
checked = mism = 0
for r in range(rounds):
    if r % every == 0:
        got = []
        for base in (cs.base, None):
            out = torch.empty(n, dtype=torch.int64, device="cuda")
            k = torch.full((1,), N.BEST_NONE, dtype=torch.int64, device="cuda")
            desc = N.SearchDesc(cs.inc_orders.data_ptr(), cs.inc_mask.data_ptr(), cs.round, 0, n, cs.moves, None,
                                base.handle if base is not None else None, 0)
            N.check(cs.lib.ps_search_round_explicit(cs.di.handle, C.byref(desc), C.c_void_p(cs.inc_chan.data_ptr()),
                                                    cs.chan_stride, C.c_void_p(k.data_ptr()),
                                                    C.c_void_p(out.data_ptr()), stream))
            torch.cuda.synchronize()
            got.append((out.cpu().numpy(), int(k.item())))
        bad = int((got[0][0] != got[1][0]).sum()) + int(got[0][1] != got[1][1])
        checked += n
        mism += bad
    cs.step()
print(json.dumps({"config": cfg, "rounds": rounds, "checked": checked, "mismatches": mism,
                  "improvements": len(cs.improvements), "final": cs.makespan}), flush=True)
