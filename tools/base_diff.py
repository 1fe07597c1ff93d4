"""Diagnostic: a base recorded afresh vs the same base re-recorded over its predecessor."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402
from paper_2510_05186_b200 import _native as N, workloads  # noqa: E402
from paper_2510_05186_b200.engine import Base  # noqa: E402
from paper_2510_05186_b200.heuristics import best_feasible  # noqa: E402
from paper_2510_05186_b200.listsched import stage_order_of  # noqa: E402
from paper_2510_05186_b200.search import LocalSearch, SearchConfig  # noqa: E402
from test_gpu_search import _base_tables  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
inst = workloads.CONFIGS[cfg]()
s0, _ = best_feasible(inst)
orders = {i: stage_order_of(s0, i) for i in range(1, inst.num_stages + 1)}
ls = LocalSearch(inst, orders, s0.offloaded, SearchConfig(seed=11, neighbours=512, shift_permille=700, max_shift=4))
pk = ls.di.packed
P, m = pk.num_stages, pk.num_microbatches
MW = (m + 31) // 32
o, mk = ls.materialize(0, 512, 2)
r = ls.di.evaluate(o, mk, peak=False)
torch.cuda.synchronize()
flags, spans = r.flags.cpu().numpy(), r.makespan.cpu().numpy()
feas = np.nonzero(flags & 1)[0]
order = feas[np.argsort(spans[feas], kind="stable")]
for idx in [int(x) for x in order[:6]]:
    fresh, again = Base(ls.di), Base(ls.di)
    fresh.record(o[idx], mk[idx])
    again.record(ls.inc_orders, ls.inc_mask)
    again.record(o[idx], mk[idx])
    info_again = np.frombuffer(again.read(N.BASE_INFO), np.int32)
    a, b = _base_tables(fresh, P, m, MW), _base_tables(again, P, m, MW)
    names = ["info", "res", "cstep", "fstep"]
    bad = [names[k] for k in range(4) if a[k] != b[k]]
    print("idx", idx, "span", spans[idx], "dbg", info_again[7], "conv_c/delta", info_again[5], info_again[6], "n_ck", info_again[0], "diff tables", bad)
    for k in range(4):
        if a[k] != b[k]:
            x, y = np.array(a[k]), np.array(b[k])
            d = np.nonzero(x != y)[0]
            print("  ", names[k], "at", d[:10], x[d[:10]], y[d[:10]])
    for c, (ca, cb) in enumerate(zip(a[4], b[4])):
        if ca != cb:
            sw = np.nonzero(np.array(ca[0]) != np.array(cb[0]))[0]
            rg = np.nonzero(np.array(ca[1]) != np.array(cb[1]))
            wn = [s for s in range(P) if ca[2][s] != cb[2][s]]
            print("   ck", c, "state words", sw[:8], np.array(ca[0])[sw[:8]], np.array(cb[0])[sw[:8]],
                  "regs (lane,word)", list(zip(*rg))[:6], "windows", wn[:4])
            if len(rg[0]):
                l, w = rg[0][0], rg[1][0]
                print("      fresh", ca[1][l], "\n      again", cb[1][l])
