"""A/B of bound pruning on whole descents: same seed, prune on vs off, trail
must be identical; prints wall time to convergence per config (two passes each, alternating).

  python tools/prune_ab.py [configs...]        (default: 1 2 3 4)
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2510_05186_b200 import workloads
    from paper_2510_05186_b200.heuristics import best_feasible
    from paper_2510_05186_b200.listsched import stage_order_of
    from paper_2510_05186_b200.search import LocalSearch, SearchConfig
    cfgs = [int(a) for a in sys.argv[1:]] or [1, 2, 3, 4]
    for c in cfgs:
        inst = workloads.CONFIGS[c]()
        s0, _ = best_feasible(inst, device=0)
        orders = {i: stage_order_of(s0, i) for i in range(1, inst.num_stages + 1)}
        res = {}
        for rep in range(2):
            for prune in (False, True):
                ls = LocalSearch(inst, orders, s0.offloaded,
                                 SearchConfig(seed=20251005, neighbours=65536, prune=prune), device=0)
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                while ls.stale < 16 and ls.round < 3000:
                    ls.step(t0)
                torch.cuda.synchronize()
                dt = time.perf_counter() - t0
                trail = [(i.round, i.makespan) for i in ls.improvements]
                key = "prune" if prune else "full"
                res.setdefault(key, []).append(round(dt, 3))
                res.setdefault(key + "_trail", trail)
                assert res[key + "_trail"] == trail
        assert res["prune_trail"] == res["full_trail"], "pruning changed the trajectory"
        print(json.dumps({"config": c, "rounds": ls.round, "best": ls.best_makespan,
                          "seconds_full": res["full"], "seconds_prune": res["prune"]}), flush=True)


if __name__ == "__main__":
    main()
