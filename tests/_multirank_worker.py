"""Worker for tests/test_gpu_multirank.py: one rank of a sharded LocalSearch (torchrun).

Ranks share cuda:0 over gloo (PS_SHARE_GPU=1) on a one-GPU test box; each writes its improvement
trail and final best structure to <out>.rank<r>.json.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2510_05186_b200 import workloads
    from paper_2510_05186_b200.heuristics import best_feasible
    from paper_2510_05186_b200.listsched import stage_order_of
    from paper_2510_05186_b200.search import LocalSearch, SearchConfig
    cfg, n, rounds, kick_moves, kicks, out = (int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]),
                                              int(sys.argv[4]), int(sys.argv[5]), sys.argv[6])
    torch.cuda.set_device(0)
    dist.init_process_group("gloo")
    inst = workloads.CONFIGS[cfg]()
    s0, _ = best_feasible(inst, device=0)
    orders = {i: stage_order_of(s0, i) for i in range(1, inst.num_stages + 1)}
    ls = LocalSearch(inst, orders, s0.offloaded, SearchConfig(seed=5, neighbours=n, kick_moves=kick_moves), device=0)
    res = ls.run(rounds=rounds) if kick_moves == 0 else ls.run(kicks=kicks)
    doc = {"rank": dist.get_rank(), "world": dist.get_world_size(), "first": ls.first, "count": ls.count,
           "trail": [[i.round, i.makespan, i.index] for i in res.improvements], "best": res.makespan,
           "rounds": ls.round, "kicks": ls.kicks,
           "orders": ls.best_orders.cpu().numpy().view(np.uint16).tolist(),
           "mask": ls.best_mask.cpu().numpy().view(np.uint32).tolist()}
    with open(f"{out}.rank{dist.get_rank()}.json", "w") as fh:
        json.dump(doc, fh)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
