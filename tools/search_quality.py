"""Where the local search converges: seeds, move ranges and restarts (config 2 by default).

  python tools/search_quality.py [--config 2] [--seeds 16] [--neighbours 4096]

For each (max_shift, shift_permille) setting and seed: a fresh LocalSearch from the best_feasible
warm start until 16 rounds bring nothing; prints the converged makespans and wall times.
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--seeds", type=int, default=16)
    ap.add_argument("--neighbours", type=int, default=4096)
    args = ap.parse_args()
    import torch
    from paper_2510_05186_b200 import workloads
    from paper_2510_05186_b200.heuristics import best_feasible
    from paper_2510_05186_b200.listsched import stage_order_of
    from paper_2510_05186_b200.search import LocalSearch, SearchConfig
    inst = workloads.CONFIGS[args.config]()
    s0, _ = best_feasible(inst, device=0)
    orders = {i: stage_order_of(s0, i) for i in range(1, inst.num_stages + 1)}
    out = []
    for max_shift, permille in [(4, 700), (8, 700), (16, 700), (32, 700), (4, 900), (16, 500)]:
        spans, secs = [], []
        for seed in range(args.seeds):
            cfg = SearchConfig(seed=seed, neighbours=args.neighbours, shift_permille=permille, max_shift=max_shift)
            ls = LocalSearch(inst, orders, s0.offloaded, cfg, device=0)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            stale = 0
            while stale < 16 and ls.round < 4000:
                stale = 0 if ls.step() else stale + 1
            secs.append(time.perf_counter() - t0)
            spans.append(ls.makespan)
        row = {"max_shift": max_shift, "shift_permille": permille, "spans": spans, "best": min(spans),
               "seconds_mean": sum(secs) / len(secs)}
        out.append(row)
        print(json.dumps(row), flush=True)


def main_ils():
    from paper_2510_05186_b200 import workloads
    cfg = int(sys.argv[sys.argv.index("--config") + 1]) if "--config" in sys.argv else 2
    inst = workloads.CONFIGS[cfg]()
    for k in (2, 4, 8, 16):
        for seed in (0, 1):
            best, its, trace = ils(inst, seed, 4096 if cfg < 3 else 65536, k, 8.0)
            print(json.dumps({"kick_moves": k, "seed": seed, "best": best, "iterations": its,
                              "trace": [(round(t, 3), s) for t, s in trace]}), flush=True)




def ils(inst, seed, neighbours, kick_moves, budget_s, device=0):
    """Iterated local search prototype: converge, keep the best, kick the best with `kick_moves`
    random moves (a kick round's neighbours 0, 1, ... applied in turn, infeasible prefixes skipped)."""
    import ctypes as C
    import torch
    from paper_2510_05186_b200 import _native as N
    from paper_2510_05186_b200.heuristics import best_feasible
    from paper_2510_05186_b200.listsched import stage_order_of
    from paper_2510_05186_b200.search import LocalSearch, SearchConfig
    s0, _ = best_feasible(inst, device=device)
    orders = {i: stage_order_of(s0, i) for i in range(1, inst.num_stages + 1)}
    cfg = SearchConfig(seed=seed, neighbours=neighbours)
    ls = LocalSearch(inst, orders, s0.offloaded, cfg, device=device)
    t0 = time.perf_counter()
    best = ls.makespan
    best_o, best_m = ls.inc_orders.clone(), ls.inc_mask.clone()
    trace = [(0.0, best)]
    KICK = 1 << 40
    it = 0
    while time.perf_counter() - t0 < budget_s:
        stale = 0
        while stale < 16:
            stale = 0 if ls.step() else stale + 1
        if ls.makespan < best:
            best = ls.makespan
            best_o.copy_(ls.inc_orders)
            best_m.copy_(ls.inc_mask)
            trace.append((time.perf_counter() - t0, best))
        # kick from the best
        ls.inc_orders.copy_(best_o)
        ls.inc_mask.copy_(best_m)
        idx = 0
        applied = 0
        while applied < kick_moves and idx < 64 * kick_moves:
            o_save, m_save = ls.inc_orders.clone(), ls.inc_mask.clone()
            N.check(ls.lib.ps_apply_move(ls.di.handle, C.c_void_p(ls.inc_orders.data_ptr()),
                                         C.c_void_p(ls.inc_mask.data_ptr()), C.byref(ls.moves), KICK + it, idx,
                                         ls._stream()))
            res = ls.di.evaluate(ls.inc_orders.view(1, *ls.inc_orders.shape), ls.inc_mask.view(1, -1), peak=False)
            idx += 1
            if int(res.flags[0].item()) & N.FLAG_FEASIBLE:
                applied += 1
                span = int(res.makespan[0].item())
            else:
                ls.inc_orders.copy_(o_save)
                ls.inc_mask.copy_(m_save)
        ls.makespan = span if applied else best
        ls.base.record(ls.inc_orders, ls.inc_mask)
        it += 1
    return best, it, trace


def channel_polish(cfg=2, ils_seconds=5.0, neighbours=4096):
    """ILS for ils_seconds, then the channel-order search (reload/offload shifts)
    from its best schedule until 16 rounds bring nothing: does reordering transfers help?"""
    from paper_2510_05186_b200 import workloads
    from paper_2510_05186_b200.heuristics import best_feasible
    from paper_2510_05186_b200.listsched import stage_order_of
    from paper_2510_05186_b200.search import ChannelSearch, LocalSearch, SearchConfig
    inst = workloads.CONFIGS[cfg]()
    s0, _ = best_feasible(inst, device=0)
    orders = {i: stage_order_of(s0, i) for i in range(1, inst.num_stages + 1)}
    ls = LocalSearch(inst, orders, s0.offloaded, SearchConfig(seed=1, neighbours=neighbours, kick_moves=4), device=0)
    res = ls.run(time_budget=ils_seconds)
    out = {"config": cfg, "ils_best": res.makespan}
    for permille in (0, 300):
        cs = ChannelSearch.from_schedule(inst, res.schedule, SearchConfig(seed=2, neighbours=neighbours,
                                                                          shift_permille=permille), device=0)
        t0 = time.perf_counter()
        r2 = cs.run(patience=16)
        out[f"channel_{permille}"] = {"best": r2.makespan, "rounds": cs.round, "seconds": time.perf_counter() - t0,
                                      "improvements": len(r2.improvements)}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    if "--channel" in sys.argv:
        for c in (2, 3):
            channel_polish(c, 5.0, 4096 if c == 2 else 65536)
    else:
        main_ils() if "--ils" in sys.argv else main()