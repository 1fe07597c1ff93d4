"""Time to best: the GPU local search vs the CPU, measured (not extrapolated).

  python tools/ttb_compare.py [--configs 1 2 3] [--out gpurun_out/r02_ttb.json]

Per config:
* gpu        LocalSearch from the best_feasible warm start (BASELINE's neighbours per round),
             until 16 rounds bring nothing: every strict improvement with its wall-clock time.
* gpu_ils    the iterated local search (kicks from the best) for the same
             wall-clock budget as the reference solver.
* cpu_port   the IDENTICAL search on the host cores: the C restatement of run_order evaluates
             every neighbour of every round (oracle/ps_oracle.c or_search_round, all threads),
             the same (makespan, index) selection, the same move applied — its improvement trail
             must equal the GPU's round for round.  Config 3's 65,536-neighbour rounds take ~15 s
             each on 16 threads, so there only the first `--cpu-rounds` rounds are run (measured),
             and the trail is compared over them.
* reference  the reference's own anytime solver (pipesched.start_session, branch and bound,
             solver.py:543-565) from the same warm start, wall-clock limited (30 s config 1,
             60 s config 2 with the recursion limit raised, solver.py:451-478), its incumbent stream.
The JSON holds each stream and the best makespan each arm has at fixed wall-clock times.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SEED = 20251005
MOVES = dict(shift_permille=700, max_shift=4)
NEIGHBOURS = {1: 4096, 2: 4096, 3: 65536}
REF_BUDGET = {1: 30.0, 2: 60.0, 3: 60.0}
MARKS = (0.01, 0.1, 1.0, 6.0, 30.0, 60.0)


def best_at(stream, t):
    best = None
    for at, span in stream:
        if at <= t:
            best = span if best is None else min(best, span)
    return best


def gpu_arm(inst, cfg):
    import torch
    from paper_2510_05186_b200.heuristics import best_feasible
    from paper_2510_05186_b200.listsched import stage_order_of
    from paper_2510_05186_b200.search import LocalSearch, SearchConfig
    t0 = time.perf_counter()
    s0, name = best_feasible(inst, device=0)
    t_warm = time.perf_counter() - t0
    orders = {i: stage_order_of(s0, i) for i in range(1, inst.num_stages + 1)}
    sc = SearchConfig(seed=SEED, neighbours=NEIGHBOURS[cfg], **MOVES)
    ls = LocalSearch(inst, orders, s0.offloaded, sc, device=0)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    stale = 0
    while stale < 16 and ls.round < 5000:
        ls.launch_round()
        stale = 0 if ls.finish_round(t1) else stale + 1
    elapsed = time.perf_counter() - t1
    stream = [(t_warm, ls.initial_makespan)] + [(t_warm + imp.timestamp, imp.makespan) for imp in ls.improvements]
    return {"warm_start": name, "warm_seconds": t_warm, "search_seconds": elapsed, "rounds": ls.round,
            "neighbours_per_round": sc.neighbours, "stream": stream,
            "trail": [[imp.round, imp.makespan, imp.index] for imp in ls.improvements]}, ls, s0


def gpu_ils_arm(inst, cfg, budget, kick_moves=4):
    """Iterated local search for `budget` seconds from the same warm start."""
    import torch
    from paper_2510_05186_b200.heuristics import best_feasible
    from paper_2510_05186_b200.listsched import stage_order_of
    from paper_2510_05186_b200.search import LocalSearch, SearchConfig
    t0 = time.perf_counter()
    s0, name = best_feasible(inst, device=0)
    t_warm = time.perf_counter() - t0
    orders = {i: stage_order_of(s0, i) for i in range(1, inst.num_stages + 1)}
    sc = SearchConfig(seed=SEED, neighbours=NEIGHBOURS[cfg], kick_moves=kick_moves, **MOVES)
    ls = LocalSearch(inst, orders, s0.offloaded, sc, device=0)
    res = ls.run(time_budget=budget - t_warm)
    stream = [(t_warm, ls.initial_makespan)] + [(t_warm + imp.timestamp, imp.makespan) for imp in res.improvements]
    return {"warm_start": name, "warm_seconds": t_warm, "budget_seconds": budget, "rounds": ls.round,
            "kicks": ls.kicks, "kick_moves": kick_moves, "neighbours_per_round": sc.neighbours,
            "stream": stream}, res.schedule


def cpu_port_arm(inst, cfg, s0, max_rounds, max_seconds):
    import numpy as np
    from oracle.oracle import Oracle
    from paper_2510_05186_b200.listsched import stage_order_of
    from paper_2510_05186_b200.packing import encode_candidate, pack_instance
    pk = pack_instance(inst)
    orc = Oracle(pk)
    threads = len(os.sched_getaffinity(0))
    o, mk, _ = encode_candidate(pk, {i: stage_order_of(s0, i) for i in range(1, pk.num_stages + 1)}, s0.offloaded)
    span = int(orc.run(o, mk)["makespan"])
    n = NEIGHBOURS[cfg]
    t0 = time.perf_counter()
    stream, trail, rnd, stale, round_s = [(0.0, span)], [], 0, 0, []
    while stale < 16 and rnd < max_rounds and time.perf_counter() - t0 < max_seconds:
        tr = time.perf_counter()
        key, _ = orc.search_round(o, mk, SEED, MOVES["shift_permille"], MOVES["max_shift"], rnd, 0, n, threads)
        round_s.append(time.perf_counter() - tr)
        if key != np.iinfo(np.int64).max and (key >> 32) < span:
            idx = key & 0xFFFFFFFF
            _, o, mk = orc.neighbour(o, mk, SEED, MOVES["shift_permille"], MOVES["max_shift"], rnd, idx)
            span = int(key >> 32)
            trail.append([rnd, span, idx])
            stream.append((time.perf_counter() - t0, span))
            stale = 0
        else:
            stale += 1
        rnd += 1
    return {"threads": threads, "rounds": rnd, "seconds": time.perf_counter() - t0, "stream": stream,
            "trail": trail, "seconds_per_round_mean": sum(round_s) / max(1, len(round_s)),
            "complete": stale >= 16}


def ref_arm(inst_ours, cfg):
    ref_root = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref_root, "pipesched")):
        return {"unavailable": "baseline/_ref not installed"}
    sys.path.insert(0, ref_root)
    import pipesched as ps
    from paper_2510_05186_b200.instance import instance_to_dict
    inst = ps.instance_from_dict(instance_to_dict(inst_ours))
    out = {}

    def run():
        sys.setrecursionlimit(1_000_000)
        t0 = time.perf_counter()
        warm, name = ps.best_feasible(inst, ps.AdaParams())
        t_warm = time.perf_counter() - t0
        sess = ps.start_session(inst, ps.SolveBudget(wall_time_limit=REF_BUDGET[cfg]), warm=warm)
        evs = list(ps.incumbent_stream(sess))
        out.update({"warm_start": name, "warm_seconds": t_warm, "status": sess.outcome.status,
                    "nodes": sess.outcome.nodes, "lower_bound": sess.outcome.lower_bound,
                    "stream": [(t_warm + e.timestamp, e.makespan) for e in evs],
                    "budget_seconds": REF_BUDGET[cfg]})

    threading.stack_size(1 << 29)
    th = threading.Thread(target=run)
    th.start()
    th.join()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", type=int, nargs="+", default=[1, 2, 3])
    ap.add_argument("--cpu-rounds", type=int, default=5, help="config-3 CPU-port rounds (the others run to the end)")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "r02_ttb.json"))
    args = ap.parse_args()
    from paper_2510_05186_b200 import workloads
    res = {"seed": SEED, "moves": MOVES, "cpu_model": None, "configs": {}}
    try:
        res["cpu_model"] = next(l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo") if l.startswith("model name"))
    except Exception:
        pass
    # CUDA context, library load and first-launch costs are paid once per process, not per search
    import torch
    from paper_2510_05186_b200.heuristics import best_feasible
    best_feasible(workloads.config1(), device=0)
    torch.cuda.synchronize()
    for cfg in args.configs:
        inst = workloads.CONFIGS[cfg]()
        row = {}
        row["gpu"], ls, s0 = gpu_arm(inst, cfg)
        row["gpu_ils"], _ = gpu_ils_arm(inst, cfg, REF_BUDGET[cfg])
        cap = args.cpu_rounds if cfg == 3 else 5000
        row["cpu_port"] = cpu_port_arm(inst, cfg, s0, cap, 900.0)
        k = len(row["cpu_port"]["trail"])
        gt = [t for t in row["gpu"]["trail"] if t[0] < row["cpu_port"]["rounds"]]
        row["cpu_port"]["trail_equals_gpu"] = row["cpu_port"]["trail"] == gt
        row["cpu_port"]["compared_improvements"] = k
        if not row["cpu_port"]["complete"]:
            per = row["cpu_port"]["seconds_per_round_mean"]
            last = row["gpu"]["trail"][-1][0] + 1 if row["gpu"]["trail"] else 0
            row["cpu_port"]["seconds_to_gpu_best_projected"] = per * last
        row["reference_bnb"] = ref_arm(inst, cfg) if cfg in (1, 2) else {"skipped": "BASELINE.md §2 plans the B&B stream for configs 1 and 2"}
        row["best_at"] = {str(t): {arm: best_at(row[arm]["stream"], t) if "stream" in row[arm] else None
                                   for arm in ("gpu", "gpu_ils", "cpu_port", "reference_bnb")} for t in MARKS}
        res["configs"][str(cfg)] = row
        print(json.dumps({cfg: row["best_at"]}), flush=True)
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as fh:
        json.dump(res, fh)


if __name__ == "__main__":
    main()
