"""Generate golden fixtures by running the REFERENCE implementation.

Run here (the reference is importable only in the build container):

    python tests/golden/make_golden.py

It imports /root/reference/pkg/src/pipesched unmodified and records, for a
corpus of instances and candidate structures, exactly what the reference
returns: run_order's compute and transfer events in commit order (or
OrderInfeasible with its stages), makespan, memory_trace(STRICT) peaks and the
unrounded bubble ratio (cli.py:156), in derived and explicit channel mode.
It also records the reference generators' outputs (best_feasible and the four
strategies) and random_instance(seed) tables.  Output: gzip JSON files next
to this script; the GPU box never needs the reference.
"""

from __future__ import annotations

import gzip
import json
import random
import sys
import time
from pathlib import Path

REF = "/root/reference/pkg/src"
HERE = Path(__file__).resolve().parent
sys.path.insert(0, REF)
sys.path.insert(0, str(HERE.parents[1]))

import pipesched as ps  # noqa: E402  (the reference)
from pipesched import heuristics as rh  # noqa: E402

from paper_2510_05186_b200 import workloads  # noqa: E402
from paper_2510_05186_b200.instance import instance_to_dict as our_to_dict  # noqa: E402

F, B, W = ps.OpKind.F, ps.OpKind.B, ps.OpKind.W


def to_ref(inst):
    return ps.instance_from_dict(our_to_dict(inst))


def enc_orders(inst, orders):
    return [[((op.microbatch - 1) << 2) | int(op.kind) for op in orders[i]]
            for i in range(1, inst.num_stages + 1)]


def enc_off(offloaded):
    return sorted([op.stage, op.microbatch] for op in offloaded)


def enc_chan(inst, chans):
    return [[[op.stage, op.microbatch, int(kind is ps.TransferKind.RELOAD)] for op, kind in chans.get(g, ())]
            for g in range(len(inst.topology_groups))]


def record(inst, orders, offloaded, chans=None):
    t0 = time.perf_counter()
    case = {"orders": enc_orders(inst, orders), "offloaded": enc_off(offloaded)}
    if chans is not None:
        case["channel_orders"] = enc_chan(inst, chans)
    try:
        s = ps.run_order(inst, orders, offloaded, chans)
    except ps.OrderInfeasible as e:
        case["infeasible"] = list(e.stages)
        case["ref_seconds"] = time.perf_counter() - t0
        return case, None
    span = ps.makespan(s, inst)
    tr = ps.memory_trace(s, inst, ps.MemorySemantics.STRICT)
    busy = sum(inst.proc_time.values())
    case.update({
        "makespan": span,
        "bubble": repr(1.0 - busy / (inst.num_stages * span)),
        "peak": [tr.peak[i] for i in range(1, inst.num_stages + 1)],
        "compute": [[e.op.stage, e.op.microbatch, int(e.op.kind), e.start] for e in s.compute],
        "transfers": [[e.op.stage, e.op.microbatch, int(e.kind is ps.TransferKind.RELOAD), e.start]
                      for e in s.transfers],
        "valid": ps.validate(s, inst).ok,
        "ref_seconds": time.perf_counter() - t0,
    })
    return case, s


def filled(inst, i, fill):
    return rh._filled_order(inst, i, fill)


def base_structures(inst):
    """Generator structures (whether or not they are feasible)."""
    P, m = inst.num_stages, inst.num_microbatches
    offl_all = frozenset(inst.offloadable_ops())
    out = []
    out.append(({i: tuple(ps.OpId(i, j, c) for j in range(1, m + 1) for c in (F, B, W))
                 for i in range(1, P + 1)}, frozenset()))
    out.append(({i: rh._one_f_one_b_order(inst, i, min(P - i + 1, m)) for i in range(1, P + 1)}, frozenset()))
    out.append(({i: filled(inst, i, 1) for i in range(1, P + 1)}, offl_all))
    fills = rh._ada_fill_counts(inst, 0)
    out.append(({i: filled(inst, i, fills[i]) for i in range(1, P + 1)}, offl_all))
    return out


def perturb(inst, orders, offloaded, rng, n_swaps, p_toggle):
    P = inst.num_stages
    new = {i: list(orders[i]) for i in orders}
    for _ in range(n_swaps):
        i = rng.randint(1, P)
        row = new[i]
        if len(row) < 2:
            continue
        a = rng.randrange(len(row))
        b = min(len(row) - 1, max(0, a + rng.choice([-3, -2, -1, 1, 2, 3])))
        row.insert(b, row.pop(a))
    off = set(offloaded)
    for x in inst.offloadable_ops():
        if rng.random() < p_toggle:
            off ^= {x}
    return {i: tuple(v) for i, v in new.items()}, frozenset(off)


def random_fills(inst, rng, p_off):
    P, m = inst.num_stages, inst.num_microbatches
    fills = sorted((rng.randint(1, m) for _ in range(P)), reverse=True)
    orders = {i: filled(inst, i, fills[i - 1]) for i in range(1, P + 1)}
    off = frozenset(x for x in inst.offloadable_ops() if rng.random() < p_off)
    return orders, off


def nonuniform_instance(rng, P, m, big=False):
    """Per-(stage, microbatch) random values through the JSON codec (not microbatch symmetric)."""
    proc, mem, act = [], [], []
    for i in range(P):
        pr, me, ac = [], [], []
        for j in range(m):
            pr.append([rng.randint(1, 5), rng.randint(1, 5), rng.randint(1, 5)])
            a = rng.randint(2, 9) if not big else rng.randint(2**33, 2**34) * 2 + 1
            dB = -((a + 1) // 2) - (rng.randint(0, 1) if a > 3 else 0)
            me.append([a, dB, -a - dB])
            ac.append([rng.choice([0, a, max(1, a // 2)]), 0, 0])
        proc.append(pr)
        mem.append(me)
        act.append(ac)
    limits = []
    for i in range(P):
        mx = max(r[0] for r in mem[i])
        limits.append(rng.randint(mx, mx * max(1, m // 2) + 1))
    groups = None
    if P >= 2 and rng.random() < 0.4:
        stages = list(range(1, P + 1))
        rng.shuffle(stages)
        cut = rng.randint(1, P - 1)
        groups = [sorted(stages[:cut]), sorted(stages[cut:])]
    d = {"num_stages": P, "num_microbatches": m, "proc_times": proc, "comm_time": rng.randint(0, 3),
         "offload_time": rng.randint(0, 4), "mem_deltas": mem, "act_sizes": act, "mem_limits": limits,
         "post_validation": rng.random() < 0.3}
    if groups:
        d["topology_groups"] = groups
    return ps.instance_from_dict(d)


def corpus_cases(name, insts, rng, per_inst, with_explicit=True):
    cases = []
    for inst in insts:
        entry = {"instance": ps.instance_to_dict(inst), "cases": []}
        structs = base_structures(inst)
        for orders, off in structs:
            c, s = record(inst, orders, off)
            entry["cases"].append(c)
            if s is not None and with_explicit:
                so = {i: ps.stage_order_of(s, i) for i in range(1, inst.num_stages + 1)}
                co = {g: ps.channel_order_of(s, inst, g) for g in range(len(inst.topology_groups))}
                entry["cases"].append(record(inst, so, s.offloaded, co)[0])
        for k in range(per_inst):
            if k % 3 == 2:
                orders, off = random_fills(inst, rng, rng.choice([0.0, 0.5, 1.0]))
            else:
                o, f = structs[rng.randrange(len(structs))]
                orders, off = perturb(inst, o, f, rng, rng.randint(0, 4), rng.choice([0.0, 0.1, 0.3]))
            c, s = record(inst, orders, off)
            entry["cases"].append(c)
            if s is not None and with_explicit and k % 2 == 0:
                so = {i: ps.stage_order_of(s, i) for i in range(1, inst.num_stages + 1)}
                co = {g: ps.channel_order_of(s, inst, g) for g in range(len(inst.topology_groups))}
                entry["cases"].append(record(inst, so, s.offloaded, co)[0])
        cases.append(entry)
    return {"name": name, "instances": cases}


def generator_golden(insts):
    out = []
    for inst in insts:
        row = {"instance": ps.instance_to_dict(inst), "generators": {}}
        for name, gen in (("sequential", ps.sequential_schedule), ("1f1b", ps.one_f_one_b),
                          ("pipeoffload", ps.pipeoffload_like),
                          ("ada", lambda i: ps.ada_offload(i, ps.AdaParams()))):
            try:
                s = gen(inst)
                row["generators"][name] = {
                    "makespan": ps.makespan(s, inst),
                    "orders": enc_orders(inst, {i: ps.stage_order_of(s, i) for i in range(1, inst.num_stages + 1)}),
                    "offloaded": enc_off(s.offloaded),
                    "peak": [ps.memory_trace(s, inst).peak[i] for i in range(1, inst.num_stages + 1)]}
            except ps.InfeasibleSchedule as e:
                row["generators"][name] = {"infeasible": str(e)}
        try:
            s, name = ps.best_feasible(inst, ps.AdaParams())
            row["best_feasible"] = {"name": name, "makespan": ps.makespan(s, inst)}
        except ps.NoFeasibleSchedule:
            row["best_feasible"] = None
        row["ada_fills"] = [rh._ada_fill_counts(inst, 0)[i] for i in range(1, inst.num_stages + 1)]
        out.append(row)
    return out


def dump(obj, fname):
    path = HERE / fname
    with gzip.open(path, "wt") as fh:
        json.dump(obj, fh, separators=(",", ":"))
    print(f"wrote {path} ({path.stat().st_size} bytes)")


def main():
    rng = random.Random(20251005)
    t0 = time.time()
    # 1. reference test-suite instances
    test_insts = [ps.make_uniform_instance(*a) for a in [
        (2, 3, 1, 1, 1, 1, 1, 2, 3), (1, 2, 1, 1, 1, 0, 1, 2, 4), (1, 2, 1, 1, 1, 0, 1, 2, 1),
        (1, 1, 1, 1, 1, 0, 1, 2, 4), (4, 6, 1, 1, 1, 0, 1, 2, 3), (2, 2, 1, 1, 1, 1, 1, 2, 4),
        (3, 4, 1, 1, 1, 1, 1, 2, 8), (4, 8, 1, 1, 1, 1, 1, 2, 4), (4, 4, 1, 1, 1, 1, 1, 2, 1),
        (3, 4, 1, 1, 1, 0, 1, 2, 12), (2, 3, 1, 1, 1, 1, 6, 2, 1), (1, 2, 2, 2, 2, 0, 1, 2, 2),
        (2, 4, 1, 1, 1, 1, 1, 2, 8), (4, 8, 2, 2, 1, 1, 1, 2, 8), (2, 3, 1, 1, 1, 0, 1, 2, 3)]]
    test_insts += [ps.make_uniform_instance(2, 1, 1, 1, 1, 1, 1, 2, 4, post_validation=True)]
    test_insts += [ps.random_instance(s, *shape, mem_profile=prof)
                   for s in range(0, 40) for shape, prof in [(((1, 3), (2, 2), (3, 2), (2, 3))[s % 4],
                                                              "tight" if s % 2 else "ample")]]
    dump(corpus_cases("reference_tests", test_insts, rng, 6), "ref_tests.json.gz")
    print("t", time.time() - t0)
    # 2. fuzz: uniform variety, topology groups, post-validation, zero comm/offload, non-uniform
    fuzz = []
    for k in range(60):
        P, m = rng.randint(1, 6), rng.randint(1, 8)
        groups = None
        if P >= 3 and rng.random() < 0.4:
            groups = [[1, 2]] + [[s] for s in range(3, P + 1)]
        fuzz.append(ps.make_uniform_instance(P, m, rng.randint(1, 4), rng.randint(1, 4), rng.randint(1, 4),
                                             rng.randint(0, 3), rng.randint(0, 5), rng.randint(2, 6),
                                             rng.randint(1, 6), post_validation=rng.random() < 0.3,
                                             topology_groups=groups))
    for k in range(40):
        fuzz.append(nonuniform_instance(rng, rng.randint(1, 5), rng.randint(1, 7)))
    for k in range(6):
        fuzz.append(nonuniform_instance(rng, rng.randint(2, 4), rng.randint(2, 5), big=True))
    dump(corpus_cases("fuzz", fuzz, rng, 8), "fuzz.json.gz")
    print("t", time.time() - t0)
    # 3. BASELINE config shapes (the reference is slow here: few candidates)
    cfg = []
    c1 = to_ref(workloads.config1())
    cfg.append(corpus_cases("config1", [c1], rng, 12)["instances"][0])
    c2 = to_ref(workloads.config2())
    cfg.append(corpus_cases("config2", [c2], rng, 4, with_explicit=False)["instances"][0])
    c3 = to_ref(workloads.config3())
    cfg.append(corpus_cases("config3", [c3], rng, 3, with_explicit=False)["instances"][0])
    dump({"name": "configs", "instances": cfg}, "configs.json.gz")
    print("t", time.time() - t0)
    # 4. generators and random_instance tables
    gen_insts = test_insts[:16] + [to_ref(workloads.config1()), to_ref(workloads.config2())]
    gens = generator_golden(gen_insts)
    rnd = [{"seed": s, "P": P, "m": m, "profile": prof,
            "instance": ps.instance_to_dict(ps.random_instance(s, P, m, mem_profile=prof))}
           for s in range(12) for (P, m, prof) in [(2, 3, "tight"), (3, 2, "ample")]]
    dump({"generators": gens, "random_instances": rnd}, "generators.json.gz")
    print("done in", time.time() - t0)


if __name__ == "__main__":
    main()
