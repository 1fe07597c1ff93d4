"""Warm-start generators, evaluated as ONE GPU batch.

The reference builds four structures — sequential, 1F1B, PipeOffload-like and
AdaOffload — and times each with ``run_order`` (heuristics.py:50-185);
AdaOffload retries ``run_order`` in a loop, backing off its deepest fill after
every OrderInfeasible (heuristics.py:167-185), and ``best_feasible`` keeps
the first minimum in generator order (heuristics.py:196-210).  The fill
back-off sequence does not depend on the timing, so here every structure of
every generator — the whole back-off sequence included — is built on the host
and evaluated in a single ``run_orders`` launch; AdaOffload's answer is the
first feasible entry of its sequence, exactly the reference loop's result.
"""

from __future__ import annotations

from dataclasses import dataclass

from .instance import OpId, OpKind, PipelineInstance

F, B, W = OpKind.F, OpKind.B, OpKind.W


class InfeasibleSchedule(Exception):
    """The generator's strategy cannot fit this instance's memory limits."""


class NoFeasibleSchedule(Exception):
    """No generator produced a feasible schedule."""


@dataclass(frozen=True)
class AdaParams:
    tolerance: int = 0

    def __post_init__(self):
        if self.tolerance < 0:
            raise ValueError("tolerance must be >= 0")


def sequential_order(inst, stage: int) -> tuple:
    return tuple(OpId(stage, j, k) for j in range(1, inst.num_microbatches + 1) for k in (F, B, W))


def filled_order(inst, stage: int, fill: int) -> tuple:
    """`fill` forwards first, then B, W and the next forward per microbatch
    (heuristics.py:87-96; 1F1B is fill = min(P - i + 1, m), heuristics.py:64-72)."""
    m = inst.num_microbatches
    seq = [OpId(stage, j, F) for j in range(1, fill + 1)]
    for k in range(1, m + 1):
        seq += [OpId(stage, k, B), OpId(stage, k, W)]
        if fill + k <= m:
            seq.append(OpId(stage, fill + k, F))
    return tuple(seq)


def _backward_estimates(inst):
    """First-backward start estimate per stage from per-stage max runtimes (heuristics.py:110-125)."""
    P, comm = inst.num_stages, inst.comm_time
    tf = {i: max(inst.proc_time[OpId(i, j, F)] for j in range(1, inst.num_microbatches + 1))
          for i in range(1, P + 1)}
    tb = {i: max(inst.proc_time[OpId(i, j, B)] for j in range(1, inst.num_microbatches + 1))
          for i in range(1, P + 1)}
    down = sum(tf.values()) + (P - 1) * comm
    return {s: down + sum(tb[i] for i in range(s + 1, P + 1)) + (P - s) * comm for s in range(1, P + 1)}


def ada_fill_counts(inst, tolerance: int = 0) -> dict:
    """Greedy per-stage fill projection (heuristics.py:128-164)."""
    P, m, toff = inst.num_stages, inst.num_microbatches, inst.offload_time
    est = _backward_estimates(inst)
    fills, f_end_prev = {}, {}
    for s in range(1, P + 1):
        fill, f_end, o_end, backlog = 0, 0, 0, 0
        for j in range(1, m + 1):
            if j > 1 and max(f_end, o_end + toff) >= est[s] + tolerance:
                break
            op = OpId(s, j, F)
            delta, gamma = inst.mem_delta[op], inst.act_size.get(op, 0)
            if j > 1 and backlog + delta > inst.mem_limit[s]:
                break
            start = f_end if s == 1 else max(f_end, f_end_prev.get((s - 1, j), 0) + inst.comm_time)
            fill = j
            f_end = start + inst.proc_time[op]
            o_end = max(o_end, f_end) + toff
            backlog += delta - gamma
            f_end_prev[(s, j)] = f_end
        for j in range(fill + 1, m + 1):
            start = f_end if s == 1 else max(f_end, f_end_prev.get((s - 1, j), 0) + inst.comm_time)
            f_end = start + inst.proc_time[OpId(s, j, F)]
            f_end_prev[(s, j)] = f_end
        fills[s] = max(fill, 1)
    return fills


def ada_backoff_sequence(inst, tolerance: int = 0) -> list:
    """Every fill vector the reference loop would try, in order (heuristics.py:172-185)."""
    fills = ada_fill_counts(inst, tolerance)
    seq = [dict(fills)]
    while True:
        reducible = [i for i in fills if fills[i] > 1]
        if not reducible:
            return seq
        deepest = max(reducible, key=lambda i: (fills[i], i))
        fills[deepest] -= 1
        seq.append(dict(fills))


def generator_structures(inst, params: AdaParams = AdaParams()):
    """(orders, offloaded) of ada (initial fills), pipeoffload, 1f1b, sequential."""
    P, m = inst.num_stages, inst.num_microbatches
    everything = frozenset(inst.offloadable_ops())
    fills = ada_fill_counts(inst, params.tolerance)
    return [
        ({i: filled_order(inst, i, fills[i]) for i in range(1, P + 1)}, everything),
        ({i: filled_order(inst, i, 1) for i in range(1, P + 1)}, everything),
        ({i: filled_order(inst, i, min(P - i + 1, m)) for i in range(1, P + 1)}, frozenset()),
        ({i: sequential_order(inst, i) for i in range(1, P + 1)}, frozenset()),
    ]


def _row_codes(m: int, fill: int) -> "np.ndarray":
    """filled_order's op codes ((microbatch - 1) << 2 | kind), the same for every stage."""
    import numpy as np
    codes = [(j << 2) | 0 for j in range(fill)]
    for k in range(m):
        codes += [(k << 2) | 1, (k << 2) | 2]
        if fill + k < m:
            codes.append(((fill + k) << 2) | 0)
    return np.asarray(codes, np.uint16)


def generate_all(inst: PipelineInstance, params: AdaParams = AdaParams(), device=None, types=None,
                 spans: dict | None = None) -> dict:
    """Every generator's schedule (or InfeasibleSchedule) from one batched evaluation.

    The whole AdaOffload back-off sequence (738 structures at 32 x 256) is encoded from one row per
    fill value (filled_order does not depend on the stage) and evaluated in one launch without
    traces; only the structures that become answers — AdaOffload's first feasible entry and the
    other three generators — are re-run with their traces and decoded into Schedules (of the
    reference's own types with ``types=``; ``spans`` receives each answer's makespan)."""
    import numpy as np
    import torch
    from .engine import device_instance
    from .listsched import OrderInfeasible, run_orders
    P, m = inst.num_stages, inst.num_microbatches
    everything = frozenset(inst.offloadable_ops())
    backoff = ada_backoff_sequence(inst, params.tolerance)
    fill_sets = [f for f in backoff] + [{i: 1 for i in range(1, P + 1)},
                                        {i: min(P - i + 1, m) for i in range(1, P + 1)}]
    n_ada = len(backoff)
    di = device_instance(inst, device)
    pk = di.packed
    n = len(fill_sets) + 1
    orders = np.zeros((n, P, pk.order_stride), np.uint16)
    masks = np.zeros((n, pk.mask_words), np.uint32)
    rows = {}
    for c, f in enumerate(fill_sets):
        for i in range(1, P + 1):
            r = rows.get(f[i])
            if r is None:
                r = rows[f[i]] = _row_codes(m, f[i])
            orders[c, i - 1, :3 * m] = r
    seq_row = np.asarray([(j << 2) | k for j in range(m) for k in range(3)], np.uint16)
    orders[n - 1, :, :3 * m] = seq_row
    for op in everything:
        b = (op[0] - 1) * m + (op[1] - 1)
        masks[:n - 2, b >> 5] |= np.uint32(1 << (b & 31))          # ada and pipeoffload offload everything
    dev = torch.device("cuda", di.device)
    res = di.evaluate(torch.from_numpy(orders.view(np.int16)).to(dev), torch.from_numpy(masks.view(np.int32)).to(dev),
                      peak=False)
    flags = res.flags.cpu().numpy()
    blocked = res.blocked.cpu().numpy()

    def stages_of(c):
        return [i + 1 for i in range(P) if (int(blocked[c]) >> i) & 1]

    ada_idx = next((c for c in range(n_ada) if flags[c] & 1), None)
    picks = {"ada": ada_idx, "pipeoffload": n_ada, "1f1b": n_ada + 1, "sequential": n_ada + 2}
    structs = {}
    for name, c in picks.items():
        if c is None or not flags[c] & 1:
            continue
        if name == "sequential":
            structs[name] = ({i: sequential_order(inst, i) for i in range(1, P + 1)}, frozenset())
        else:
            f = fill_sets[c]
            structs[name] = ({i: filled_order(inst, i, f[i]) for i in range(1, P + 1)},
                             frozenset() if name == "1f1b" else everything)
    names = list(structs)
    decoded = dict(zip(names, run_orders(inst, [structs[k] for k in names], device=device, types=types)))
    if spans is not None:
        makespans = res.makespan.cpu().numpy()
        spans.update({name: int(makespans[c]) for name, c in picks.items() if c is not None and flags[c] & 1})
    seq_ok = all(inst.mem_delta[OpId(i, j, F)] <= inst.mem_limit[i]
                 for i in range(1, P + 1) for j in range(1, m + 1))
    out = {}
    for name in GENERATOR_ORDER:
        got = decoded.get(name)
        if name == "sequential" and not seq_ok:
            out[name] = InfeasibleSchedule("a stage cannot hold one activation")
            continue
        if got is not None and not isinstance(got, OrderInfeasible):
            out[name] = got
            continue
        c = picks[name] if name != "ada" else n_ada - 1
        if name == "ada" or name == "pipeoffload":
            out[name] = InfeasibleSchedule(f"offload-everything exceeds memory (blocked stages: {stages_of(c)})")
        elif name == "1f1b":
            out[name] = InfeasibleSchedule(f"1F1B exceeds memory (blocked stages: {stages_of(c)})")
        else:
            out[name] = InfeasibleSchedule(f"sequential blocked (stages {stages_of(c)})")
    return out


def _pick(inst, name, params):
    r = generate_all(inst, params)[name]
    if isinstance(r, Exception):
        raise r
    return r


def sequential_schedule(inst):
    return _pick(inst, "sequential", AdaParams())


def one_f_one_b(inst):
    return _pick(inst, "1f1b", AdaParams())


def pipeoffload_like(inst):
    return _pick(inst, "pipeoffload", AdaParams())


def ada_offload(inst, params: AdaParams = AdaParams()):
    return _pick(inst, "ada", params)


GENERATOR_ORDER = ("ada", "pipeoffload", "1f1b", "sequential")


def best_feasible(inst, params: AdaParams = AdaParams(), device=None):
    """Minimum-makespan generator output as (schedule, name); first wins ties (heuristics.py:196-210)."""
    from .schedule import makespan
    allr = generate_all(inst, params, device)
    best = None
    for name in GENERATOR_ORDER:
        s = allr[name]
        if isinstance(s, Exception):
            continue
        span = makespan(s, inst)
        if best is None or span < best[0]:
            best = (span, s, name)
    if best is None:
        raise NoFeasibleSchedule("all generators failed on this instance")
    return best[1], best[2]


def fill_profile(s, inst) -> dict:
    """Per stage: forwards started before the stage's first backward (heuristics.py:38-45)."""
    out = {}
    for i in range(1, inst.num_stages + 1):
        evs = [ev for ev in s.compute if ev.op.stage == i]
        first_b = min(ev.start for ev in evs if ev.op.kind is B)
        out[i] = sum(1 for ev in evs if ev.op.kind is F and ev.start < first_b)
    return out
