"""Drop-in ``run_order`` on the B200 evaluator.

Same signature, argument meaning and error behaviour as the reference
``pipesched.listsched.run_order`` (listsched.py:167-269): per-stage op orders,
the offloaded F ops, optional explicit per-channel transfer orders in, a
``Schedule`` whose events are in commit order out, ``OrderInfeasible(msg,
stages)`` when no event can start.  The timing is computed by the sm_100a
kernel (``csrc/ps_eval.cuh``) through ``ps_eval_batch``; this module only
encodes the structure and decodes the kernel's commit trace.

``stage_order_of`` / ``channel_order_of`` extract a structure from a timed
schedule (listsched.py:37-49).  ``run_orders`` is the batched form used by
the generators and the cache.
"""

from __future__ import annotations

import weakref

import numpy as np

from . import _native as N
from .instance import OpId, OpKind
from .packing import decode_op, encode_candidate
from . import schedule as _sched


class OrderInfeasible(Exception):
    """The structure admits no feasible timing for this instance."""

    def __init__(self, msg, stages=()):
        super().__init__(msg)
        self.stages = tuple(stages)


def stage_order_of(s, stage: int) -> tuple:
    evs = sorted((ev for ev in s.compute if ev.op.stage == stage), key=lambda e: (e.start, e.op))
    return tuple(ev.op for ev in evs)


def channel_order_of(s, inst, channel: int) -> tuple:
    evs = sorted((ev for ev in s.transfers if inst.stage_channel(ev.op.stage) == channel),
                 key=lambda e: (e.start, e.op, e.kind.value))
    return tuple((ev.op, ev.kind) for ev in evs)


def _events_from_trace(pk, codes, starts, count, types):
    """Rebuild commit-ordered events from the kernel trace (include/pipesched_b200.h): the fields
    are decoded with numpy, the event objects built in one pass."""
    Reload, Offload = types.TransferKind.RELOAD, types.TransferKind.OFFLOAD
    Op, Kind = getattr(types, "OpId", OpId), getattr(types, "OpKind", OpKind)   # the caller's op types
    code = np.asarray(codes[:count]).astype(np.uint32)
    t = np.asarray(starts[:count]).astype(np.int64)
    rank = code >> 30
    i0 = ((code >> 24) & 63).astype(np.int64)
    j0 = ((code >> 2) & 0x3FFFFF).astype(np.int64)
    k = (code & 3).astype(np.int64)
    comp = rank == 0
    end = t + np.where(comp, pk.proc_time[i0, j0, np.where(comp, k, 0)], pk.offload_time)
    kinds = [Kind(x) for x in range(3)]
    compute, transfers = [], []
    CE, TE = types.ComputeEvent, types.TransferEvent
    for r, a, b, kk, s0, e0 in zip(rank.tolist(), i0.tolist(), j0.tolist(), k.tolist(), t.tolist(), end.tolist()):
        op = Op(a + 1, b + 1, kinds[kk])
        if r == 0:
            compute.append(CE(op, s0, e0))
        else:
            transfers.append(TE(op, Reload if r == 1 else Offload, s0, e0))
    return compute, transfers


def run_orders(inst, candidates, explicit=False, device=None, types=None):
    """Evaluate many structures in one kernel launch.

    candidates: list of (stage_orders, offloaded[, channel_orders]).  Returns a
    list with a Schedule per feasible candidate and an OrderInfeasible
    instance per deadlocked one.
    """
    import torch
    from .engine import device_instance
    types = types or _sched
    di = device_instance(inst, device)
    try:
        inst_ref = weakref.ref(inst)
    except TypeError:
        inst_ref = None
    pk = di.packed
    n = len(candidates)
    if n == 0:
        return []
    orders = np.zeros((n, pk.num_stages, pk.order_stride), np.uint16)
    masks = np.zeros((n, pk.mask_words), np.uint32)
    chans = None
    if explicit:
        width = max([len(seq) for c in candidates for seq in c[2].values()] + [1])
        chans = np.full((n, pk.num_channels, width), 0xFFFFFFFF, np.uint32)
    for c, cand in enumerate(candidates):
        encode_candidate(pk, cand[0], cand[1], cand[2] if explicit else None, orders[c], masks[c],
                         chans[c] if explicit else None)
    dev = torch.device("cuda", di.device)
    t_orders = torch.from_numpy(orders.view(np.int16)).to(dev)
    t_masks = torch.from_numpy(masks.view(np.int32)).to(dev)
    t_chans = torch.from_numpy(chans.view(np.int32)).to(dev) if chans is not None else None
    res = di.evaluate(t_orders, t_masks, t_chans, peak=True, trace=True)
    flags = res.flags.cpu().numpy()
    makespan = res.makespan.cpu().numpy()
    bubble = res.bubble.cpu().numpy()
    peak = res.peak.cpu().numpy()
    blocked = res.blocked.cpu().numpy()
    need = [c for c in range(n) if flags[c] & N.FLAG_FEASIBLE]
    codes = res.trace_code.cpu().numpy() if need else None
    starts = res.trace_start.cpu().numpy() if need else None
    out = []
    for c, cand in enumerate(candidates):
        f = int(flags[c])
        if f & N.FLAG_FEASIBLE:
            n_off = len(cand[1])
            count = 3 * pk.num_stages * pk.num_microbatches + 2 * n_off
            comp, trans = _events_from_trace(pk, codes[c], starts[c], count, types)
            metrics = None
            if types is _sched:
                metrics = _sched.EvalMetrics(int(makespan[c]), float(bubble[c]),
                                             {i + 1: int(peak[c, i]) for i in range(pk.num_stages)},
                                             inst_ref)
                out.append(_sched.Schedule.build(comp, trans, cand[1], metrics))
            else:
                out.append(types.Schedule.build(comp, trans, cand[1]))
        elif f & N.FLAG_DEADLOCK:
            m = int(blocked[c]) & 0xFFFFFFFF
            stages = [i + 1 for i in range(pk.num_stages) if (m >> i) & 1]
            out.append(OrderInfeasible(f"no event can start (stages blocked: {stages})", stages))
        elif f & N.FLAG_RANGE:
            raise ValueError(f"candidate {c}: an event time passes 2^31 - 1 quanta, beyond the int32 trace "
                             "output (DESIGN.md §7)")
        else:
            raise ValueError(f"candidate {c} is malformed (flags {f:#x})")
    return out


def run_order(inst, stage_orders: dict, offloaded, channel_orders: dict | None = None, *,
              device=None, types=None):
    """Replay a structure to a timed schedule on the GPU.  Raises OrderInfeasible."""
    offloaded = frozenset(offloaded)
    explicit = channel_orders is not None
    cand = (stage_orders, offloaded, channel_orders) if explicit else (stage_orders, offloaded)
    res = run_orders(inst, [cand], explicit=explicit, device=device, types=types)[0]
    if isinstance(res, OrderInfeasible):
        raise res
    return res
