"""Dense encodings shared by the host API, the C ABI and the oracle.

Instance tables (``pack_instance``) follow ``ps_instance_desc``; candidates
(``encode_candidates``) follow ``ps_cand_batch``:

* stage order row i: u16 op codes ``(j-1) << 2 | kind`` padded to
  ``order_stride`` (a multiple of 8, >= 3m);
* offload mask: bit ``(i-1)*m + (j-1)`` of ``ceil(P*m/32)`` u32 words;
* explicit channel orders: u32 ``kind << 31 | (i-1) << 16 | (j-1)``
  (kind 1 = reload), padded with 0xFFFFFFFF.

Stage/microbatch indices are 1-based in ``OpId`` exactly as in the reference
(instance.py:51-59); every encoding here is 0-based.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .instance import OpId, OpKind

PAD_CHANNEL = 0xFFFFFFFF


@dataclass(frozen=True)
class PackedInstance:
    num_stages: int
    num_microbatches: int
    proc_time: np.ndarray      # int64 [P, m, 3]
    mem_delta: np.ndarray      # int64 [P, m, 3]
    act_size: np.ndarray       # int64 [P, m]
    mem_limit: np.ndarray      # int64 [P]
    stage_channel: np.ndarray  # int32 [P]
    num_channels: int
    comm_time: int
    offload_time: int
    post_validation: bool

    @property
    def order_stride(self) -> int:
        return (3 * self.num_microbatches + 7) & ~7

    @property
    def mask_words(self) -> int:
        return (self.num_stages * self.num_microbatches + 31) // 32

    @property
    def busy_time(self) -> int:
        return int(self.proc_time.sum())


def pack_instance(inst) -> PackedInstance:
    """Dense tables of a PipelineInstance (ours or the reference's: duck-typed)."""
    P, m = inst.num_stages, inst.num_microbatches
    proc = np.empty((P, m, 3), np.int64)
    delta = np.empty((P, m, 3), np.int64)
    act = np.zeros((P, m), np.int64)
    for i in range(1, P + 1):
        for j in range(1, m + 1):
            for k in range(3):
                op = OpId(i, j, OpKind(k))
                proc[i - 1, j - 1, k] = inst.proc_time[op]
                delta[i - 1, j - 1, k] = inst.mem_delta[op]
            act[i - 1, j - 1] = inst.act_size.get(OpId(i, j, OpKind.F), 0)
    limit = np.array([inst.mem_limit[i] for i in range(1, P + 1)], np.int64)
    chan = np.array([inst.stage_channel(i) for i in range(1, P + 1)], np.int32)
    return PackedInstance(P, m, proc, delta, act, limit, chan, len(inst.topology_groups),
                          int(inst.comm_time), int(inst.offload_time), bool(inst.post_validation))


def op_code(op) -> int:
    return ((op[1] - 1) << 2) | int(op[2])


def decode_op(stage0: int, code: int) -> OpId:
    return OpId(stage0 + 1, (code >> 2) + 1, OpKind(code & 3))


ROW_END = 0xFFFF          # stage-row terminator for rows shorter than 3m (include/pipesched_b200.h)


class ChannelMismatch(ValueError):
    """An explicit channel order lists a transfer of a stage that the instance's topology serves
    on another channel.  The reference replays such an order on the listed channel
    (listsched.py:233-239); the kernels serve each stage's transfers on its own channel only, so
    the drop-in rejects the order instead: ``cache.adapt_batch`` reports the entry
    as not adaptable (None) and the integrate wrapper raises the reference's OrderInfeasible."""


def _kind_is_reload(kind) -> bool:
    return getattr(kind, "value", kind) == "reload"


def encode_candidate(pk: PackedInstance, stage_orders, offloaded, channel_orders=None,
                     orders_out=None, mask_out=None, chan_out=None):
    """One candidate into preallocated rows (or fresh arrays).  Raises
    ValueError for structurally malformed input and KeyError (as the
    reference does at listsched.py:157/201) for offloading an op that has no
    offloadable activation."""
    P, m = pk.num_stages, pk.num_microbatches
    if orders_out is None:
        orders_out = np.zeros((P, pk.order_stride), np.uint16)
    if mask_out is None:
        mask_out = np.zeros(pk.mask_words, np.uint32)
    for i in range(1, P + 1):
        try:
            row = stage_orders[i]
        except KeyError:
            raise KeyError(i) from None
        n = len(row)
        if n > 3 * m:
            raise ValueError(f"stage {i} order has {n} ops, more than the stage's {3 * m}")
        codes = np.fromiter(((op[1] - 1) << 2 | int(op[2]) for op in row), np.int64, n)
        stages = np.fromiter((op[0] for op in row), np.int64, n)
        mbs = codes >> 2
        if (stages != i).any() or (mbs < 0).any() or (mbs >= m).any():
            raise ValueError(f"stage {i} order holds ops of another stage or microbatch range")
        # a row that repeats ops or is short is replayed literally, as the reference does
        # (listsched.py:206-252): it ends in OrderInfeasible (ps_literal.cu)
        orders_out[i - 1, :n] = codes
        if n < 3 * m:
            orders_out[i - 1, n] = ROW_END
    mask_out[:] = 0
    for op in offloaded:
        i, j, k = op
        if int(k) != 0 or not (1 <= i <= P and 1 <= j <= m) or pk.act_size[i - 1, j - 1] <= 0:
            raise KeyError(op)
        b = (i - 1) * m + (j - 1)
        mask_out[b >> 5] |= np.uint32(1 << (b & 31))
    if channel_orders is not None:
        width = chan_out.shape[1] if chan_out is not None else max(
            [len(v) for v in channel_orders.values()] + [1])
        if chan_out is None:
            chan_out = np.full((pk.num_channels, width), PAD_CHANNEL, np.uint32)
        chan_out[:] = PAD_CHANNEL
        off = set(tuple(x) for x in offloaded)
        for g in range(pk.num_channels):
            seq = channel_orders.get(g, ())
            if len(seq) > width:
                raise ValueError(f"channel {g} order longer than chan_stride {width}")
            seen = set()
            for q, (op, kind) in enumerate(seq):
                i, j, k = op
                if tuple(op) not in off:
                    raise KeyError(op)
                if pk.stage_channel[i - 1] != g:
                    raise ChannelMismatch(f"{op} is not served by channel {g}")
                rel = _kind_is_reload(kind)
                if (tuple(op), rel) in seen:
                    raise ValueError(f"duplicate transfer {op} on channel {g}")
                seen.add((tuple(op), rel))
                chan_out[g, q] = (int(rel) << 31) | ((i - 1) << 16) | (j - 1)
    return orders_out, mask_out, chan_out


def encode_candidates(pk: PackedInstance, candidates, explicit: bool = False):
    """List of (stage_orders, offloaded[, channel_orders]) -> dense numpy batch."""
    n = len(candidates)
    orders = np.zeros((n, pk.num_stages, pk.order_stride), np.uint16)
    masks = np.zeros((n, pk.mask_words), np.uint32)
    chans = None
    if explicit:
        width = max([len(seq) for c in candidates for seq in c[2].values()] + [1])
        chans = np.full((n, pk.num_channels, width), PAD_CHANNEL, np.uint32)
    for c, cand in enumerate(candidates):
        encode_candidate(pk, cand[0], cand[1], cand[2] if explicit else None, orders[c], masks[c],
                         chans[c] if explicit else None)
    return orders, masks, chans


def decode_orders(pk: PackedInstance, orders_row: np.ndarray) -> dict:
    """[P, stride] op codes -> {stage: tuple(OpId)}."""
    L = 3 * pk.num_microbatches
    return {i + 1: tuple(decode_op(i, int(c)) for c in orders_row[i, :L]) for i in range(pk.num_stages)}


def decode_mask(pk: PackedInstance, mask_row: np.ndarray) -> frozenset:
    m = pk.num_microbatches
    out = []
    for b in range(pk.num_stages * m):
        if (int(mask_row[b >> 5]) >> (b & 31)) & 1:
            out.append(OpId(b // m + 1, b % m + 1, OpKind.F))
    return frozenset(out)


def delta_encode(ref_orders: np.ndarray, ref_mask: np.ndarray, orders: np.ndarray, masks: np.ndarray,
                 chunk: int = 4096):
    """A batch as differences from one reference structure (ps_delta_batch): returns
    (diff_offset uint32 [N+1], diffs uint32 [D][2] = (stage << 16 | pos, code),
     flip_offset uint32 [N+1], flips uint32 [F] = offload bit index)."""
    n = int(orders.shape[0])
    ref_orders = np.asarray(ref_orders, np.uint16)
    ref_mask = np.asarray(ref_mask, np.uint32)
    d_parts, f_parts = [], []
    dcount = np.zeros(n, np.int64)
    fcount = np.zeros(n, np.int64)
    for lo in range(0, n, chunk):
        o = np.asarray(orders[lo:lo + chunk]).view(np.uint16)
        nn, ss, pp = np.nonzero(o != ref_orders[None])
        dcount[lo:lo + len(o)] = np.bincount(nn, minlength=len(o))
        d_parts.append(np.stack([(ss.astype(np.uint32) << 16) | pp.astype(np.uint32),
                                 o[nn, ss, pp].astype(np.uint32)], axis=1))
        x = np.asarray(masks[lo:lo + chunk]).view(np.uint32) ^ ref_mask[None]
        bits = np.unpackbits(x.view(np.uint8), axis=1, bitorder="little")
        cn, cb = np.nonzero(bits)
        fcount[lo:lo + len(o)] = np.bincount(cn, minlength=len(o))
        f_parts.append(cb.astype(np.uint32))
    doff = np.zeros(n + 1, np.uint32)
    doff[1:] = np.cumsum(dcount)
    foff = np.zeros(n + 1, np.uint32)
    foff[1:] = np.cumsum(fcount)
    diffs = np.ascontiguousarray(np.concatenate(d_parts) if d_parts else np.zeros((0, 2), np.uint32))
    flips = np.ascontiguousarray(np.concatenate(f_parts) if f_parts else np.zeros(0, np.uint32))
    return doff, diffs, foff, flips
