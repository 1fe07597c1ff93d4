"""Batched candidate evaluation on the GPU (the hot path behind ``run_order``).

``DeviceInstance`` owns one ``ps_instance`` handle (dense tables resident in
HBM); ``evaluate`` / ``evaluate_host`` run ``ps_eval_batch`` /
``ps_eval_batch_host`` over a batch of candidate structures and return
makespan, fp64 bubble ratio, per-stage STRICT peaks, feasibility flags, the
blocked-stage mask of deadlocked candidates and optionally the commit-ordered
event trace.  PyTorch provides device memory and the stream; the kernels are
the hand-written sm_100a code in ``csrc/``.
"""

from __future__ import annotations

import ctypes as C
import threading
import weakref
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .packing import PackedInstance, pack_instance


@dataclass
class EvalResult:
    makespan: object       # int64 [N]; -1 unless feasible
    bubble: object         # float64 [N]
    flags: object          # int32 [N] (PS_FLAG_* bits)
    peak: object = None    # int64 [N, P]
    blocked: object = None  # int32 [N]
    trace_code: object = None   # int32 [N, E]
    trace_start: object = None  # int32 [N, E]

    def feasible(self):
        return (self.flags & N.FLAG_FEASIBLE) != 0


def _ptr(t):
    if t is None:
        return None
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    return t.data_ptr()


class DeviceInstance:
    """A PipelineInstance's tables on one CUDA device."""

    def __init__(self, inst, device: int | None = None, packed: PackedInstance | None = None):
        import torch
        N.require_cuda()
        self.lib = N.load_library()
        self.device = torch.cuda.current_device() if device is None else int(device)
        self.packed = packed if packed is not None else pack_instance(inst)
        pk = self.packed
        self._keep = [np.ascontiguousarray(a) for a in
                      (pk.proc_time, pk.mem_delta, pk.act_size, pk.mem_limit, pk.stage_channel)]
        desc = N.InstanceDesc(pk.num_stages, pk.num_microbatches,
                              *[a.ctypes.data for a in self._keep],
                              pk.num_channels, pk.comm_time, pk.offload_time, int(pk.post_validation))
        h = C.c_void_p()
        N.check(self.lib.ps_instance_create(C.byref(desc), self.device, C.byref(h)))
        self.handle = h
        info = N.InstanceInfo()
        N.check(self.lib.ps_instance_get_info(h, C.byref(info)))
        self.info = info
        self._finalizer = weakref.finalize(self, self.lib.ps_instance_destroy, h)

    @property
    def P(self):
        return self.packed.num_stages

    @property
    def m(self):
        return self.packed.num_microbatches

    def _stream(self, stream):
        import torch
        if stream is None:
            stream = torch.cuda.current_stream(self.device)
        return C.c_void_p(stream.cuda_stream)

    def alloc_results(self, n: int, peak=True, trace=False, blocked=True):
        import torch
        dev = torch.device("cuda", self.device)
        E = self.info.max_events
        return EvalResult(
            makespan=torch.empty(n, dtype=torch.int64, device=dev),
            bubble=torch.empty(n, dtype=torch.float64, device=dev),
            flags=torch.empty(n, dtype=torch.int32, device=dev),
            peak=torch.empty((n, self.P), dtype=torch.int64, device=dev) if peak else None,
            blocked=torch.empty(n, dtype=torch.int32, device=dev) if blocked else None,
            trace_code=torch.empty((n, E), dtype=torch.int32, device=dev) if trace else None,
            trace_start=torch.empty((n, E), dtype=torch.int32, device=dev) if trace else None)

    def _batch_structs(self, n, orders, masks, chans, res: EvalResult, base=None):
        # uint8 op codes (m <= 64) halve what crosses PCIe; int16/uint16 are the general form
        one_byte = str(orders.dtype) in ("uint8", "torch.uint8")
        cb = N.CandBatch(n, _ptr(orders), _ptr(masks), _ptr(chans),
                         int(chans.shape[-1]) if chans is not None else 0,
                         base.handle if base is not None else None, 1 if one_byte else 2)
        rb = N.ResultBatch(_ptr(res.makespan), _ptr(res.bubble), _ptr(res.peak), _ptr(res.flags),
                           _ptr(res.blocked), _ptr(res.trace_code), _ptr(res.trace_start),
                           int(res.trace_code.shape[-1]) if res.trace_code is not None else 0)
        return cb, rb

    def evaluate(self, orders, masks, chans=None, out: EvalResult | None = None, peak=True,
                 trace=False, stream=None, base: "Base | None" = None) -> EvalResult:
        """Device tensors in, device tensors out; asynchronous on `stream`.  With a recorded
        `base`, candidates resume from its last checkpoint before they first differ from it."""
        n = int(orders.shape[0])
        self._check_batch(n, orders, masks, chans, host=False)
        res = out if out is not None else self.alloc_results(n, peak=peak, trace=trace)
        cb, rb = self._batch_structs(n, orders, masks, chans, res, base)
        N.check(self.lib.ps_eval_batch(self.handle, C.byref(cb), C.byref(rb), self._stream(stream)))
        return res

    def evaluate_host(self, orders: np.ndarray, masks: np.ndarray, chans=None, peak=True,
                      trace=False, out: EvalResult | None = None, stream=None,
                      base: "Base | None" = None) -> EvalResult:
        """Host (ideally pinned) numpy buffers in and out: copies inside the call."""
        n = int(orders.shape[0])
        if out is None:
            E = self.info.max_events
            out = EvalResult(np.empty(n, np.int64), np.empty(n, np.float64), np.empty(n, np.int32),
                             np.empty((n, self.P), np.int64) if peak else None, np.empty(n, np.int32),
                             np.empty((n, E), np.int32) if trace else None,
                             np.empty((n, E), np.int32) if trace else None)
        # the library reads these through raw pointers during the call: keep the (possibly
        # converted) arrays bound to locals until it returns
        h_orders, h_masks, h_chans = self._check_batch(n, orders, masks, chans, host=True)
        cb, rb = self._batch_structs(n, h_orders, h_masks, h_chans, out, base)
        N.check(self.lib.ps_eval_batch_host(self.handle, C.byref(cb), C.byref(rb), self._stream(stream)))
        del h_orders, h_masks, h_chans
        return out

    def evaluate_host_delta(self, ref_orders, ref_mask, diff_offset, diffs, flip_offset, flips, peak=True,
                            out: EvalResult | None = None, stream=None, base: "Base | None" = None) -> EvalResult:
        """A host batch given as differences from one reference structure (packing.delta_encode):
        only the differences cross PCIe (ps_eval_batch_host_delta)."""
        n = int(len(diff_offset)) - 1
        if out is None:
            out = EvalResult(np.empty(n, np.int64), np.empty(n, np.float64), np.empty(n, np.int32),
                             np.empty((n, self.P), np.int64) if peak else None, np.empty(n, np.int32))
        keep = [np.ascontiguousarray(ref_orders, np.uint16), np.ascontiguousarray(ref_mask, np.uint32),
                np.ascontiguousarray(diff_offset, np.uint32), np.ascontiguousarray(diffs, np.uint32),
                np.ascontiguousarray(flip_offset, np.uint32), np.ascontiguousarray(flips, np.uint32)]
        pk = self.packed
        if keep[0].shape != (pk.num_stages, pk.order_stride) or keep[1].shape != (pk.mask_words,):
            raise ValueError("reference structure has the wrong shape")
        db = N.DeltaBatch(n, *[a.ctypes.data for a in keep], base.handle if base is not None else None)
        rb = N.ResultBatch(_ptr(out.makespan), _ptr(out.bubble), _ptr(out.peak), _ptr(out.flags),
                           _ptr(out.blocked), None, None, 0, None)
        N.check(self.lib.ps_eval_batch_host_delta(self.handle, C.byref(db), C.byref(rb), self._stream(stream)))
        del keep
        return out

    def _check_batch(self, n, orders, masks, chans, host):
        """Shapes and element types the C ABI reads (include/pipesched_b200.h ps_cand_batch):
        orders [N][P][order_stride] of uint16 (or uint8 when 4m <= 256), masks [N][mask_words]
        of 32-bit words, channel orders [N][G][width] of 32-bit words, all contiguous."""
        pk = self.packed
        if tuple(orders.shape) != (n, pk.num_stages, pk.order_stride):
            raise ValueError(f"orders must be [{n}, {pk.num_stages}, {pk.order_stride}], got {tuple(orders.shape)}")
        if tuple(masks.shape) != (n, pk.mask_words):
            raise ValueError(f"masks must be [{n}, {pk.mask_words}], got {tuple(masks.shape)}")
        if chans is not None and (chans.ndim != 3 or tuple(chans.shape[:2]) != (n, pk.num_channels)):
            raise ValueError(f"channel orders must be [{n}, {pk.num_channels}, width], got {tuple(chans.shape)}")
        if host:
            od = np.dtype(orders.dtype)
            if od == np.uint8 and 4 * pk.num_microbatches > 256:
                raise ValueError("uint8 op codes need 4m <= 256")
            if od not in (np.dtype(np.uint8), np.dtype(np.uint16), np.dtype(np.int16)):
                raise TypeError(f"orders must be uint8/uint16/int16 op codes, got {od}")
            if np.dtype(masks.dtype).itemsize != 4 or np.dtype(masks.dtype).kind not in "iu":
                raise TypeError(f"masks must be 32-bit words, got {masks.dtype}")
            if chans is not None and (np.dtype(chans.dtype).itemsize != 4 or np.dtype(chans.dtype).kind not in "iu"):
                raise TypeError(f"channel orders must be 32-bit words, got {chans.dtype}")
            return (np.ascontiguousarray(orders), np.ascontiguousarray(masks),
                    None if chans is None else np.ascontiguousarray(chans))
        import torch
        if orders.dtype not in (torch.uint8, torch.int16, torch.uint16):
            raise TypeError(f"orders must be uint8/int16/uint16 op codes, got {orders.dtype}")
        if orders.dtype == torch.uint8 and 4 * pk.num_microbatches > 256:
            raise ValueError("uint8 op codes need 4m <= 256")
        if masks.dtype not in (torch.int32, torch.uint32):
            raise TypeError(f"masks must be 32-bit words, got {masks.dtype}")
        if chans is not None and chans.dtype not in (torch.int32, torch.uint32):
            raise TypeError(f"channel orders must be 32-bit words, got {chans.dtype}")
        for name, t in (("orders", orders), ("masks", masks), ("channel orders", chans)):
            if t is not None and (not t.is_cuda or not t.is_contiguous()):
                raise ValueError(f"{name} must be a contiguous CUDA tensor")
        return orders, masks, chans


class Base:
    """A recorded base candidate (``ps_base``) for prefix sharing."""

    def __init__(self, di: DeviceInstance):
        self.di = di
        h = C.c_void_p()
        N.check(di.lib.ps_base_create(di.handle, C.byref(h)))
        self.handle = h
        self._finalizer = weakref.finalize(self, di.lib.ps_base_destroy, h)

    def record(self, orders, mask, stream=None):
        """orders: device int16 [P, stride]; mask: device int32 [mask_words]."""
        N.check(self.di.lib.ps_base_record(self.handle, C.c_void_p(orders.data_ptr()),
                                           C.c_void_p(mask.data_ptr()), self.di._stream(stream)))

    def record_explicit(self, orders, mask, chans, stream=None):
        """With explicit channel orders: chans device int32 [G, width] (ps_base_record_explicit)."""
        N.check(self.di.lib.ps_base_record_explicit(self.handle, C.c_void_p(orders.data_ptr()),
                                                    C.c_void_p(mask.data_ptr()), C.c_void_p(chans.data_ptr()),
                                                    int(chans.shape[-1]), self.di._stream(stream)))

    def read(self, what: int):
        """One recorded table (N.BASE_*) as raw bytes (synchronises the device)."""
        n = C.c_size_t(0)
        N.check(self.di.lib.ps_base_read(self.handle, what, None, C.byref(n)))
        buf = C.create_string_buffer(n.value)
        N.check(self.di.lib.ps_base_read(self.handle, what, buf, C.byref(n)))
        return buf.raw


_CACHE: dict = {}
_CACHE_LOCK = threading.Lock()


def device_instance(inst, device: int | None = None) -> DeviceInstance:
    """Cached DeviceInstance per (instance object, device)."""
    import torch
    N.require_cuda()
    dev = torch.cuda.current_device() if device is None else int(device)
    key = (id(inst), dev)
    with _CACHE_LOCK:
        hit = _CACHE.get(key)
        if hit is not None and hit[0]() is inst:
            return hit[1]
    di = DeviceInstance(inst, dev)
    try:
        ref = weakref.ref(inst, lambda _r, k=key: _CACHE.pop(k, None))
    except TypeError:
        return di
    with _CACHE_LOCK:
        _CACHE[key] = (ref, di)
    return di
