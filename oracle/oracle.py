"""ctypes binding of the C oracle (ps_oracle.c).  TEST INFRASTRUCTURE ONLY.

A CPU restatement of the reference hot path (listsched.run_order + makespan +
memory_trace(STRICT) + bubble, see ps_oracle.h for the line map) and of the
local-search move definition.  Only tests/, __graft_entry__.smoke() and the
CPU-baseline legs of bench.py may import this module, and only as the checker
or the timed CPU baseline — the product path never routes through it.
Parity of this restatement with the reference is pinned by
tests/test_oracle.py against the reference-generated fixtures in tests/golden.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "_build" / "libps_oracle.so"


def build() -> Path:
    src = [HERE / "ps_oracle.c", HERE / "ps_oracle.h", HERE / "Makefile"]
    if not LIB.exists() or any(p.stat().st_mtime > LIB.stat().st_mtime for p in src):
        subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB


class _Inst(C.Structure):
    _fields_ = [("P", C.c_int32), ("m", C.c_int32), ("G", C.c_int32),
                ("proc", C.c_void_p), ("delta", C.c_void_p), ("act", C.c_void_p),
                ("limit", C.c_void_p), ("chan", C.c_void_p),
                ("comm", C.c_int64), ("toff", C.c_int64), ("post", C.c_int32)]


class _Res(C.Structure):
    _fields_ = [("makespan", C.c_int64), ("bubble", C.c_double), ("peak", C.c_void_p),
                ("flags", C.c_uint32), ("blocked", C.c_uint32), ("trace_code", C.c_void_p),
                ("trace_start", C.c_void_p), ("n_events", C.c_int32)]


class _Moves(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("shift_permille", C.c_uint32), ("max_shift", C.c_uint32)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(str(build()))
        _lib.or_run_order.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p,
                                      C.c_int32, C.POINTER(_Res)]
        _lib.or_eval_batch.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_int32, C.c_void_p,
                                       C.c_int32, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p,
                                       C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32]
        _lib.or_philox4x32_10.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        _lib.or_neighbour.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p,
                                      C.POINTER(_Moves), C.c_uint64, C.c_uint64, C.c_void_p, C.c_void_p]
        _lib.or_neighbour.restype = C.c_int
        _lib.or_search_round.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p,
                                         C.POINTER(_Moves), C.c_uint64, C.c_int64, C.c_int64,
                                         C.c_void_p, C.c_int32]
        _lib.or_search_round.restype = C.c_int64
        _lib.or_neighbour_explicit.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p,
                                               C.c_int32, C.POINTER(_Moves), C.c_uint64, C.c_uint64, C.c_void_p,
                                               C.c_void_p, C.c_void_p]
        _lib.or_neighbour_explicit.restype = C.c_int
        _lib.or_search_round_explicit.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p,
                                                  C.c_int32, C.POINTER(_Moves), C.c_uint64, C.c_int64, C.c_int64,
                                                  C.c_void_p, C.c_int32]
        _lib.or_search_round_explicit.restype = C.c_int64
        _lib.or_bound.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_int32]
        _lib.or_bound.restype = C.c_int64
    return _lib


class Oracle:
    """Oracle bound to one PackedInstance (paper_2510_05186_b200.packing)."""

    def __init__(self, pk):
        self.pk = pk
        self._arrs = [np.ascontiguousarray(a) for a in
                      (pk.proc_time, pk.mem_delta, pk.act_size, pk.mem_limit, pk.stage_channel)]
        self._inst = _Inst(pk.num_stages, pk.num_microbatches, pk.num_channels,
                           *[a.ctypes.data for a in self._arrs],
                           pk.comm_time, pk.offload_time, int(pk.post_validation))
        self.lib = lib()

    def run(self, orders, mask, chans=None):
        """One candidate -> dict(makespan, bubble, peak, flags, blocked, trace_code, trace_start)."""
        pk = self.pk
        orders = np.ascontiguousarray(orders, np.uint16)
        mask = np.ascontiguousarray(mask, np.uint32)
        E = 5 * pk.num_stages * pk.num_microbatches
        peak = np.zeros(pk.num_stages, np.int64)
        codes = np.zeros(E, np.uint32)
        starts = np.zeros(E, np.int32)
        r = _Res(0, 0.0, peak.ctypes.data, 0, 0, codes.ctypes.data, starts.ctypes.data, 0)
        cptr, cstride = None, 0
        if chans is not None:
            chans = np.ascontiguousarray(chans, np.uint32)
            cptr, cstride = chans.ctypes.data, chans.shape[-1]
        self.lib.or_run_order(C.byref(self._inst), orders.ctypes.data, orders.shape[-1],
                              mask.ctypes.data, cptr, cstride, C.byref(r))
        n = r.n_events
        return dict(makespan=r.makespan, bubble=r.bubble, peak=peak, flags=r.flags,
                    blocked=r.blocked, trace_code=codes[:n], trace_start=starts[:n])

    def eval_batch(self, orders, masks, chans=None, threads=0):
        pk = self.pk
        orders = np.ascontiguousarray(orders, np.uint16)
        masks = np.ascontiguousarray(masks, np.uint32)
        n = orders.shape[0]
        out = dict(makespan=np.zeros(n, np.int64), bubble=np.zeros(n, np.float64),
                   peak=np.zeros((n, pk.num_stages), np.int64), flags=np.zeros(n, np.uint32),
                   blocked=np.zeros(n, np.uint32))
        cptr, cstride = None, 0
        if chans is not None:
            chans = np.ascontiguousarray(chans, np.uint32)
            cptr, cstride = chans.ctypes.data, chans.shape[-1]
        self.lib.or_eval_batch(C.byref(self._inst), n, orders.ctypes.data, orders.shape[-1],
                               masks.ctypes.data, masks.shape[-1], cptr, cstride,
                               out["makespan"].ctypes.data, out["bubble"].ctypes.data,
                               out["peak"].ctypes.data, out["flags"].ctypes.data,
                               out["blocked"].ctypes.data, int(threads))
        return out

    def neighbour(self, inc_orders, inc_mask, seed, shift_permille, max_shift, rnd, index):
        o = np.zeros_like(np.ascontiguousarray(inc_orders, np.uint16))
        mk = np.zeros_like(np.ascontiguousarray(inc_mask, np.uint32))
        mv = _Moves(seed, shift_permille, max_shift)
        inc_o = np.ascontiguousarray(inc_orders, np.uint16)
        inc_m = np.ascontiguousarray(inc_mask, np.uint32)
        t = self.lib.or_neighbour(C.byref(self._inst), inc_o.ctypes.data, inc_o.shape[-1],
                                  inc_m.ctypes.data, C.byref(mv), rnd, index, o.ctypes.data,
                                  mk.ctypes.data)
        return t, o, mk

    def search_round(self, inc_orders, inc_mask, seed, shift_permille, max_shift, rnd, first,
                     count, threads=0, want_makespans=False):
        inc_o = np.ascontiguousarray(inc_orders, np.uint16)
        inc_m = np.ascontiguousarray(inc_mask, np.uint32)
        mv = _Moves(seed, shift_permille, max_shift)
        ms = np.zeros(count, np.int64) if want_makespans else None
        best = self.lib.or_search_round(C.byref(self._inst), inc_o.ctypes.data, inc_o.shape[-1],
                                        inc_m.ctypes.data, C.byref(mv), rnd, first, count,
                                        ms.ctypes.data if ms is not None else None, int(threads))
        return best, ms


def neighbour_explicit(orc: "Oracle", inc_orders, inc_mask, inc_chan, seed, shift_permille, max_shift, rnd, index):
    """Channel-order neighbour -> (type, orders, mask, chans)."""
    inc_o = np.ascontiguousarray(inc_orders, np.uint16)
    inc_m = np.ascontiguousarray(inc_mask, np.uint32)
    inc_c = np.ascontiguousarray(inc_chan, np.uint32)
    o, mk, ch = np.zeros_like(inc_o), np.zeros_like(inc_m), np.zeros_like(inc_c)
    mv = _Moves(seed, shift_permille, max_shift)
    t = orc.lib.or_neighbour_explicit(C.byref(orc._inst), inc_o.ctypes.data, inc_o.shape[-1], inc_m.ctypes.data,
                                      inc_c.ctypes.data, inc_c.shape[-1], C.byref(mv), rnd, index, o.ctypes.data,
                                      mk.ctypes.data, ch.ctypes.data)
    return t, o, mk, ch


def search_round_explicit(orc: "Oracle", inc_orders, inc_mask, inc_chan, seed, shift_permille, max_shift, rnd,
                          first, count, threads=0, want_makespans=False):
    inc_o = np.ascontiguousarray(inc_orders, np.uint16)
    inc_m = np.ascontiguousarray(inc_mask, np.uint32)
    inc_c = np.ascontiguousarray(inc_chan, np.uint32)
    mv = _Moves(seed, shift_permille, max_shift)
    ms = np.zeros(count, np.int64) if want_makespans else None
    best = orc.lib.or_search_round_explicit(C.byref(orc._inst), inc_o.ctypes.data, inc_o.shape[-1], inc_m.ctypes.data,
                                            inc_c.ctypes.data, inc_c.shape[-1], C.byref(mv), rnd, first, count,
                                            ms.ctypes.data if ms is not None else None, int(threads))
    return best, ms


def bound(orc: "Oracle", t, sfree, start, post) -> int:
    """B&B node lower bound (solver.py:321-383); start [P][m][3] int64 with -1 = uncommitted."""
    sf = np.ascontiguousarray(sfree, np.int64)
    st = np.ascontiguousarray(start, np.int64)
    return int(orc.lib.or_bound(C.byref(orc._inst), int(t), sf.ctypes.data, st.ctypes.data, int(bool(post))))


def philox4x32_10(ctr, key):
    c = np.array(ctr, np.uint32)
    k = np.array(key, np.uint32)
    out = np.zeros(4, np.uint32)
    lib().or_philox4x32_10(c.ctypes.data, k.ctypes.data, out.ctypes.data)
    return [int(x) for x in out]
