"""ctypes binding of the C ABI in ``include/pipesched_b200.h``.

The shared library is built in-tree (``build.py``) and loaded from
``_lib/libpipesched_b200.so``.  There is no CPU fallback: if the library is
missing or no CUDA device is visible, every entry point raises
``NativeUnavailable`` with the reason.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(os.environ.get("PS_LIBRARY") or Path(__file__).resolve().parent / "_lib" / "libpipesched_b200.so")

PS_OK = 0
FLAG_FEASIBLE = 1
FLAG_DEADLOCK = 2
FLAG_MALFORMED = 4
FLAG_RANGE = 16          # an event time reached 2^29 quanta (include/pipesched_b200.h)
MAX_STAGES = 32
MAX_MICROBATCHES = 4096
BEST_NONE = (1 << 63) - 1
BASE_CHECKPOINTS, BASE_CSTEP, BASE_FSTEP, BASE_INFO, BASE_RESULT, BASE_LAYOUT = range(6)   # ps_base_read


class NativeUnavailable(RuntimeError):
    """The CUDA extension is missing or cannot run here."""


class NativeError(RuntimeError):
    """A C-ABI call returned an error code."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"pipesched_b200 error {code}: {msg}")
        self.code = code


class InstanceDesc(C.Structure):
    _fields_ = [
        ("num_stages", C.c_int32),
        ("num_microbatches", C.c_int32),
        ("proc_time", C.c_void_p),
        ("mem_delta", C.c_void_p),
        ("act_size", C.c_void_p),
        ("mem_limit", C.c_void_p),
        ("stage_channel", C.c_void_p),
        ("num_channels", C.c_int32),
        ("comm_time", C.c_int64),
        ("offload_time", C.c_int64),
        ("post_validation", C.c_int32),
    ]


class InstanceInfo(C.Structure):
    _fields_ = [
        ("num_stages", C.c_int32),
        ("num_microbatches", C.c_int32),
        ("order_stride", C.c_int32),
        ("mask_words", C.c_int32),
        ("max_events", C.c_int32),
        ("value_bits", C.c_int32),
        ("memory_unit", C.c_int64),
        ("busy_time", C.c_int64),
        ("lanes_per_candidate", C.c_int32),
        ("device", C.c_int32),
    ]


class CandBatch(C.Structure):
    _fields_ = [
        ("num_candidates", C.c_int64),
        ("stage_orders", C.c_void_p),
        ("offload_mask", C.c_void_p),
        ("channel_orders", C.c_void_p),
        ("chan_stride", C.c_int32),
        ("base", C.c_void_p),
        ("order_bytes", C.c_int32),
    ]


class DeltaBatch(C.Structure):
    _fields_ = [
        ("num_candidates", C.c_int64),
        ("ref_orders", C.c_void_p),
        ("ref_mask", C.c_void_p),
        ("diff_offset", C.c_void_p),
        ("diffs", C.c_void_p),
        ("flip_offset", C.c_void_p),
        ("flips", C.c_void_p),
        ("base", C.c_void_p),
    ]


class ResultBatch(C.Structure):
    _fields_ = [
        ("makespan", C.c_void_p),
        ("bubble", C.c_void_p),
        ("peak", C.c_void_p),
        ("flags", C.c_void_p),
        ("blocked", C.c_void_p),
        ("trace_code", C.c_void_p),
        ("trace_start", C.c_void_p),
        ("trace_stride", C.c_int32),
        ("events_total", C.c_void_p),
    ]


class MoveParams(C.Structure):
    _fields_ = [
        ("seed", C.c_uint64),
        ("shift_permille", C.c_uint32),
        ("max_shift", C.c_uint32),
    ]


class SearchDesc(C.Structure):
    _fields_ = [
        ("inc_orders", C.c_void_p),
        ("inc_mask", C.c_void_p),
        ("round", C.c_uint64),
        ("first_index", C.c_int64),
        ("count", C.c_int64),
        ("moves", MoveParams),
        ("events_total", C.c_void_p),
        ("base", C.c_void_p),
        ("dedup", C.c_int32),
        ("cutoff", C.c_int64),
    ]


class BoundBatch(C.Structure):
    _fields_ = [
        ("num_nodes", C.c_int64),
        ("clock", C.c_void_p),
        ("stage_free", C.c_void_p),
        ("comp_start", C.c_void_p),
    ]


EXPORTS = {
    "ps_version": (C.c_char_p, []),
    "ps_last_error": (C.c_char_p, []),
    "ps_instance_create": (C.c_int, [C.POINTER(InstanceDesc), C.c_int, C.POINTER(C.c_void_p)]),
    "ps_instance_destroy": (C.c_int, [C.c_void_p]),
    "ps_instance_get_info": (C.c_int, [C.c_void_p, C.POINTER(InstanceInfo)]),
    "ps_eval_batch": (C.c_int, [C.c_void_p, C.POINTER(CandBatch), C.POINTER(ResultBatch), C.c_void_p]),
    "ps_eval_batch_host": (C.c_int, [C.c_void_p, C.POINTER(CandBatch), C.POINTER(ResultBatch), C.c_void_p]),
    "ps_search_round": (C.c_int, [C.c_void_p, C.POINTER(SearchDesc), C.c_void_p, C.c_void_p, C.c_void_p]),
    "ps_search_round_sharded": (C.c_int, [C.c_void_p, C.POINTER(SearchDesc), C.c_void_p, C.c_void_p,
                                          C.c_void_p, C.c_void_p]),
    "ps_eval_batch_host_delta": (C.c_int, [C.c_void_p, C.POINTER(DeltaBatch), C.POINTER(ResultBatch), C.c_void_p]),
    "ps_search_round_explicit": (C.c_int, [C.c_void_p, C.POINTER(SearchDesc), C.c_void_p, C.c_int32,
                                           C.c_void_p, C.c_void_p, C.c_void_p]),
    "ps_materialize_moves_explicit": (C.c_int, [C.c_void_p, C.POINTER(SearchDesc), C.c_void_p, C.c_int32,
                                                C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "ps_apply_move_explicit": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.POINTER(MoveParams),
                                         C.c_uint64, C.c_uint64, C.c_void_p]),
    "ps_materialize_moves": (C.c_int, [C.c_void_p, C.POINTER(SearchDesc), C.c_void_p, C.c_void_p, C.c_void_p]),
    "ps_apply_move": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(MoveParams),
                                C.c_uint64, C.c_uint64, C.c_void_p]),
    "ps_int32_probe": (C.c_int, [C.c_int64, C.c_void_p, C.c_void_p]),
    "ps_base_create": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p)]),
    "ps_base_destroy": (C.c_int, [C.c_void_p]),
    "ps_base_record": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "ps_base_record_explicit": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p]),
    "ps_base_read": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.POINTER(C.c_size_t)]),
    "ps_bound_batch_eval": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
}

_lib = None


def load_library(path: os.PathLike | None = None) -> C.CDLL:
    """Load (once) and type the C-ABI library.  Does not need a GPU."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path else LIB_PATH
    if not p.exists():
        raise NativeUnavailable(
            f"{p} is missing: build it with `python -m paper_2510_05186_b200.build` "
            "(there is no CPU fallback for the evaluator)")
    lib = C.CDLL(str(p))
    for name, (res, args) in EXPORTS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _lib = lib
    return lib


def check(rc: int) -> None:
    if rc != PS_OK:
        raise NativeError(rc, load_library().ps_last_error().decode())


def require_cuda():
    """The evaluator only runs on a CUDA device; fail loudly otherwise."""
    import torch
    if not torch.cuda.is_available():
        raise NativeUnavailable("no CUDA device is visible: the B200 evaluator has no CPU fallback")
    load_library()
