"""CPU-side checks of the boundary: the C-ABI library loads and exports every declared symbol."""

import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    text = (ROOT / "include" / "pipesched_b200.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(ps_\w+)\s*\(", text, re.M)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for name in ("ps_instance_create", "ps_instance_destroy", "ps_eval_batch", "ps_eval_batch_host",
                 "ps_search_round", "ps_last_error"):
        assert name in syms


def test_library_exports_every_declared_symbol():
    from paper_2510_05186_b200 import build
    from paper_2510_05186_b200 import _native
    build.build()
    lib = _native.load_library()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert set(_native.EXPORTS) == set(declared_symbols())
    assert b"sm_100a" in lib.ps_version()


def test_library_rejects_bad_instances_without_a_gpu():
    """Argument validation runs before any CUDA call, so it is testable on CPU."""
    import ctypes as C
    import numpy as np
    from paper_2510_05186_b200 import _native
    lib = _native.load_library()
    P, m = 2, 2
    proc = np.ones((P, m, 3), np.int64)
    delta = np.tile(np.array([2, -1, -1], np.int64), (P, m, 1))
    act = np.full((P, m), 2, np.int64)
    limit = np.full(P, 4, np.int64)
    chan = np.arange(P, dtype=np.int32)
    delta[1, 1, 1] = -2          # F+B+W != 0
    d = _native.InstanceDesc(P, m, proc.ctypes.data, delta.ctypes.data, act.ctypes.data,
                             limit.ctypes.data, chan.ctypes.data, P, 1, 1, 0)
    h = C.c_void_p()
    assert lib.ps_instance_create(C.byref(d), 0, C.byref(h)) == -1
    assert b"mem_delta sum nonzero" in lib.ps_last_error()
    d.num_stages = 33
    assert lib.ps_instance_create(C.byref(d), 0, C.byref(h)) == -2


def test_product_path_fails_loudly_without_cuda(monkeypatch):
    import torch
    from paper_2510_05186_b200 import _native, make_uniform_instance, run_order
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    inst = make_uniform_instance(1, 1, 1, 1, 1, 0, 1, 2, 4)
    with pytest.raises(_native.NativeUnavailable):
        run_order(inst, {1: tuple(inst.stage_ops(1))}, frozenset())


def test_cache_records_parse_in_the_reference_format(tmp_path):
    from paper_2510_05186_b200.cache import load_entries
    rec = ('{"key": {"P": 1, "m": 1, "ratios": [1.0, 1.0, 0.0, 1.0, 2.0], "post_validation": false}, '
           '"order": {"stages": [[[1, "F"], [1, "B"], [1, "W"]]], "offloaded": [[1, 1]], '
           '"channels": [[[1, 1, "F", "O"], [1, 1, "F", "R"]]]}, "makespan_ratio": 3.0}')
    p = tmp_path / "cache.jsonl"
    p.write_text(rec + "\n")
    (e,) = load_entries(p)
    assert e.num_stages == 1 and len(e.stage_orders[0]) == 3 and len(e.channel_orders[0]) == 2
    assert e.channel_orders[0][1][1].value == "reload"
