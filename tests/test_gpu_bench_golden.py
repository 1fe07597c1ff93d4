"""The bench's own neighbours at the BASELINE shapes vs the UNMODIFIED reference.

tests/golden/make_bench_golden.py ran the reference ``pipesched.run_order`` (+ makespan,
memory_trace(STRICT), the cli.py:156 bubble) on neighbours of fixed search rounds: config 3
(8 x 64) early (AdaOffload incumbent, round 5) and late (the search's round-320 incumbent,
round 320), config 4 (16 x 128) and config 5 (32 x 256).  Here, for every recorded neighbour:

* the device move decoder (``ps_materialize_moves``) produces exactly the recorded neighbour
  (the recorded diff against the incumbent);
* ``ps_eval_batch`` (no base, full trace) gives the reference's makespan, bubble ``repr``,
  peaks, ``OrderInfeasible.stages`` and commit-ordered trace (SHA-256, and event by event
  where the fixture holds the full trace);
* the search round as the bench runs it (``ps_search_round`` with the recorded base, prefix and
  suffix sharing) gives the reference's makespan for the same (round, index);
* ``ps_eval_batch_host`` with the base (the bench's e2e path) gives the same answers.
"""

import ctypes as C
import gzip
import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

from _golden import split_trace

pytestmark = pytest.mark.gpu

GOLDEN = Path(__file__).resolve().parent / "golden"
FILES = sorted(GOLDEN.glob("bench_config*.json.gz"))


def _digest(comp, tr):
    h = hashlib.sha256()
    for e in comp:
        h.update(("C %d %d %d %d\n" % tuple(e)).encode())
    for e in tr:
        h.update(("T %d %d %d %d\n" % tuple(e)).encode())
    return h.hexdigest()


def _load(path):
    with gzip.open(path, "rt") as fh:
        return json.load(fh)


def _structure_arrays(pk, orders_codes, offloaded):
    o = np.zeros((pk.num_stages, pk.order_stride), np.uint16)
    for i, row in enumerate(orders_codes):
        o[i, :len(row)] = row
    mk = np.zeros(pk.mask_words, np.uint32)
    for i, j in offloaded:
        b = (i - 1) * pk.num_microbatches + (j - 1)
        mk[b >> 5] |= np.uint32(1 << (b & 31))
    return o, mk


def _check_answer(case, flags, makespan, bubble, peak, blocked, trace, P):
    if "infeasible" in case:
        assert flags == 2, (case["index"], flags)
        assert [i + 1 for i in range(P) if (blocked >> i) & 1] == case["infeasible"]
        return
    assert flags == 1, (case["index"], flags)
    assert makespan == case["makespan"]
    assert repr(float(bubble)) == case["bubble"]
    assert [int(x) for x in peak] == case["peak"]
    if trace is not None:
        comp, tr = trace
        assert (len(comp), len(tr)) == (case["n_compute"], case["n_transfers"])
        if "compute" in case:
            assert comp == case["compute"] and tr == case["transfers"]
        assert _digest(comp, tr) == case["trace_sha256"]


@pytest.mark.skipif(not FILES, reason="no bench-shape fixtures")
@pytest.mark.parametrize("path", FILES, ids=[p.name for p in FILES])
def test_bench_neighbours_match_the_reference(cuda_ok, path):
    import torch
    from paper_2510_05186_b200 import _native as N
    from paper_2510_05186_b200.engine import Base, DeviceInstance
    from paper_2510_05186_b200.instance import instance_from_dict
    from paper_2510_05186_b200.packing import pack_instance

    doc = _load(path)
    inst = instance_from_dict(doc["instance"])
    pk = pack_instance(inst)
    di = DeviceInstance(inst, packed=pk)
    P, L = pk.num_stages, 3 * pk.num_microbatches
    moves = N.MoveParams(doc["seed"], doc["moves"]["shift_permille"], doc["moves"]["max_shift"])
    stream = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    checked = 0
    for st in doc["sets"]:
        inc = st["incumbent"]
        o, mk = _structure_arrays(pk, inc["orders"], inc["offloaded"])
        d_o = torch.from_numpy(o.view(np.int16)).cuda()
        d_m = torch.from_numpy(mk.view(np.int32)).cuda()
        cases = st["neighbours"]
        n = len(cases)
        # 1. the device move decoder reproduces every recorded neighbour
        orders = torch.empty((n, P, pk.order_stride), dtype=torch.int16, device="cuda")
        masks = torch.empty((n, pk.mask_words), dtype=torch.int32, device="cuda")
        for k, case in enumerate(cases):
            desc = N.SearchDesc(d_o.data_ptr(), d_m.data_ptr(), st["round"], case["index"], 1, moves)
            N.check(di.lib.ps_materialize_moves(di.handle, C.byref(desc), C.c_void_p(orders[k].data_ptr()),
                                                C.c_void_p(masks[k].data_ptr()), stream))
        h_orders = orders.cpu().numpy().view(np.uint16)
        h_masks = masks.cpu().numpy().view(np.uint32)
        for k, case in enumerate(cases):
            want = o.copy()
            for i, p, c in case["order_diff"]:
                want[i, p] = c
            assert (h_orders[k, :, :L] == want[:, :L]).all(), case["index"]
            wm = mk.copy()
            for i, j in case["offload_flips"]:
                b = (i - 1) * pk.num_microbatches + (j - 1)
                wm[b >> 5] ^= np.uint32(1 << (b & 31))
            assert (h_masks[k] == wm).all(), case["index"]
        # 2. the evaluator, no base, full trace: every reference output
        res = di.evaluate(orders, masks, peak=True, trace=True)
        r = {k: (v.cpu().numpy() if v is not None else None) for k, v in vars(res).items()}
        for k, case in enumerate(cases):
            ev = None
            if "infeasible" not in case:
                cnt = case["n_compute"] + case["n_transfers"]
                ev = split_trace(r["trace_code"][k][:cnt], r["trace_start"][k][:cnt])
            _check_answer(case, int(r["flags"][k]), int(r["makespan"][k]), r["bubble"][k], r["peak"][k],
                          int(r["blocked"][k]) & 0xFFFFFFFF, ev, P)
            checked += 1
        # the incumbent itself
        one = di.evaluate(d_o.view(1, P, -1), d_m.view(1, -1), peak=True, trace=True)
        cnt = inc["n_compute"] + inc["n_transfers"]
        ev = split_trace(one.trace_code[0].cpu().numpy()[:cnt], one.trace_start[0].cpu().numpy()[:cnt])
        _check_answer(dict(inc, index=-1), int(one.flags[0]), int(one.makespan[0]), one.bubble[0].item(),
                      one.peak[0].cpu().numpy(), 0, ev, P)
        # 3. the search round as the bench runs it: recorded base, prefix/suffix sharing
        base = Base(di)
        base.record(d_o, d_m)
        span = {c["index"]: (c["makespan"] if "makespan" in c else -1) for c in cases}
        lo, hi = min(span), max(span) + 1
        ms = torch.empty(hi - lo, dtype=torch.int64, device="cuda")
        best = torch.full((1,), N.BEST_NONE, dtype=torch.int64, device="cuda")
        desc = N.SearchDesc(d_o.data_ptr(), d_m.data_ptr(), st["round"], lo, hi - lo, moves, None, base.handle, 0)
        N.check(di.lib.ps_search_round(di.handle, C.byref(desc), C.c_void_p(best.data_ptr()),
                                       C.c_void_p(ms.data_ptr()), stream))
        got = ms.cpu().numpy()
        for idx, want in span.items():
            assert int(got[idx - lo]) == want, (st["name"], idx)
        # 4. the e2e path: host buffers, the base, uint8 codes where they fit
        u8 = 4 * pk.num_microbatches <= 256
        ho = h_orders.astype(np.uint8) if u8 else h_orders.copy()
        out = di.evaluate_host(ho, h_masks.copy(), peak=True, base=base)
        for k, case in enumerate(cases):
            _check_answer(case, int(out.flags[k]), int(out.makespan[k]), out.bubble[k], out.peak[k],
                          int(out.blocked[k]) & 0xFFFFFFFF, None, P)
    assert checked == sum(len(st["neighbours"]) for st in doc["sets"])
