"""The int64 ledger variant (stage usages that do not fit int32 after gcd reduction): search
rounds, prefix/suffix sharing against a recorded base, re-recording and a whole search, each
against the CPU restatement or the plain simulation — the same bar the int32 variant meets in
test_gpu_search.py."""

import numpy as np
import pytest

from test_gpu_search import MAXSHIFT, PERMILLE, SEED, _base_tables, _eval_both

pytestmark = pytest.mark.gpu


def _odd_bytes_config3():
    """Config 3 with per-stage activations made odd and distinct: the byte gcd is 1, so one
    stage's usage (4 activations of limit + 64 deltas of 2.28 GB) needs 64-bit ledger words."""
    from paper_2510_05186_b200 import workloads as W
    from paper_2510_05186_b200.instance import _per_stage_instance
    P, m = 8, 64
    rows, limits = [], []
    for i in range(1, P + 1):
        extra = W.LLAMA7B_HEAD if i == P else 0
        act = W.LLAMA7B_ACT + 2 * i + 1
        rows.append((W.LLAMA7B_TF + extra, W.LLAMA7B_TB + extra, W.LLAMA7B_TW + extra, act))
        limits.append(4 * act)
    return _per_stage_instance(P, m, rows, W.LLAMA7B_COMM, W.LLAMA7B_OFFLOAD, limits, None, False)


@pytest.fixture(scope="module")
def setup64():
    from paper_2510_05186_b200.heuristics import best_feasible
    from paper_2510_05186_b200.listsched import stage_order_of
    inst = _odd_bytes_config3()
    s, _ = best_feasible(inst)
    orders = {i: stage_order_of(s, i) for i in range(1, inst.num_stages + 1)}
    return inst, orders, s.offloaded


def _search(setup64, n, **kw):
    from paper_2510_05186_b200.search import LocalSearch, SearchConfig
    inst, orders, off = setup64
    return LocalSearch(inst, orders, off, SearchConfig(seed=SEED, neighbours=n, shift_permille=PERMILLE,
                                                       max_shift=MAXSHIFT, **kw))


def test_instance_takes_the_int64_ledger(cuda_ok, setup64):
    ls = _search(setup64, 64)
    assert ls.di.info.value_bits == 64 and ls.di.info.memory_unit == 1


def test_search_round_matches_cpu_round(cuda_ok, setup64):
    import torch
    from oracle.oracle import Oracle
    n = 2048
    ls = _search(setup64, n)
    ms = torch.empty(n, dtype=torch.int64, device="cuda")
    ls.launch_round(ms)
    torch.cuda.synchronize()
    orc = Oracle(ls.di.packed)
    best, want = orc.search_round(ls.inc_orders.cpu().numpy().view(np.uint16),
                                  ls.inc_mask.cpu().numpy().view(np.uint32), SEED, PERMILLE, MAXSHIFT,
                                  0, 0, n, want_makespans=True)
    assert (ms.cpu().numpy() == want).all()
    assert int(ls.best_key.item()) == best


def test_prefix_sharing_and_rerecording_are_exact(cuda_ok, setup64):
    import torch
    from paper_2510_05186_b200.engine import Base
    n = 1024
    ls = _search(setup64, n, share_prefix=True)
    o, mk = ls.materialize(0, n, 0)
    r = _eval_both(ls.di, o, mk, ls.base)
    flags, spans = r.flags.cpu().numpy(), r.makespan.cpu().numpy()
    assert (flags & 1).any() and (flags & 2).any()
    h_m = mk.cpu().numpy()
    for ho in (o.cpu().numpy(), o.cpu().numpy().astype(np.uint8)):
        host = ls.di.evaluate_host(ho, h_m, peak=True, base=ls.base)
        assert (host.flags == flags).all() and (host.makespan == spans).all()
        assert (host.peak == r.peak.cpu().numpy()).all()
    pk = ls.di.packed
    P, m, MW = pk.num_stages, pk.num_microbatches, (pk.num_microbatches + 31) // 32
    feas = np.nonzero(flags & 1)[0]
    order = feas[np.argsort(spans[feas], kind="stable")]
    picks = [int(order[0]), int(order[-1]), int(np.nonzero(flags & 2)[0][0])]
    for idx in picks:
        fresh, again = Base(ls.di), Base(ls.di)
        fresh.record(o[idx], mk[idx])
        again.record(ls.inc_orders, ls.inc_mask)
        again.record(o[idx], mk[idx])
        torch.cuda.synchronize()
        a, b = _base_tables(fresh, P, m, MW, vw=2), _base_tables(again, P, m, MW, vw=2)
        assert a[:4] == b[:4], idx
        assert len(a[4]) == len(b[4]), idx
        for c, (ca, cb) in enumerate(zip(a[4], b[4])):
            for part, name in enumerate(("state words", "lane scalars", "windows", "event steps")):
                assert ca[part] == cb[part], (idx, c, name)
        _eval_both(ls.di, o, mk, again)


def test_identical_best_schedule_for_equal_budgets(cuda_ok, setup64):
    from oracle.oracle import Oracle
    from paper_2510_05186_b200 import makespan, validate
    inst = setup64[0]
    n, rounds = 1024, 5
    ls = _search(setup64, n)
    orc = Oracle(ls.di.packed)
    inc_o = ls.inc_orders.cpu().numpy().view(np.uint16)
    inc_m = ls.inc_mask.cpu().numpy().view(np.uint32)
    span = ls.makespan
    trail = []
    for rnd in range(rounds):
        best, _ = orc.search_round(inc_o, inc_m, SEED, PERMILLE, MAXSHIFT, rnd, 0, n)
        if best != (1 << 63) - 1 and (best >> 32) < span:
            span = best >> 32
            _, inc_o, inc_m = orc.neighbour(inc_o, inc_m, SEED, PERMILLE, MAXSHIFT, rnd, best & 0xFFFFFFFF)
            trail.append((rnd, span))
    res = ls.run(rounds=rounds)
    assert trail and [(i.round, i.makespan) for i in res.improvements] == trail
    assert validate(res.schedule, inst).ok and makespan(res.schedule, inst) == span
