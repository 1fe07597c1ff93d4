"""Whole searches on random non-uniform instances (per-(stage, microbatch) times and bytes, shared
transfer channels, post-validation, zero comm/offload times): every 4th round, every neighbour's
makespan with prefix/suffix sharing against the recorded incumbent equals the CPU restatement's
(oracle/ps_oracle.c), and the rounds in between adopt the same moves as the restatement would.
The BASELINE configs are uniform across microbatches and give each stage its own channel; these
instances reach the convergence rules through the other cases."""

import random

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def random_tables(rng: random.Random, P: int, m: int, big: bool = False) -> dict:
    """A reference-format instance dict (instance.py's JSON codec) with independent values per
    (stage, microbatch); the memory limit lies between one activation and ~1/3 of them all.
    `big`: byte counts near 2^34 with odd gcd structure (the 64-bit device ledger)."""
    proc, mem, act = [], [], []
    for _ in range(P):
        pr, me, ac = [], [], []
        for _ in range(m):
            pr.append([rng.randint(1, 9), rng.randint(1, 9), rng.randint(1, 9)])
            a = rng.randint(2, 12) if not big else rng.randint(2**33, 2**34) * 2 + 1
            d_b = -((a + 1) // 2) - (rng.randint(0, 1) if a > 3 else 0)
            me.append([a, d_b, -a - d_b])
            ac.append([rng.choice([0, a, a, max(1, a // 2)]), 0, 0])
        proc.append(pr)
        mem.append(me)
        act.append(ac)
    limits = []
    for i in range(P):
        lo = 2 * max(r[0] for r in mem[i])
        limits.append(rng.randint(lo, max(lo, sum(r[0] for r in mem[i]) // 3 + 13)))
    d = {"num_stages": P, "num_microbatches": m, "proc_times": proc, "comm_time": rng.randint(0, 3),
         "offload_time": rng.randint(0, 5), "mem_deltas": mem, "act_sizes": act, "mem_limits": limits,
         "post_validation": rng.random() < 0.3}
    if P >= 2 and rng.random() < 0.5:
        stages = list(range(1, P + 1))
        rng.shuffle(stages)
        cuts = sorted(rng.sample(range(1, P), min(P - 1, rng.randint(1, 3))))
        d["topology_groups"] = [sorted(stages[a:b]) for a, b in zip([0] + cuts, cuts + [P])]
    return d


def soak_case(seed: int, stages=(2, 12), microbatches=(4, 40), n=2048, rounds=24, big=False):
    """One random instance's search; returns (P, m, neighbours checked) or None (no warm start)."""
    import torch
    from oracle.oracle import Oracle
    from paper_2510_05186_b200 import InfeasibleSchedule, NoFeasibleSchedule, instance_from_dict
    from paper_2510_05186_b200.heuristics import best_feasible
    from paper_2510_05186_b200.listsched import stage_order_of
    from paper_2510_05186_b200.search import LocalSearch, SearchConfig
    rng = random.Random(1000 + seed)
    for _ in range(20):
        P, m = rng.randint(*stages), rng.randint(*microbatches)
        inst = instance_from_dict(random_tables(rng, P, m, big))
        try:
            s0, _ = best_feasible(inst)
        except (InfeasibleSchedule, NoFeasibleSchedule):
            continue
        break
    else:
        return None
    cfg = SearchConfig(seed=seed, neighbours=n, shift_permille=600, max_shift=6)
    ls = LocalSearch(inst, {i: stage_order_of(s0, i) for i in range(1, P + 1)}, s0.offloaded, cfg)
    orc = Oracle(ls.di.packed)
    ms = torch.empty(n, dtype=torch.int64, device="cuda")
    checked = 0
    for rnd in range(rounds):
        inc_o = ls.inc_orders.cpu().numpy().view(np.uint16).copy()
        inc_m = ls.inc_mask.cpu().numpy().view(np.uint32).copy()
        best, want = orc.search_round(inc_o, inc_m, cfg.seed, cfg.shift_permille, cfg.max_shift,
                                      ls.round, 0, n, want_makespans=rnd % 4 == 0)
        if rnd % 4 == 0:
            ls.launch_round(ms)
            torch.cuda.synchronize()
            got = ms.cpu().numpy()
            bad = np.flatnonzero(got != want)
            assert bad.size == 0, (seed, rnd, P, m, bad[:8], got[bad[:8]], want[bad[:8]])
            checked += n
        else:
            ls.launch_round()
        assert int(ls.best_key.item()) == best, (seed, rnd)
        ls.finish_round()
    return P, m, checked


@pytest.mark.parametrize("seed", range(12))
def test_search_on_random_instances_matches_the_cpu_restatement(cuda_ok, seed):
    r = soak_case(seed)
    if r is None:
        pytest.skip("no feasible warm start drawn")
    assert r[2] == 2048 * 6


@pytest.mark.parametrize("seed", range(4))
def test_search_on_random_wide_instances_with_a_64_bit_ledger(cuda_ok, seed):
    r = soak_case(100 + seed, stages=(12, 32), microbatches=(16, 96), n=512, rounds=8, big=True)
    if r is None:
        pytest.skip("no feasible warm start drawn")
    assert r[2] == 512 * 2


def _random_start(seed, stages, microbatches, big=False):
    from paper_2510_05186_b200 import InfeasibleSchedule, NoFeasibleSchedule, instance_from_dict
    from paper_2510_05186_b200.heuristics import best_feasible
    rng = random.Random(1000 + seed)
    for _ in range(20):
        P, m = rng.randint(*stages), rng.randint(*microbatches)
        inst = instance_from_dict(random_tables(rng, P, m, big))
        try:
            s0, _ = best_feasible(inst)
        except (InfeasibleSchedule, NoFeasibleSchedule):
            continue
        return inst, s0
    return None


def soak_channel_case(seed: int, stages=(2, 12), microbatches=(4, 40), n=2048, rounds=16, big=False):
    """Channel-order search (explicit mode) with the incumbent recorded in explicit
    mode, on one random instance: every 4th round every neighbour's makespan against
    or_search_round_explicit, every round's best key, across re-recordings."""
    import torch
    from oracle.oracle import Oracle, search_round_explicit
    from paper_2510_05186_b200.search import ChannelSearch, SearchConfig
    start = _random_start(seed, stages, microbatches, big)
    if start is None:
        return None
    inst, s0 = start
    cfg = SearchConfig(seed=seed, neighbours=n, shift_permille=400, max_shift=6)
    cs = ChannelSearch.from_schedule(inst, s0, cfg)
    orc = Oracle(cs.di.packed)
    ms = torch.empty(n, dtype=torch.int64, device="cuda")
    checked = 0
    for rnd in range(rounds):
        inc = [t.cpu().numpy().view(dt).copy() for t, dt in
               ((cs.inc_orders, np.uint16), (cs.inc_mask, np.uint32), (cs.inc_chan, np.uint32))]
        best, want = search_round_explicit(orc, *inc, cfg.seed, cfg.shift_permille, cfg.max_shift, cs.round, 0, n,
                                           want_makespans=rnd % 4 == 0)
        if rnd % 4 == 0:
            cs.launch_round(ms)
            torch.cuda.synchronize()
            got = ms.cpu().numpy()
            bad = np.flatnonzero(got != want)
            assert bad.size == 0, (seed, rnd, inst.num_stages, inst.num_microbatches, bad[:8], got[bad[:8]],
                                   want[bad[:8]])
            checked += n
        cs.step()
        assert int(cs.best_key.item()) == best, (seed, rnd)
    return inst.num_stages, inst.num_microbatches, checked


def soak_batch_case(seed: int, stages=(2, 12), microbatches=(4, 40), n=2048, big=False):
    """The batch entry points on one random instance's search neighbours (materialised): device rows
    with and without a recorded base, and the delta-encoded host batch, each against the oracle's
    makespan, flags, peaks and bubble."""
    import torch
    from oracle.oracle import Oracle
    from paper_2510_05186_b200.engine import Base
    from paper_2510_05186_b200.listsched import stage_order_of
    from paper_2510_05186_b200.packing import delta_encode
    from paper_2510_05186_b200.search import LocalSearch, SearchConfig
    start = _random_start(seed, stages, microbatches, big)
    if start is None:
        return None
    inst, s0 = start
    P = inst.num_stages
    ls = LocalSearch(inst, {i: stage_order_of(s0, i) for i in range(1, P + 1)}, s0.offloaded,
                     SearchConfig(seed=seed, neighbours=n, shift_permille=600, max_shift=6))
    o, mk = ls.materialize(0, n, 3)
    # a third of the batch gets a second move (rebuilt in HBM by the delta path)
    o2, mk2 = ls.materialize(0, n, 4)
    on, mkn = o.cpu().numpy().view(np.uint16).copy(), mk.cpu().numpy().view(np.uint32).copy()
    o2n, mk2n = o2.cpu().numpy().view(np.uint16), mk2.cpu().numpy().view(np.uint32)
    inc_o = ls.inc_orders.cpu().numpy().view(np.uint16)
    inc_m = ls.inc_mask.cpu().numpy().view(np.uint32)
    for c in range(0, n, 3):
        st = np.flatnonzero((o2n[c] != inc_o).any(axis=1))
        if st.size and not (on[c, st[0]] != inc_o[st[0]]).any():
            on[c, st[0]] = o2n[c, st[0]]
        mkn[c] ^= mk2n[c] ^ inc_m
    want = Oracle(ls.di.packed).eval_batch(on, mkn)
    ok = want["flags"] == 1
    base = Base(ls.di)
    base.record(ls.inc_orders, ls.inc_mask)
    dev_o = torch.from_numpy(on.view(np.int16)).cuda()
    dev_m = torch.from_numpy(mkn.view(np.int32)).cuda()
    outs = {"rows": ls.di.evaluate(dev_o, dev_m, peak=True),
            "rows+base": ls.di.evaluate(dev_o, dev_m, peak=True, base=base)}
    torch.cuda.synchronize()
    outs = {k: {f: getattr(r, f).cpu().numpy() for f in ("flags", "makespan", "peak", "bubble")}
            for k, r in outs.items()}
    d = delta_encode(inc_o, inc_m, on, mkn)
    r = ls.di.evaluate_host_delta(inc_o, inc_m, *d, peak=True, base=base)
    outs["delta"] = {f: np.asarray(getattr(r, f)) for f in ("flags", "makespan", "peak", "bubble")}
    for k, g in outs.items():
        assert (g["flags"] == want["flags"]).all(), (seed, k)
        assert (g["makespan"] == want["makespan"]).all(), (seed, k)
        assert (g["peak"][ok] == want["peak"][ok]).all(), (seed, k)
        assert (g["bubble"][ok] == want["bubble"][ok]).all(), (seed, k)
    return P, inst.num_microbatches, n * len(outs)


@pytest.mark.parametrize("seed", range(8))
def test_channel_search_on_random_instances_matches_the_cpu_restatement(cuda_ok, seed):
    r = soak_channel_case(200 + seed)
    if r is None:
        pytest.skip("no feasible warm start drawn")
    assert r[2] == 2048 * 4


@pytest.mark.parametrize("seed", range(8))
def test_batch_paths_on_random_instances_match_the_oracle(cuda_ok, seed):
    r = soak_batch_case(300 + seed, big=seed % 2 == 1)
    if r is None:
        pytest.skip("no feasible warm start drawn")
    assert r[2] == 2048 * 3


def soak_ils_case(seed: int, stages=(2, 10), microbatches=(4, 24), n=512, kicks=3, kick_moves=4, big=False):
    """Iterated local search (descents, kicks from the best) on one random instance
    against the CPU restatement (tests/_search_cpu.py): the same improvement trail, round and kick
    counts and best structure."""
    from _search_cpu import cpu_search
    from oracle.oracle import Oracle
    from paper_2510_05186_b200.listsched import stage_order_of
    from paper_2510_05186_b200.search import LocalSearch, SearchConfig
    start = _random_start(seed, stages, microbatches, big)
    if start is None:
        return None
    inst, s0 = start
    P = inst.num_stages
    cfg = SearchConfig(seed=seed, neighbours=n, shift_permille=600, max_shift=6, kick_moves=kick_moves)
    ls = LocalSearch(inst, {i: stage_order_of(s0, i) for i in range(1, P + 1)}, s0.offloaded, cfg)
    want = cpu_search(Oracle(ls.di.packed), ls.inc_orders.cpu().numpy().view(np.uint16),
                      ls.inc_mask.cpu().numpy().view(np.uint32), cfg.seed, cfg.shift_permille, cfg.max_shift, n,
                      kick_moves=kick_moves, kicks=kicks)
    res = ls.run(kicks=kicks)
    assert [(i.round, i.makespan, i.index) for i in res.improvements] == want["trail"], seed
    assert (ls.round, ls.kicks) == (want["rounds"], want["kicks"]), seed
    assert res.makespan == want["best_span"]
    assert (ls.best_orders.cpu().numpy().view(np.uint16) == want["best_orders"]).all()
    assert (ls.best_mask.cpu().numpy().view(np.uint32) == want["best_mask"]).all()
    return P, inst.num_microbatches, ls.round * n


@pytest.mark.parametrize("seed", range(6))
def test_iterated_local_search_on_random_instances_follows_the_cpu_restatement(cuda_ok, seed):
    r = soak_ils_case(400 + seed, big=seed % 3 == 2)
    if r is None:
        pytest.skip("no feasible warm start drawn")
