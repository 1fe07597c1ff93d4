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
