"""The anytime solver API (start_session / solve / incumbent_stream / online_sim) on the GPU search."""

import pytest

from _golden import CORPORA, corpus


@pytest.mark.gpu
def test_lower_bound_is_the_reference_root_bound(cuda_ok):
    """lower_bound == the reference solver's root bound (the first node it bounds, solver.py:481)."""
    import gzip
    import json
    from pathlib import Path
    from paper_2510_05186_b200.instance import instance_from_dict
    from paper_2510_05186_b200.solver import lower_bound
    d = json.load(gzip.open(Path(__file__).parent / "golden" / "bounds.json.gz", "rt"))
    n = 0
    for r in d["rows"]:
        root = r["nodes"][0]
        assert root["t"] == 0 and not root["comp"]
        assert lower_bound(instance_from_dict(r["instance"]), r["post"]) == root["lb"]
        n += 1
    assert n >= 20


@pytest.mark.gpu
def test_lower_bound_is_valid_on_every_reference_schedule(cuda_ok):
    from paper_2510_05186_b200.solver import lower_bound
    checked = 0
    for name in CORPORA:
        for inst, pk, cases in corpus(name):
            lb = lower_bound(inst, inst.post_validation)
            for case in cases:
                if "makespan" in case:
                    assert case["makespan"] >= lb
                    checked += 1
    assert checked > 1000


@pytest.mark.gpu
def test_start_session_streams_strict_improvements(cuda_ok):
    from paper_2510_05186_b200 import makespan, validate, workloads
    from paper_2510_05186_b200.search import SearchConfig
    from paper_2510_05186_b200.solver import (SessionClosed, SolveBudget, incumbent_stream, online_sim,
                                              solve, start_session)
    inst = workloads.config2()
    cfg = SearchConfig(seed=3, neighbours=2048)
    session = start_session(inst, SolveBudget(wall_time_limit=None, node_limit=6 * 2048), search=cfg)
    events = list(incumbent_stream(session))
    with pytest.raises(SessionClosed):
        incumbent_stream(session)
    spans = [ev.makespan for ev in events]
    assert all(a > b for a, b in zip(spans, spans[1:]))
    assert events[-1].status == session.outcome.status in ("Feasible", "Optimal")
    out = session.outcome
    assert out.incumbent_makespan == spans[-1] == makespan(out.incumbent, inst)
    assert validate(out.incumbent, inst).ok
    assert out.lower_bound <= out.incumbent_makespan
    assert out.nodes == 6 * 2048
    assert solve(inst, budget=SolveBudget(wall_time_limit=0.0)).incumbent_makespan == spans[0]
    rep = online_sim(inst, 3)
    assert rep.steps[0].source == "warm" and rep.total_time == 3 * spans[0]


@pytest.mark.gpu
def test_batched_cache_adapt_matches_reference_replays(cuda_ok):
    """Explicit channel-order replays of reference schedules, one launch for all entries."""
    from _golden import structure
    from paper_2510_05186_b200.cache import CachedOrder, adapt_batch, best_adapted
    inst, pk, cases = corpus("ref_tests")[0]
    entries, want = [], []
    for case in cases:
        if "channel_orders" not in case:
            continue
        orders, off, chans = structure(case)
        entries.append(CachedOrder(inst.num_stages, inst.num_microbatches,
                                   tuple(orders[i] for i in range(1, inst.num_stages + 1)), off,
                                   tuple(chans[g] for g in range(len(inst.topology_groups)))))
        want.append(case.get("makespan"))
    got = adapt_batch(entries, inst)
    from paper_2510_05186_b200 import makespan
    for s, w in zip(got, want):
        assert (s is None) == (w is None)
        if s is not None:
            assert makespan(s, inst) == w
    s, k = best_adapted(entries, inst)
    assert makespan(s, inst) == min(w for w in want if w is not None)
