"""The UNMODIFIED reference package with the B200 path installed, on the GPU.

The reference ships to the GPU box as ``baseline/_ref`` (pip-installed from /root/reference,
git-ignored).  With ``integrate.install(pipesched)`` the reference's own call
sites time every structure on the GPU; everything the reference computes from them must be
``==`` to its CPU path, commit order included:

* ``best_feasible`` / ``ada_offload`` / ``one_f_one_b`` (heuristics.py:61-210) at config 2;
* ``cache.adapt`` on the known answers of the reference's tests (tests/test_cache.py:148-176:
  same makespan, exactly 2x under doubled times, None under a tighter limit) and an
  explicit-channel replay at config 2 (cache.py:224-240);
* ``start_session(warm=<GPU local-search winner>)`` — the reference branch-and-bound run from the
  search's winner (solver.py:543-565), node-limited so both runs see the same budget.

With ``install(pipesched, search=WarmSearch(...))`` the reference's own ``online_sim``
(online.py:48-81) starts from the GPU search's winner: its trajectory opens with the search's
strict improvements and its solver outcome equals the CPU reference solver run from that winner.
"""

import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]
CANDIDATES = (ROOT / "baseline" / "_ref", Path("/root/reference/pkg/src"))


@pytest.fixture(scope="module")
def ps():
    for p in CANDIDATES:
        if (p / "pipesched" / "__init__.py").is_file():
            if str(p) not in sys.path:
                sys.path.insert(0, str(p))
            import pipesched
            return pipesched
    pytest.skip("reference package not installed (baseline/_ref)")


def _scaled(ps, inst, k):
    d = ps.instance_to_dict(inst)
    d["proc_times"] = [[[t * k for t in ops] for ops in row] for row in d["proc_times"]]
    d["comm_time"] *= k
    d["offload_time"] *= k
    return ps.instance_from_dict(d)


def _answers(ps, c1, c2, small, warm1):
    F, B, W = ps.OpKind.F, ps.OpKind.B, ps.OpKind.W
    out = {}
    out["best"] = ps.best_feasible(c2, ps.AdaParams())
    out["ada"] = ps.ada_offload(c2, ps.AdaParams())
    try:
        out["1f1b"] = ps.one_f_one_b(c2)
    except ps.InfeasibleSchedule as e:
        out["1f1b"] = ("infeasible", str(e))
    sol = ps.solve(small, budget=ps.SolveBudget(wall_time_limit=None, node_limit=20000))
    entry = ps.entry_from_schedule(small, sol.incumbent)
    out["solve_small"] = (sol.status, sol.incumbent_makespan, sol.lower_bound, sol.nodes, sol.incumbent)
    out["adapt_same"] = ps.adapt(entry, small)
    doubled = _scaled(ps, small, 2)
    out["adapt_doubled"] = ps.adapt(entry, doubled)
    one = ps.make_uniform_instance(1, 2, 1, 1, 1, 0, 1, 2, 2)
    both_first = ps.run_order(one, {1: (ps.OpId(1, 1, F), ps.OpId(1, 2, F), ps.OpId(1, 1, B),
                                        ps.OpId(1, 1, W), ps.OpId(1, 2, B), ps.OpId(1, 2, W))}, frozenset())
    d = ps.instance_to_dict(one)
    d["mem_limits"] = [2]
    out["adapt_tighter"] = ps.adapt(ps.entry_from_schedule(one, both_first), ps.instance_from_dict(d))
    out["adapt_c2"] = ps.adapt(ps.entry_from_schedule(c2, out["best"][0]), c2)
    budget = ps.SolveBudget(wall_time_limit=None, node_limit=3000)
    sess = ps.start_session(c1, budget, warm=warm1)
    evs = [(e.schedule, e.makespan, e.lower_bound, e.status) for e in ps.incumbent_stream(sess)]
    o = sess.outcome
    out["session"] = (o.status, o.incumbent_makespan, o.lower_bound, o.nodes, o.prunes_bound, o.dead_ends,
                      o.incumbent, evs)
    return out, (small, doubled, sol)


def _instances(ps):
    from paper_2510_05186_b200 import workloads
    from paper_2510_05186_b200.instance import instance_to_dict
    c1 = ps.instance_from_dict(instance_to_dict(workloads.config1()))
    c2 = ps.instance_from_dict(instance_to_dict(workloads.config2()))
    small = ps.random_instance(3, 2, 2, mem_profile="tight")
    return c1, c2, small


def test_installed_reference_equals_its_cpu_path(cuda_ok, ps):
    from paper_2510_05186_b200 import integrate
    from paper_2510_05186_b200.search import SearchConfig
    c1, c2, small = _instances(ps)
    integrate.install(ps)
    try:
        assert "GPU" in ps.heuristics.run_order.__doc__ and "GPU" in ps.cache.run_order.__doc__
        w0, _ = ps.best_feasible(c1, ps.AdaParams())
        warm1, events = integrate.search_warm_start(
            ps, c1, w0, integrate.WarmSearch(SearchConfig(seed=7, neighbours=8192), patience=8))
        assert isinstance(warm1, ps.Schedule) and ps.validate(warm1, c1, ps.MemorySemantics.STRICT).ok
        spans = [e.makespan for e in events]
        assert spans == sorted(spans, reverse=True) and len(set(spans)) == len(spans)
        assert ps.makespan(warm1, c1) == spans[-1] <= ps.makespan(w0, c1)
        gpu, (small_i, doubled, sol) = _answers(ps, c1, c2, small, warm1)
    finally:
        integrate.uninstall(ps)
    assert "GPU" not in (ps.heuristics.run_order.__doc__ or "")
    cpu, _ = _answers(ps, c1, c2, small, warm1)
    for key in cpu:
        assert gpu[key] == cpu[key], key
    # the reference's own adapt known answers hold on the GPU path (tests/test_cache.py:148-176)
    assert ps.makespan(gpu["adapt_same"], small_i) == sol.incumbent_makespan
    assert ps.makespan(gpu["adapt_doubled"], doubled) == 2 * sol.incumbent_makespan
    assert gpu["adapt_tighter"] is None
    assert gpu["adapt_c2"] == gpu["best"][0]


def test_reference_online_sim_starts_from_the_gpu_search(cuda_ok, ps):
    from paper_2510_05186_b200 import integrate
    from paper_2510_05186_b200.search import SearchConfig
    c1, _, _ = _instances(ps)
    budget = ps.SolveBudget(wall_time_limit=None, node_limit=2000)
    search = integrate.WarmSearch(SearchConfig(seed=3, neighbours=8192), patience=8)
    integrate.install(ps, search=search)
    try:
        assert "GPU" in ps.online.start_session.__doc__
        rep = ps.online_sim(c1, iterations=6, budget=budget)
        warm, _ = ps.best_feasible(c1, ps.AdaParams())
        winner, events = integrate.search_warm_start(ps, c1, warm, search)
    finally:
        integrate.uninstall(ps)
    assert ps.online.start_session is ps.solver.start_session
    spans = [s for _, s in rep.trajectory]
    n_search = len(events) - 1
    # the trajectory opens with the warm start and the search's improvements, in order
    assert spans[:n_search + 1] == [e.makespan for e in events]
    assert rep.steps[0].span == ps.makespan(warm, c1)
    assert min(st.span for st in rep.steps) <= ps.makespan(winner, c1)
    # the solver part is the CPU reference branch-and-bound run from the winner
    cpu = ps.start_session(c1, budget, warm=winner)
    assert rep.solver_status == cpu.outcome.status
    assert spans[n_search:] == [e.makespan for e in ps.incumbent_stream(cpu)]


def _ev(s):
    if s is None:
        return None
    return ([(e.op.stage, e.op.microbatch, int(e.op.kind), e.start, e.end) for e in s.compute],
            [(e.op.stage, e.op.microbatch, e.kind.value, e.start, e.end) for e in s.transfers])


def test_radius_adapt_equals_reference_adapt_of_every_entry(cuda_ok, ps, tmp_path):
    """cache.adapt_radius re-times every entry within the lookup radius in one launch; each result
    equals the reference's own adapt of that entry (cache.py:224-240), and the best is at least as
    good as the reference's single lookup hit (cache.py:243-259)."""
    from test_integrate import _near_instances
    from paper_2510_05186_b200.cache import adapt_radius, entry_from_record
    insts = _near_instances(ps)
    db = ps.CacheDb(tmp_path / "c.jsonl")
    for inst in insts:
        for s in (ps.sequential_schedule(inst), ps.best_feasible(inst, ps.AdaParams())[0]):
            db.append(ps.entry_from_schedule(inst, s))
    entries = db.entries()
    records = [entry_from_record(e.to_dict()) for e in entries]
    compared = 0
    for inst in insts:
        best, k, allr = adapt_radius(records, inst)
        for idx, s in allr:
            assert _ev(s) == _ev(ps.adapt(entries[idx], inst)), idx
            compared += 1
        hit = ps.lookup(db, ps.discretize(inst))
        if hit is not None:
            ref = ps.adapt(hit, inst)
            if ref is not None:
                from paper_2510_05186_b200 import makespan as our_makespan
                assert best is not None and ps.makespan(ref, inst) >= our_makespan(best, inst)
    assert compared >= len(insts)
