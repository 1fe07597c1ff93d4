"""The reference-side binding: install/uninstall patch exactly the call sites."""

import os
import sys

import pytest

REF = "/root/reference/pkg/src"


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference sources only exist in the build container")
def test_install_points_every_reference_call_site_at_the_gpu_path():
    sys.path.insert(0, REF)
    try:
        import pipesched
        from pipesched import cache, heuristics, listsched
        from paper_2510_05186_b200 import integrate
        from pipesched import online
        cpu = listsched.run_order
        cpu_best = heuristics.best_feasible
        cpu_ada = heuristics.ada_offload
        integrate.install(pipesched)
        try:
            for mod in (listsched, heuristics, cache, pipesched):
                assert mod.run_order is not cpu
                assert "GPU" in mod.run_order.__doc__
            for mod in (heuristics, cache, online, pipesched):
                assert mod.best_feasible is not cpu_best and "GPU-batched" in mod.best_feasible.__doc__
            assert heuristics.ada_offload is not cpu_ada and pipesched.ada_offload is heuristics.ada_offload
        finally:
            integrate.uninstall(pipesched)
        for mod in (listsched, heuristics, cache, pipesched):
            assert mod.run_order is cpu
        for mod in (heuristics, cache, online, pipesched):
            assert mod.best_feasible is cpu_best
        assert heuristics.ada_offload is cpu_ada and pipesched.ada_offload is cpu_ada
    finally:
        sys.path.remove(REF)


def _reference():
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    for p in (root / "baseline" / "_ref", Path(REF)):
        if (p / "pipesched" / "__init__.py").is_file():
            if str(p) not in sys.path:
                sys.path.insert(0, str(p))
            import pipesched
            return pipesched
    pytest.skip("reference package not available")


def _near_instances(ps):
    """Instances around config 2 whose fingerprints fall within a grid step of each other."""
    from paper_2510_05186_b200 import workloads
    from paper_2510_05186_b200.instance import instance_to_dict
    base = instance_to_dict(workloads.config2())
    out = []
    for tb, toff, lim in [(100, 150, 4), (110, 150, 4), (100, 170, 4), (120, 140, 4), (100, 150, 5), (90, 160, 4)]:
        d = dict(base)
        d["proc_times"] = [[[100, tb, 100] for _ in row] for row in base["proc_times"]]
        d["offload_time"] = toff
        d["mem_limits"] = [lim * (64 << 20)] * len(base["mem_limits"])
        out.append(ps.instance_from_dict(d))
    return out + [ps.random_instance(s, 3, 4, mem_profile="tight") for s in range(4)]


def test_fingerprint_and_radius_follow_the_reference_lookup(tmp_path):
    """cache.fingerprint == discretize (cache.py:111-131); within_radius ranks like lookup
    (cache.py:207-221), so its first index is lookup's hit."""
    ps = _reference()
    from paper_2510_05186_b200 import cache
    from paper_2510_05186_b200.cache import entry_from_record, fingerprint, within_radius
    insts = _near_instances(ps)
    for inst in insts:
        k = ps.discretize(inst)
        assert fingerprint(inst) == (k.num_stages, k.num_microbatches, tuple(k.ratios), k.post_validation)
    # a db of structures recorded on each instance (sequential orders: no solver needed)
    db = ps.CacheDb(tmp_path / "c.jsonl")
    for inst in insts:
        s = ps.sequential_schedule(inst)
        db.append(ps.entry_from_schedule(inst, s))
    records = [entry_from_record(e.to_dict()) for e in db.entries()]
    for inst in insts:
        hit = ps.lookup(db, ps.discretize(inst))
        idx = within_radius(records, inst)
        ref_idx = within_radius(list(db.entries()), inst)
        assert idx == ref_idx
        if hit is None:
            assert idx == []
        else:
            assert db.entries()[idx[0]] == hit
    assert cache.GRID_STEP == 0.25
