"""The host mirror types (instance.py, schedule.py) against the reference's own, where its sources
exist (this container): the same seeded instances and JSON payloads, and for schedules the reference
times itself, the same makespan, memory traces (both semantics) and validation verdicts — also on
perturbed schedules that break rules."""

import os
import random
import sys

import pytest

REF = "/root/reference/pkg/src"

pytestmark = pytest.mark.skipif(not os.path.isdir(REF), reason="reference sources only exist in the build container")


@pytest.fixture(scope="module")
def ref():
    sys.path.insert(0, REF)
    try:
        import pipesched.heuristics as RH
        import pipesched.instance as RI
        import pipesched.schedule as RS
        yield RI, RS, RH
    finally:
        sys.path.remove(REF)


def test_instances_and_payloads_match(ref):
    RI, _, _ = ref
    from paper_2510_05186_b200 import instance as OI
    for seed in range(120):
        rng = random.Random(seed)
        P, m = rng.randint(1, 4), rng.randint(1, 5)
        if 3 * P * m > 60:
            continue
        prof = rng.choice(["ample", "tight"])
        a, b = RI.random_instance(seed, P, m, mem_profile=prof), OI.random_instance(seed, P, m, mem_profile=prof)
        d = RI.instance_to_dict(a)
        assert OI.instance_to_dict(b) == d
        assert OI.instance_to_dict(OI.instance_from_dict(d)) == d
    args = (8, 32, 100, 100, 100, 5, 150, 64 << 20, 4)
    assert OI.instance_to_dict(OI.make_uniform_instance(*args)) == RI.instance_to_dict(RI.make_uniform_instance(*args))


def test_schedules_time_and_validate_alike(ref):
    RI, RS, RH = ref
    from paper_2510_05186_b200 import instance as OI, schedule as OS
    n = 0
    for seed in range(40):
        rng = random.Random(seed)
        P, m = rng.randint(1, 4), rng.randint(1, 5)
        if 3 * P * m > 60:
            continue
        ri = RI.random_instance(seed, P, m, mem_profile=rng.choice(["ample", "tight"]),
                                post_validation=rng.random() < 0.3)
        oi = OI.instance_from_dict(RI.instance_to_dict(ri))
        for gen in (RH.one_f_one_b, RH.sequential_schedule, RH.pipeoffload_like, RH.ada_offload):
            try:
                rs = gen(ri)
            except Exception:
                continue
            d = RS.schedule_to_dict(rs)
            os_ = OS.schedule_from_dict(d)
            assert OS.schedule_to_dict(os_) == d
            assert OS.makespan(os_, oi) == RS.makespan(rs, ri)
            for sem in RS.MemorySemantics:
                osem = OS.MemorySemantics.parse(sem.value)
                try:
                    rt = RS.memory_trace(rs, ri, sem)
                except RS.NegativeUsage:
                    rt = None
                try:
                    ot = OS.memory_trace(os_, oi, osem)
                except OS.NegativeUsage:
                    ot = None
                assert (rt is None) == (ot is None)
                if rt is not None:
                    assert (rt.breakpoints, rt.peak) == (ot.breakpoints, ot.peak)
                rv, ov = RS.validate(rs, ri, sem), OS.validate(os_, oi, osem)
                assert rv.ok == ov.ok
                assert sorted(map(str, rv.violations)) == sorted(map(str, ov.violations))
            # a compute event moved later: dependency / exclusivity violations
            c = list(d["compute"])
            k = rng.randrange(len(c))
            c[k] = dict(c[k], start=c[k]["start"] + 1, end=c[k]["end"] + 1)
            rv = RS.validate(RS.schedule_from_dict(dict(d, compute=c)), ri)
            ov = OS.validate(OS.schedule_from_dict(dict(d, compute=c)), oi)
            assert rv.ok == ov.ok and sorted(map(str, rv.violations)) == sorted(map(str, ov.violations))
            n += 1
    assert n >= 60
