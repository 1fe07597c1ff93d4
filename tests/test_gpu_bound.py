"""GPU batched B&B node bounds vs the reference solver's recorded bounds and the C restatement."""

import gzip
import json
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_bounds_match_reference_solver_nodes(cuda_ok):
    import torch
    from paper_2510_05186_b200.bound import BoundEvaluator
    from paper_2510_05186_b200.instance import instance_from_dict
    d = json.load(gzip.open(Path(__file__).parent / "golden" / "bounds.json.gz", "rt"))
    total = 0
    for r in d["rows"]:
        inst = instance_from_dict(r["instance"])
        P, m = inst.num_stages, inst.num_microbatches
        nodes = r["nodes"]
        clock = np.array([x["t"] for x in nodes], np.int32)
        sfree = np.array([x["sfree"] for x in nodes], np.int32)
        start = np.full((len(nodes), P, m, 3), -1, np.int32)
        for n, x in enumerate(nodes):
            for i, j, k, s in x["comp"]:
                start[n, i - 1, j - 1, k] = s
        ev = BoundEvaluator(inst)
        got = ev.bounds(torch.from_numpy(clock).cuda(), torch.from_numpy(sfree).cuda(),
                        torch.from_numpy(start).cuda()).cpu().numpy()
        assert (got == np.array([x["lb"] for x in nodes])).all(), r["instance"].get("num_stages")
        total += len(nodes)
    assert total > 5000


@pytest.mark.parametrize("cfg", [2, 3, 4])
def test_bounds_match_restatement_on_partial_schedules(cuda_ok, cfg):
    """Nodes cut from real schedules at BASELINE shapes (a prefix of a generator's commit order
    committed, the clock at the cut) — kernel vs or_bound, post-validation on and off."""
    import dataclasses
    import torch
    from oracle.oracle import Oracle, bound
    from paper_2510_05186_b200 import workloads
    from paper_2510_05186_b200.bound import BoundEvaluator, node_arrays
    from paper_2510_05186_b200.heuristics import best_feasible
    from paper_2510_05186_b200.packing import pack_instance
    rng = np.random.default_rng(cfg)
    base = workloads.CONFIGS[cfg]()
    for post in (False, True):
        inst = dataclasses.replace(base, post_validation=post) if dataclasses.is_dataclass(base) else base
        s, _ = best_feasible(inst)
        ev_list = sorted(s.compute, key=lambda e: (e.start, e.op))
        nodes = []
        for cut in sorted(rng.integers(0, len(ev_list) + 1, size=24).tolist()):
            comp = {e.op: e.start for e in ev_list[:cut]}
            t = ev_list[cut - 1].start if cut else 0
            sf = {i: 0 for i in range(1, inst.num_stages + 1)}
            for e in ev_list[:cut]:
                sf[e.op.stage] = max(sf[e.op.stage], e.start + inst.proc_time[e.op])
            nodes.append((t, sf, comp))
        clock, sfree, start = node_arrays(inst, nodes)
        got = BoundEvaluator(inst).bounds(torch.from_numpy(clock).cuda(), torch.from_numpy(sfree).cuda(),
                                          torch.from_numpy(start).cuda()).cpu().numpy()
        orc = Oracle(pack_instance(inst))
        want = [bound(orc, clock[n], sfree[n], start[n].astype(np.int64), inst.post_validation)
                for n in range(len(nodes))]
        assert got.tolist() == want
