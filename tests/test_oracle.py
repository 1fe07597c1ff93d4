"""Pin the C oracle (oracle/ps_oracle.c) against reference-generated golden vectors (CPU)."""

import numpy as np
import pytest

from _golden import CORPORA, case_arrays, corpus, split_trace
from oracle.oracle import Oracle, philox4x32_10


@pytest.mark.parametrize("name", CORPORA)
def test_oracle_matches_reference_fixtures(name):
    n_feasible = n_infeasible = 0
    for inst, pk, cases in corpus(name):
        orc = Oracle(pk)
        for case in cases:
            orders, mask, chans = case_arrays(pk, case)
            r = orc.run(orders, mask, chans)
            if "infeasible" in case:
                assert r["flags"] == 2, case
                stages = [i + 1 for i in range(pk.num_stages) if (r["blocked"] >> i) & 1]
                assert stages == case["infeasible"]
                n_infeasible += 1
                continue
            assert r["flags"] == 1
            assert r["makespan"] == case["makespan"]
            assert repr(r["bubble"]) == case["bubble"]          # bit-exact fp64
            assert list(r["peak"]) == case["peak"]
            comp, tr = split_trace(r["trace_code"], r["trace_start"])
            assert comp == case["compute"]                      # commit order included
            assert tr == case["transfers"]
            n_feasible += 1
    assert n_feasible > 0


def test_oracle_batch_matches_single():
    inst, pk, cases = corpus("ref_tests")[4]
    orc = Oracle(pk)
    arrs = [case_arrays(pk, c) for c in cases if "channel_orders" not in c]
    orders = np.stack([a[0] for a in arrs])
    masks = np.stack([a[1] for a in arrs])
    out = orc.eval_batch(orders, masks, threads=3)
    for k, (o, mk, _) in enumerate(arrs):
        r = orc.run(o, mk)
        assert out["makespan"][k] == r["makespan"]
        assert out["flags"][k] == r["flags"]


def test_philox_known_answers():
    # Random123 known-answer vectors for philox4x32-10
    assert philox4x32_10([0, 0, 0, 0], [0, 0]) == [0x6627e8d5, 0xe169c58d, 0xbc57ac4c, 0x9b00dbd8]
    assert philox4x32_10([0xffffffff] * 4, [0xffffffff] * 2) == [0x408f276d, 0x41c83b0e, 0xa20bc7c6, 0x6d5451fd]
    assert philox4x32_10([0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344], [0xa4093822, 0x299f31d0]) == \
        [0xd16cfe09, 0x94fdcceb, 0x5001e420, 0x24126ea1]


def test_malformed_rows_follow_the_reference():
    """Rows with a repeated op, a missing op, a cut tail or nothing at all: the reference replays
    them literally and raises OrderInfeasible with the rows not yet exhausted
    (tests/golden/malformed.json.gz, make_malformed_golden.py)."""
    n = 0
    for inst, pk, cases in corpus("malformed"):
        orc = Oracle(pk)
        for case in cases:
            orders, mask, chans = case_arrays(pk, case)
            r = orc.run(orders, mask, chans)
            assert r["flags"] == 2, case["damage"]
            assert [i + 1 for i in range(pk.num_stages) if (r["blocked"] >> i) & 1] == case["infeasible"], case["damage"]
            n += 1
    assert n >= 150


def test_codes_naming_no_op_are_malformed():
    inst, pk, cases = corpus("ref_tests")[0]
    orc = Oracle(pk)
    orders, mask, _ = case_arrays(pk, cases[0])
    bad = orders.copy()
    bad[0, 1] = (pk.num_microbatches + 2) << 2     # microbatch out of range
    assert orc.run(bad, mask)["flags"] == 4
    bad = orders.copy()
    bad[0, 1] = bad[0, 1] | 3                       # kind 3
    assert orc.run(bad, mask)["flags"] == 4


def test_bound_restatement_matches_reference_solver():
    """or_bound (the C restatement of solver.py:321-383) equals the bound the reference solver
    computed at every recorded node (tests/golden/bounds.json.gz, make_bound_golden.py)."""
    import gzip
    import json
    from pathlib import Path
    import numpy as np
    from oracle.oracle import Oracle, bound
    from paper_2510_05186_b200.instance import instance_from_dict
    from paper_2510_05186_b200.packing import pack_instance
    d = json.load(gzip.open(Path(__file__).parent / "golden" / "bounds.json.gz", "rt"))
    n = 0
    for r in d["rows"]:
        pk = pack_instance(instance_from_dict(r["instance"]))
        orc = Oracle(pk)
        P, m = pk.num_stages, pk.num_microbatches
        for node in r["nodes"]:
            st = np.full((P, m, 3), -1, np.int64)
            for i, j, k, s in node["comp"]:
                st[i - 1, j - 1, k] = s
            assert bound(orc, node["t"], node["sfree"], st, r["post"]) == node["lb"]
            n += 1
    assert n > 5000


def test_channel_neighbours_restate_the_stage_shift_and_keep_channel_lengths():
    """or_neighbour_explicit: with shift_permille 1000 it is or_neighbour's stage
    shift; its transfer shifts permute one channel's entries and never change the offload bits."""
    import numpy as np
    from oracle.oracle import Oracle, neighbour_explicit
    from _golden import case_arrays, corpus
    for inst, pk, cases in corpus("ref_tests"):
        sel = [c for c in cases if "channel_orders" in c and "makespan" in c and any(c["channel_orders"])]
        if not sel:
            continue
        orc = Oracle(pk)
        o, mk, ch = case_arrays(pk, sel[0])
        seen = set()
        for idx in range(64):
            t0, o0, m0 = orc.neighbour(o, mk, 5, 700, 4, 3, idx)
            t1, o1, m1, c1 = neighbour_explicit(orc, o, mk, ch, 5, 1000, 4, 3, idx)
            if t0 == 1:
                assert t1 == 1 and (o1 == o0).all()
            t2, o2, m2, c2 = neighbour_explicit(orc, o, mk, ch, 5, 0, 4, 3, idx)
            seen.add(t2)
            assert (m2 == mk).all() and (o2 == o).all()
            for g in range(ch.shape[0]):
                assert sorted(c2[g].tolist()) == sorted(ch[g].tolist())
        assert 3 in seen
        return
    raise AssertionError("no explicit-mode fixture with transfers")
