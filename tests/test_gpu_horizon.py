"""Instances whose horizon bound passes 2^29 quanta (e.g. 32 x 256 with 40 ms ops in microseconds).

The evaluator packs event times in 32-bit words, so it needs every event to end below 2^29 quanta.
Such instances are accepted: every candidate whose schedule stays in range is evaluated by the
evaluator, and one that leaves it (a generator structure whose makespan passes 2^29) is finished
in 64-bit time by the literal replay pass (ps_literal.cu).  Both are checked against the C oracle's
int64 restatement, and the drop-in returns the reference's schedule for it."""

import dataclasses

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_long_horizon_instance_is_exact(cuda_ok):
    import torch
    from oracle.oracle import Oracle
    from paper_2510_05186_b200 import listsched, make_uniform_instance, makespan, memory_trace, validate
    from paper_2510_05186_b200.engine import DeviceInstance
    from paper_2510_05186_b200.heuristics import generator_structures
    from paper_2510_05186_b200.packing import encode_candidate, pack_instance
    inst = make_uniform_instance(32, 256, 40000, 40000, 40000, 84, 60000, 1 << 30, 4)
    pk = pack_instance(inst)
    di = DeviceInstance(inst, packed=pk)          # rejected before round 2 (horizon > 2^29)
    structs = generator_structures(inst)
    enc = [encode_candidate(pk, o, f) for o, f in structs]
    orders = np.stack([e[0] for e in enc])
    masks = np.stack([e[1] for e in enc])
    res = di.evaluate(torch.from_numpy(orders.view(np.int16)).cuda(), torch.from_numpy(masks.view(np.int32)).cuda(),
                      peak=True)
    flags = res.flags.cpu().numpy().astype(np.uint32)
    want = Oracle(pk).eval_batch(orders, masks)
    in_range = want["makespan"] < (1 << 29)
    assert (~in_range).any() and in_range.any()
    seq = int(np.nonzero(~in_range)[0][0])         # a structure whose schedule leaves the range
    assert want["flags"][seq] == 1 and want["makespan"][seq] >= (1 << 29)
    for k in range(len(structs)):
        assert flags[k] == want["flags"][k], k
        if flags[k] == 1:
            assert res.makespan[k].item() == want["makespan"][k], k
            assert (res.peak[k].cpu().numpy() == want["peak"][k]).all(), k
            assert res.bubble[k].item() == want["bubble"][k], k
    # the drop-in: the commit-ordered trace of the 64-bit replay, as a reference Schedule
    sched = listsched.run_order(inst, *structs[seq])
    sched = dataclasses.replace(sched, metrics=None)     # recompute from the events, as the reference does
    assert validate(sched, inst).ok
    assert makespan(sched, inst) == want["makespan"][seq]
    assert [memory_trace(sched, inst).peak[i + 1] for i in range(32)] == list(want["peak"][seq])
