"""GPU evaluator (C ABI -> sm_100a kernel) vs the reference fixtures and the C oracle."""

import numpy as np
import pytest

from _golden import CORPORA, case_arrays, corpus, split_trace, structure

pytestmark = pytest.mark.gpu


def _eval_cases(inst, pk, cases, explicit):
    import torch
    from paper_2510_05186_b200.engine import DeviceInstance
    sel = [c for c in cases if ("channel_orders" in c) == explicit]
    if not sel:
        return [], None
    arrs = [case_arrays(pk, c) for c in sel]
    orders = torch.from_numpy(np.stack([a[0] for a in arrs]).view(np.int16)).cuda()
    masks = torch.from_numpy(np.stack([a[1] for a in arrs]).view(np.int32)).cuda()
    chans = None
    if explicit:
        width = max(a[2].shape[1] for a in arrs)
        ch = np.full((len(arrs), pk.num_channels, width), 0xFFFFFFFF, np.uint32)
        for k, a in enumerate(arrs):
            ch[k, :, :a[2].shape[1]] = a[2]
        chans = torch.from_numpy(ch.view(np.int32)).cuda()
    di = DeviceInstance(inst, packed=pk)
    res = di.evaluate(orders, masks, chans, peak=True, trace=True)
    torch.cuda.synchronize()
    return sel, {k: (v.cpu().numpy() if v is not None else None) for k, v in vars(res).items()}


def _check(sel, r, pk):
    for k, case in enumerate(sel):
        flags = int(r["flags"][k])
        if "infeasible" in case:
            assert flags == 2, (k, flags)
            blocked = int(r["blocked"][k]) & 0xFFFFFFFF
            assert [i + 1 for i in range(pk.num_stages) if (blocked >> i) & 1] == case["infeasible"]
            continue
        assert flags == 1, (k, flags, case)
        assert int(r["makespan"][k]) == case["makespan"]
        assert repr(float(r["bubble"][k])) == case["bubble"]
        assert [int(x) for x in r["peak"][k]] == case["peak"]
        n = len(case["compute"]) + len(case["transfers"])
        comp, tr = split_trace(r["trace_code"][k][:n], r["trace_start"][k][:n])
        assert comp == case["compute"]
        assert tr == case["transfers"]


@pytest.mark.parametrize("name", CORPORA)
@pytest.mark.parametrize("explicit", [False, True])
def test_kernel_matches_reference_fixtures(cuda_ok, name, explicit):
    checked = 0
    for inst, pk, cases in corpus(name):
        sel, r = _eval_cases(inst, pk, cases, explicit)
        if sel:
            _check(sel, r, pk)
            checked += len(sel)
    assert checked > 0


def test_drop_in_run_order_equals_reference_schedule(cuda_ok):
    from paper_2510_05186_b200 import OrderInfeasible, run_order, makespan, memory_trace, validate
    inst, pk, cases = corpus("ref_tests")[0]
    for case in cases[:20]:
        orders, off, chans = structure(case)
        if "infeasible" in case:
            with pytest.raises(OrderInfeasible) as err:
                run_order(inst, orders, off, chans)
            assert list(err.value.stages) == case["infeasible"]
            continue
        s = run_order(inst, orders, off, chans)
        assert [[e.op.stage, e.op.microbatch, int(e.op.kind), e.start] for e in s.compute] == case["compute"]
        assert makespan(s, inst) == case["makespan"]
        assert [memory_trace(s, inst).peak[i] for i in range(1, pk.num_stages + 1)] == case["peak"]
        assert validate(s, inst).ok


def test_kernel_matches_oracle_on_config_samples(cuda_ok):
    """Larger batches at BASELINE shapes: kernel vs C oracle on perturbed generator orders."""
    import torch
    from oracle.oracle import Oracle
    from paper_2510_05186_b200 import workloads
    from paper_2510_05186_b200.engine import DeviceInstance
    from paper_2510_05186_b200.heuristics import generator_structures
    from paper_2510_05186_b200.packing import encode_candidate, pack_instance
    rng = np.random.default_rng(7)
    for cfg, n in ((1, 256), (2, 128), (3, 64), (4, 8), (5, 4)):
        inst = workloads.CONFIGS[cfg]()
        pk = pack_instance(inst)
        base = [encode_candidate(pk, o, f) for o, f in generator_structures(inst)]
        orders = np.zeros((n, pk.num_stages, pk.order_stride), np.uint16)
        masks = np.zeros((n, pk.mask_words), np.uint32)
        for c in range(n):
            o, mk, _ = base[c % len(base)]
            o, mk = o.copy(), mk.copy()
            for _ in range(int(rng.integers(0, 4))):
                i = int(rng.integers(pk.num_stages))
                a = int(rng.integers(3 * pk.num_microbatches - 1))
                o[i, a], o[i, a + 1] = o[i, a + 1], o[i, a]
            if pk.act_size.any() and rng.random() < 0.5:
                b = int(rng.integers(pk.num_stages * pk.num_microbatches))
                mk[b >> 5] ^= np.uint32(1 << (b & 31))
            orders[c], masks[c] = o, mk
        di = DeviceInstance(inst, packed=pk)
        res = di.evaluate(torch.from_numpy(orders.view(np.int16)).cuda(),
                          torch.from_numpy(masks.view(np.int32)).cuda(), peak=True)
        want = Oracle(pk).eval_batch(orders, masks)
        assert (res.flags.cpu().numpy() == want["flags"].astype(np.int32)).all(), cfg
        assert (res.makespan.cpu().numpy() == want["makespan"]).all(), cfg
        ok = want["flags"] == 1
        assert (res.peak.cpu().numpy()[ok] == want["peak"][ok]).all(), cfg
        assert (res.bubble.cpu().numpy()[ok] == want["bubble"][ok]).all(), cfg
