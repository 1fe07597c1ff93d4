"""Edge cases of the batch API on the GPU: empty batches, malformed candidates (with and without a
recorded base, in the register seen-set path m <= 64 and the shared-memory one m > 64), and the
drop-in's error behaviour.  Rows that repeat an op, miss one or are cut short follow the
reference (replayed literally, OrderInfeasible with its blocked stages: tests/golden/malformed.json.gz
recorded by the reference, and the C oracle pinned to it); op codes that name no op stay
PS_FLAG_MALFORMED."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _setup(cfg):
    from paper_2510_05186_b200 import workloads
    from paper_2510_05186_b200.engine import DeviceInstance
    from paper_2510_05186_b200.heuristics import generator_structures
    from paper_2510_05186_b200.packing import encode_candidate, pack_instance
    inst = workloads.CONFIGS[cfg]()
    pk = pack_instance(inst)
    base = [encode_candidate(pk, o, f) for o, f in generator_structures(inst)]
    return inst, pk, base, DeviceInstance(inst, packed=pk)


def _malformed_batch(pk, base, rng):
    """Well-formed neighbours interleaved with every kind of structural damage."""
    P, m = pk.num_stages, pk.num_microbatches
    offl = np.argwhere(pk.act_size > 0)
    not_offl = np.argwhere(pk.act_size <= 0)
    rows, masks, kinds = [], [], []
    for c in range(48):
        o, mk, _ = base[c % len(base)]
        o, mk = o.copy(), mk.copy()
        i = int(rng.integers(P))
        a = int(rng.integers(3 * m - 1))
        kind = c % 6
        if kind == 0:          # well formed: an adjacent swap
            o[i, a], o[i, a + 1] = o[i, a + 1], o[i, a]
        elif kind == 1:        # duplicate op (and one op missing)
            o[i, a + 1] = o[i, a]
        elif kind == 2:        # op kind 3 does not exist
            o[i, a] = (o[i, a] & ~np.uint16(3)) | np.uint16(3)
        elif kind == 3:        # microbatch out of range
            o[i, a] = np.uint16((m + int(rng.integers(0, 4))) << 2)
        elif kind == 4:        # late damage: the last op of the last stage repeats the first
            o[P - 1, 3 * m - 1] = o[P - 1, 0]
        else:                  # offload bit on an F without an offloadable activation
            if len(not_offl):
                s, j = not_offl[int(rng.integers(len(not_offl)))]
                b = int(s) * m + int(j)
                mk[b >> 5] |= np.uint32(1 << (b & 31))
            elif len(offl):    # everything offloadable: toggle a real bit instead (well formed)
                s, j = offl[0]
                b = int(s) * m + int(j)
                mk[b >> 5] ^= np.uint32(1 << (b & 31))
        rows.append(o)
        masks.append(mk)
        kinds.append(kind)
    return np.stack(rows), np.stack(masks), kinds


@pytest.mark.parametrize("cfg", [2, 4])
@pytest.mark.parametrize("with_base", [False, True])
def test_malformed_candidates_match_the_oracle(cuda_ok, cfg, with_base):
    import torch
    from oracle.oracle import Oracle
    from paper_2510_05186_b200.engine import Base
    inst, pk, base, di = _setup(cfg)
    orders, masks, kinds = _malformed_batch(pk, base, np.random.default_rng(11 + cfg))
    b = None
    if with_base:
        o0, mk0, _ = base[0]
        b = Base(di)
        b.record(torch.from_numpy(o0.view(np.int16)).cuda(), torch.from_numpy(mk0.view(np.int32)).cuda())
    res = di.evaluate(torch.from_numpy(orders.view(np.int16)).cuda(),
                      torch.from_numpy(masks.view(np.int32)).cuda(), peak=True, base=b)
    want = Oracle(pk).eval_batch(orders, masks)
    flags = res.flags.cpu().numpy().astype(np.uint32)
    assert (flags == want["flags"]).all(), (cfg, with_base, list(zip(kinds, flags, want["flags"])))
    # codes naming no op are malformed; repeated ops end in OrderInfeasible like the reference
    for k, f in zip(kinds, flags):
        if k in (2, 3):
            assert f == 4, (k, f)
        elif k in (1, 4):
            assert f == 2, (k, f)
    assert (res.blocked.cpu().numpy().astype(np.uint32)[flags == 2] == want["blocked"][flags == 2]).all()
    ok = want["flags"] == 1
    assert (res.makespan.cpu().numpy()[ok] == want["makespan"][ok]).all()
    assert (res.peak.cpu().numpy()[ok] == want["peak"][ok]).all()


def test_host_path_flags_malformed_candidates(cuda_ok):
    from oracle.oracle import Oracle
    inst, pk, base, di = _setup(2)
    orders, masks, _ = _malformed_batch(pk, base, np.random.default_rng(5))
    res = di.evaluate_host(orders.astype(np.uint8) if pk.num_microbatches <= 64 else orders, masks)
    want = Oracle(pk).eval_batch(orders, masks)
    assert (res.flags.astype(np.uint32) == want["flags"]).all()
    ok = want["flags"] == 1
    assert (res.makespan[ok] == want["makespan"][ok]).all()
    dl = want["flags"] == 2
    assert (res.blocked.astype(np.uint32)[dl] == want["blocked"][dl]).all()


def test_empty_batches(cuda_ok):
    import torch
    inst, pk, base, di = _setup(2)
    P, stride, w = pk.num_stages, pk.order_stride, pk.mask_words
    res = di.evaluate(torch.zeros((0, P, stride), dtype=torch.int16, device="cuda"),
                      torch.zeros((0, w), dtype=torch.int32, device="cuda"), peak=True)
    torch.cuda.synchronize()
    assert res.makespan.numel() == 0 and res.flags.numel() == 0
    out = di.evaluate_host(np.zeros((0, P, stride), np.uint16), np.zeros((0, w), np.uint32))
    assert out.makespan.shape == (0,)


def test_drop_in_run_order_on_malformed_structures(cuda_ok):
    """A row with a repeated op raises OrderInfeasible with the reference's stages; an op of
    another stage or an overlong row is a ValueError; offloading an op without an
    activation is the reference's KeyError."""
    from paper_2510_05186_b200 import listsched, workloads
    from paper_2510_05186_b200.heuristics import generator_structures
    from paper_2510_05186_b200.instance import OpId, OpKind
    inst = workloads.config2()
    orders, off = generator_structures(inst)[0]
    bad = dict(orders)
    row = list(bad[1])
    row[1] = row[0]
    bad[1] = tuple(row)
    with pytest.raises(listsched.OrderInfeasible):
        listsched.run_order(inst, bad, off)
    foreign = dict(orders)
    foreign[1] = (OpId(2, 1, OpKind.F),) + tuple(orders[1][1:])
    with pytest.raises(ValueError):
        listsched.run_order(inst, foreign, off)
    with pytest.raises(KeyError):
        listsched.run_order(inst, orders, set(off) | {OpId(1, 1, OpKind.B)})


@pytest.mark.parametrize("explicit", [False, True])
def test_malformed_rows_match_the_reference(cuda_ok, explicit):
    """The reference-recorded outcomes of damaged rows (tests/golden/malformed.json.gz) through
    ps_eval_batch and through the drop-in run_order (OrderInfeasible.stages)."""
    import torch
    from _golden import case_arrays, corpus, structure
    from paper_2510_05186_b200 import listsched
    from paper_2510_05186_b200.engine import DeviceInstance
    n = 0
    for inst, pk, cases in corpus("malformed"):
        sel = [c for c in cases if ("channel_orders" in c) == explicit]
        if not sel:
            continue
        arrs = [case_arrays(pk, c) for c in sel]
        chans = None
        if explicit:
            width = max(a[2].shape[1] for a in arrs)
            ch = np.full((len(arrs), pk.num_channels, width), 0xFFFFFFFF, np.uint32)
            for k, a in enumerate(arrs):
                ch[k, :, :a[2].shape[1]] = a[2]
            chans = torch.from_numpy(ch.view(np.int32)).cuda()
        di = DeviceInstance(inst, packed=pk)
        res = di.evaluate(torch.from_numpy(np.stack([a[0] for a in arrs]).view(np.int16)).cuda(),
                          torch.from_numpy(np.stack([a[1] for a in arrs]).view(np.int32)).cuda(), chans, peak=True)
        flags = res.flags.cpu().numpy()
        blocked = res.blocked.cpu().numpy().astype(np.uint32)
        for k, case in enumerate(sel):
            assert flags[k] == 2, case["damage"]
            assert [i + 1 for i in range(pk.num_stages) if (blocked[k] >> i) & 1] == case["infeasible"]
            orders, off, ch = structure(case)
            with pytest.raises(listsched.OrderInfeasible) as err:
                listsched.run_order(inst, orders, off, ch)
            assert list(err.value.stages) == case["infeasible"]
            n += 1
    assert n >= (20 if explicit else 150)


def test_delta_encoded_host_batch_equals_the_full_rows(cuda_ok):
    """ps_eval_batch_host_delta (candidates as differences from a reference structure, only the
    differences cross PCIe) gives the same outputs as ps_eval_batch_host on the full rows, with
    and without a recorded base, config 2 (m <= 64) and config 4 (m > 64)."""
    import torch
    from paper_2510_05186_b200.engine import Base
    from paper_2510_05186_b200.packing import delta_encode
    for cfg in (2, 4):
        inst, pk, base, di = _setup(cfg)
        rng = np.random.default_rng(cfg)
        o0, mk0, _ = base[-1]
        orders, masks, kinds = _malformed_batch(pk, [(o0, mk0, None)], rng)
        keep = [k for k, kind in enumerate(kinds) if kind in (0, 1, 4)]      # codes that name ops
        orders, masks = orders[keep], masks[keep]
        b = Base(di)
        b.record(torch.from_numpy(o0.view(np.int16)).cuda(), torch.from_numpy(mk0.view(np.int32)).cuda())
        enc = delta_encode(o0, mk0, orders, masks)
        assert int(enc[0][-1]) < orders.size // 4          # far fewer entries than the full rows
        for bb in (None, b):
            want = di.evaluate_host(orders, masks, peak=True, base=bb)
            got = di.evaluate_host_delta(o0, mk0, *enc, peak=True, base=bb)
            for f in ("flags", "makespan", "peak", "blocked"):
                assert (getattr(got, f) == getattr(want, f)).all(), (cfg, f)
            ok = want.flags == 1
            assert (got.bubble[ok] == want.bubble[ok]).all()


@pytest.mark.parametrize("cfg", [3, 4, 5])
def test_delta_batch_moves_and_general_candidates(cuda_ok, cfg):
    """ps_eval_batch_host_delta evaluates a candidate that is one move of the reference (a shift's
    rotated run, one offloadable bit, nothing) on the move-encoded kernel and anything else
    materialised.  A batch mixing search neighbours with two-move candidates, wider
    rotations, unsorted entries, a shift plus a flip and malformed rows gives exactly the full-row
    outputs without a base — with the reference's recorded base, with no base, and with a base
    recorded on another structure; an out-of-range entry fails the call."""
    import torch
    from paper_2510_05186_b200 import _native as N
    from paper_2510_05186_b200.engine import Base
    from paper_2510_05186_b200.packing import delta_encode
    from paper_2510_05186_b200.search import LocalSearch, SearchConfig
    from paper_2510_05186_b200.heuristics import best_feasible
    from paper_2510_05186_b200.listsched import stage_order_of
    from paper_2510_05186_b200 import workloads
    inst = workloads.CONFIGS[cfg]()
    s0, _ = best_feasible(inst)
    ls = LocalSearch(inst, {i: stage_order_of(s0, i) for i in range(1, inst.num_stages + 1)}, s0.offloaded,
                     SearchConfig(seed=3, neighbours=512, shift_permille=700, max_shift=4))
    di, pk = ls.di, ls.di.packed
    n = 512 if cfg != 5 else 128
    o, mk = ls.materialize(0, n, 0)
    o = o.cpu().numpy().view(np.uint16).copy()
    mk = mk.cpu().numpy().view(np.uint32).copy()
    ref_o = ls.inc_orders.cpu().numpy().view(np.uint16).copy()
    ref_m = ls.inc_mask.cpu().numpy().view(np.uint32).copy()
    rng = np.random.default_rng(cfg)
    L = 3 * pk.num_microbatches
    extra_o, extra_m = [], []
    for k in range(48):
        a, b = o[k].copy(), mk[k].copy()
        kind = k % 6
        if kind == 0:                       # two moves: this neighbour's and the next one's
            a2 = o[k + 1]
            d = a2 != ref_o
            a[d] = a2[d]
            b ^= mk[k + 1] ^ ref_m
        elif kind == 1:                     # a run rotated by two (not a single move)
            s, q = int(rng.integers(pk.num_stages)), int(rng.integers(L - 3))
            a = ref_o.copy()
            a[s, q:q + 3] = np.roll(ref_o[s, q:q + 3], 2)
            b = ref_m.copy()
        elif kind == 2:                     # a shift and a flipped bit together
            s = int(rng.integers(pk.num_stages))
            a = ref_o.copy()
            a[s, 5:7] = ref_o[s, 5:7][::-1]
            b = ref_m.copy()
            b[0] ^= 1
        elif kind == 3:                     # a repeated op (malformed: literal replay)
            s = int(rng.integers(pk.num_stages))
            a = ref_o.copy()
            a[s, 4] = a[s, 3]
            b = ref_m.copy()
        elif kind == 4:                     # swap of two far positions in one stage
            s = int(rng.integers(pk.num_stages))
            a = ref_o.copy()
            a[s, [2, 9]] = a[s, [9, 2]]
            b = ref_m.copy()
        else:                               # two flipped bits
            a = ref_o.copy()
            b = ref_m.copy()
            b[0] ^= 3
        extra_o.append(a)
        extra_m.append(b)
    orders = np.concatenate([o, np.stack(extra_o)])
    masks = np.concatenate([mk, np.stack(extra_m)])
    want = di.evaluate_host(orders, masks, peak=True, base=None)
    doff, diffs, foff, flips = delta_encode(ref_o, ref_m, orders, masks)
    # the same entries in reverse order within each candidate (unsorted: not classified as moves)
    diffs_rev = diffs.copy()
    for c in range(0, len(orders), 7):
        diffs_rev[doff[c]:doff[c + 1]] = diffs[doff[c]:doff[c + 1]][::-1]
    other = Base(di)
    other.record(torch.from_numpy(orders[n + 4].view(np.int16)).cuda(), torch.from_numpy(masks[n + 4].view(np.int32)).cuda())
    for bb in (ls.base, None, other):
        for dd in (diffs, diffs_rev):
            got = di.evaluate_host_delta(ref_o, ref_m, doff, dd, foff, flips, peak=True, base=bb)
            for f in ("flags", "makespan", "peak", "blocked"):
                assert (getattr(got, f) == getattr(want, f)).all(), (cfg, f, bb is None)
            ok = want.flags == 1
            assert (got.bubble[ok] == want.bubble[ok]).all()
    assert (want.flags == 1).any() and (want.flags == 2).any()
    bad = diffs.copy()
    bad[int(doff[3]), 0] = (pk.num_stages << 16)           # stage out of range
    with pytest.raises(N.NativeError):
        di.evaluate_host_delta(ref_o, ref_m, doff, bad, foff, flips, peak=True, base=ls.base)


def test_explicit_channel_entries_out_of_range_are_malformed(cuda_ok):
    """Explicit channel orders through the C ABI with entries that name a microbatch past m, a
    stage on another channel or an activation that is not offloaded: the candidate is
    PS_FLAG_MALFORMED (no out-of-range state access), its neighbours in the batch are unaffected."""
    import torch
    from paper_2510_05186_b200 import _native as N, workloads
    from paper_2510_05186_b200.heuristics import best_feasible
    from paper_2510_05186_b200.search import ChannelSearch, SearchConfig
    for cfg in (2, 4):
        inst = workloads.CONFIGS[cfg]()
        s, _ = best_feasible(inst)
        cs = ChannelSearch.from_schedule(inst, s, SearchConfig(seed=1, neighbours=64, share_prefix=False))
        o, mk, ch = cs.materialize(0, 8, 0)
        ch = ch.clone()
        m = inst.num_microbatches
        e = int(ch[1, 0, 0].item()) & 0xFFFFFFFF
        ch[1, 0, 0] = torch.tensor(((e & ~0xFFFF) | (m + 3)) - (1 << 32) if (e & ~0xFFFF) | (m + 3) >= 1 << 31
                                   else (e & ~0xFFFF) | (m + 3), dtype=torch.int32)          # microbatch past m
        other = 1 if cs.di.packed.num_channels > 1 else 0
        e2 = int(ch[2, other, 0].item()) & 0xFFFFFFFF
        ch[2, 0, 0] = torch.tensor(e2 - (1 << 32) if e2 >= 1 << 31 else e2, dtype=torch.int32)  # stage of another channel
        mk = mk.clone()
        st, j = (e >> 16) & 0x7FFF, e & 0xFFFF
        b = st * m + j
        mk[3, b >> 5] ^= torch.tensor((1 << (b & 31)) - (1 << 32) if (b & 31) == 31 else 1 << (b & 31),
                                      dtype=torch.int32)                                     # not offloaded
        r = cs.di.evaluate(o, mk, ch, peak=False)
        torch.cuda.synchronize()
        flags = r.flags.cpu().numpy()
        assert flags[1] == N.FLAG_MALFORMED and flags[3] == N.FLAG_MALFORMED, (cfg, flags)
        if other:
            assert flags[2] == N.FLAG_MALFORMED, (cfg, flags)
        good = [0] + list(range(4, 8))
        r0 = cs.di.evaluate(o[good], mk[good], ch[good], peak=False)
        torch.cuda.synchronize()
        assert (r0.flags.cpu().numpy() == flags[good]).all()
        assert (r0.makespan.cpu().numpy() == r.makespan.cpu().numpy()[good]).all()


@pytest.mark.parametrize("m", [1024, 1280])
def test_search_rounds_at_the_stage_limit(cuda_ok, m):
    """P = 32 (PS_MAX_STAGES) with a long incumbent: at m = 1024 the move-encoded kernel runs with
    one-warp blocks (the incumbent takes 196 KB of shared memory); at m = 1280 it no longer fits and
    the round materialises its neighbours. Every neighbour's makespan, the round's
    best key and the delta-encoded host batch of the same neighbours against the oracle."""
    import torch
    from oracle.oracle import Oracle
    from paper_2510_05186_b200 import make_uniform_instance
    from paper_2510_05186_b200.heuristics import generator_structures
    from paper_2510_05186_b200.packing import delta_encode
    from paper_2510_05186_b200.search import LocalSearch, SearchConfig
    inst = make_uniform_instance(32, m, 3, 2, 2, 1, 4, 2, 6)
    o, f = generator_structures(inst)[-1]
    n = 16
    ls = LocalSearch(inst, o, f, SearchConfig(seed=5, neighbours=n, shift_permille=700, max_shift=4))
    inc_o = ls.inc_orders.cpu().numpy().view(np.uint16).copy()
    inc_m = ls.inc_mask.cpu().numpy().view(np.uint32).copy()
    ms = torch.empty(n, dtype=torch.int64, device="cuda")
    ls.launch_round(ms)
    torch.cuda.synchronize()
    best, want = Oracle(ls.di.packed).search_round(inc_o, inc_m, 5, 700, 4, 0, 0, n, want_makespans=True)
    assert (ms.cpu().numpy() == want).all()
    assert int(ls.best_key.item()) == best
    mo, mm = ls.materialize(0, n, 0)
    d = delta_encode(inc_o, inc_m, mo.cpu().numpy().view(np.uint16), mm.cpu().numpy().view(np.uint32))
    r = ls.di.evaluate_host_delta(inc_o, inc_m, *d, peak=False, base=ls.base)
    assert (np.asarray(r.makespan) == want).all()
