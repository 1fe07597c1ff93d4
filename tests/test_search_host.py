"""Host-side logic of the sharded local search, multi-process on CPU (gloo, world size 2).

The neighbour evaluations here come from the CPU oracle (test infrastructure) standing in for
each rank's GPU shard; what is under test is the product's sharding, key packing, MIN
all-reduce and strict-improvement acceptance (paper_2510_05186_b200/search.py).
"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2510_05186_b200.search import combine_keys, improves, pack_key, shard_range, unpack_key

SEED, PERMILLE, MAXSHIFT = 7, 700, 4


def test_shards_partition_the_index_space():
    for total in (1, 7, 4096, 65536):
        for world in (1, 2, 3, 4, 8):
            seen = []
            for r in range(world):
                first, count = shard_range(total, r, world)
                seen.extend(range(first, first + count))
            assert seen == list(range(total))


def test_key_order_is_makespan_then_lowest_index():
    assert pack_key(10, 5) < pack_key(10, 6) < pack_key(11, 0)
    assert unpack_key(pack_key(123456, 4242)) == (123456, 4242)
    assert improves(pack_key(9, 3), 10) and not improves(pack_key(10, 3), 10)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _small_problem():
    from paper_2510_05186_b200 import make_uniform_instance
    from paper_2510_05186_b200.heuristics import generator_structures
    from paper_2510_05186_b200.packing import encode_candidate, pack_instance
    inst = make_uniform_instance(4, 8, 2, 2, 1, 1, 3, 2, 3)
    pk = pack_instance(inst)
    o, f = generator_structures(inst)[0]
    orders, mask, _ = encode_candidate(pk, o, f)
    return pk, orders, mask


def _rank_main(rank, world, port, total, rounds, out):
    import torch
    import torch.distributed as dist
    from oracle.oracle import Oracle
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    pk, inc_o, inc_m = _small_problem()
    orc = Oracle(pk)
    span = orc.run(inc_o, inc_m)["makespan"]
    first, count = shard_range(total, rank, world)
    trail = []
    for rnd in range(rounds):
        best, _ = orc.search_round(inc_o, inc_m, SEED, PERMILLE, MAXSHIFT, rnd, first, count, threads=1)
        key = torch.tensor([best], dtype=torch.int64)
        combine_keys(key)
        k = int(key.item())
        if improves(k, span):
            span, idx = unpack_key(k)
            _, inc_o, inc_m = orc.neighbour(inc_o, inc_m, SEED, PERMILLE, MAXSHIFT, rnd, idx)
        trail.append((k, span))
    out[rank] = (trail, inc_o.tobytes(), inc_m.tobytes())
    dist.destroy_process_group()


def _run(world, total=256, rounds=4):
    ctx = mp.get_context("spawn")
    out = ctx.Manager().dict()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, total, rounds, out)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    return dict(out)


@pytest.mark.timeout(300)
def test_sharded_search_selects_the_same_incumbent_at_world_1_and_2():
    one = _run(1)
    two = _run(2)
    assert one[0][0] == two[0][0] == two[1][0]           # same keys and spans every round
    assert one[0][1] == two[0][1] == two[1][1]           # identical final structure on every rank
    assert one[0][2] == two[0][2]
    assert any(k != (1 << 63) - 1 for k, _ in one[0][0])
