"""The five BASELINE.json configurations as synthetic instances.

All values are integer quanta (microseconds) and integer bytes.  Per-stage
values are constant across microbatches, the reference convention
(instance.py:325-327).  Every instance is also loadable by the reference via
``instance_to_dict`` / ``instance_from_dict``.
"""

from __future__ import annotations

from random import Random

from .instance import PipelineInstance, _per_stage_instance, make_uniform_instance

MIB = 1 << 20


def config1() -> PipelineInstance:
    """4 stages x 8 microbatches, uniform F/B/W, B/W split, nothing offloadable."""
    base = make_uniform_instance(4, 8, 2, 2, 1, 1, 1, 2, 8)
    return PipelineInstance(
        num_stages=4, num_microbatches=8, proc_time=base.proc_time, comm_time=base.comm_time,
        offload_time=base.offload_time, mem_delta=base.mem_delta, act_size={},
        mem_limit=base.mem_limit, topology_groups=base.topology_groups)


def config2() -> PipelineInstance:
    """8 x 32 zero-bubble B/W split, per-stage cap of 4 activations, 64 MiB activations."""
    return make_uniform_instance(8, 32, 100, 100, 100, 5, 150, 64 * MIB, 4)


# Llama-style 7B on 8 stages: 32 layers -> 4 per stage, h=4096, s=4096, microbatch 1, bf16.
LLAMA7B_ACT = 34 * 4096 * 4096 * 4          # 2,281,701,376 B of activations per stage per microbatch
LLAMA7B_TF, LLAMA7B_TB, LLAMA7B_TW = 16000, 16500, 15500
LLAMA7B_HEAD = 2300                         # LM head on the last stage, per op
LLAMA7B_OFFLOAD = 45600                     # act / ~50 GB/s PCIe Gen5 x16 effective, in us
LLAMA7B_COMM = 84


def config3() -> PipelineInstance:
    """Llama-style 7B, 8 x 64, PCIe-bandwidth-limited offload, limit 4 activations per stage."""
    P, m = 8, 64
    rows = []
    for i in range(1, P + 1):
        extra = LLAMA7B_HEAD if i == P else 0
        rows.append((LLAMA7B_TF + extra, LLAMA7B_TB + extra, LLAMA7B_TW + extra, LLAMA7B_ACT))
    return _per_stage_instance(P, m, rows, LLAMA7B_COMM, LLAMA7B_OFFLOAD, [4 * LLAMA7B_ACT] * P,
                               None, False)


def config4() -> PipelineInstance:
    """Interleaved v=2 encoding, 16 x 128: virtual stages d and d+8 share device d's host link
    (topology group); each virtual stage gets half the time and half the activation of a full
    stage and half of a tight 6-activation device budget."""
    P, m = 16, 128
    act = LLAMA7B_ACT // 2
    rows = [(LLAMA7B_TF // 2, LLAMA7B_TB // 2, LLAMA7B_TW // 2, act)] * P
    groups = [[d, d + 8] for d in range(1, 9)]
    return _per_stage_instance(P, m, rows, LLAMA7B_COMM, LLAMA7B_OFFLOAD // 2, [3 * act] * P,
                               groups, False)


def config5(seed: int = 5) -> PipelineInstance:
    """32 x 256 sweep: seeded per-stage times in [50, 200] us, activations in [32, 128] MiB,
    cap 3-6 activations per stage."""
    P, m = 32, 256
    rng = Random(seed)
    rows, limits = [], []
    for _ in range(P):
        act = rng.randint(32, 128) * MIB
        rows.append((rng.randint(50, 200), rng.randint(50, 200), rng.randint(50, 200), act))
        limits.append(rng.randint(3, 6) * act)
    return _per_stage_instance(P, m, rows, 5, 100, limits, None, False)


CONFIGS = {1: config1, 2: config2, 3: config3, 4: config4, 5: config5}
CANDIDATES_PER_ROUND = {1: 4096, 2: 4096, 3: 65536, 4: 16384, 5: 131072}
