"""Load the reference-generated fixtures in tests/golden (see make_golden.py)."""

import gzip
import json
from functools import lru_cache
from pathlib import Path

import numpy as np

from paper_2510_05186_b200.instance import OpId, OpKind, instance_from_dict
from paper_2510_05186_b200.packing import PAD_CHANNEL, pack_instance

GOLDEN = Path(__file__).resolve().parent / "golden"
CORPORA = ("ref_tests", "fuzz", "configs", "random")
MALFORMED = "malformed"


@lru_cache(maxsize=None)
def load_raw(name):
    with gzip.open(GOLDEN / f"{name}.json.gz", "rt") as fh:
        return json.load(fh)


def corpus(name):
    """[(instance, packed, [case, ...]), ...] with our own instance model."""
    out = []
    for e in load_raw(name)["instances"]:
        inst = instance_from_dict(e["instance"])
        out.append((inst, pack_instance(inst), e["cases"]))
    return out


def case_arrays(pk, case):
    P, m = pk.num_stages, pk.num_microbatches
    orders = np.zeros((P, pk.order_stride), np.uint16)
    for i, row in enumerate(case["orders"]):
        orders[i, :len(row)] = row
        if len(row) < 3 * m:
            orders[i, len(row)] = 0xFFFF          # short row: terminator (PS_ROW_END)
    mask = np.zeros(pk.mask_words, np.uint32)
    for i, j in case["offloaded"]:
        b = (i - 1) * m + (j - 1)
        mask[b >> 5] |= np.uint32(1 << (b & 31))
    chans = None
    if "channel_orders" in case:
        width = max([len(c) for c in case["channel_orders"]] + [1])
        chans = np.full((pk.num_channels, width), PAD_CHANNEL, np.uint32)
        for g, seq in enumerate(case["channel_orders"]):
            for q, (i, j, rel) in enumerate(seq):
                chans[g, q] = (rel << 31) | ((i - 1) << 16) | (j - 1)
    return orders, mask, chans


def structure(case):
    """Case -> (stage_orders dict of OpId, offloaded frozenset, channel_orders or None)."""
    from paper_2510_05186_b200.schedule import TransferKind
    orders = {i + 1: tuple(OpId(i + 1, (c >> 2) + 1, OpKind(c & 3)) for c in row)
              for i, row in enumerate(case["orders"])}
    off = frozenset(OpId(i, j, OpKind.F) for i, j in case["offloaded"])
    chans = None
    if "channel_orders" in case:
        chans = {g: tuple((OpId(i, j, OpKind.F), TransferKind.RELOAD if rel else TransferKind.OFFLOAD)
                          for i, j, rel in seq)
                 for g, seq in enumerate(case["channel_orders"])}
    return orders, off, chans


def split_trace(codes, starts):
    """Commit-ordered trace -> (compute [[i,j,k,start]], transfers [[i,j,reload,start]]) 1-based."""
    comp, tr = [], []
    for c, t in zip(codes, starts):
        c = int(c) & 0xFFFFFFFF
        rank, i, j, k = c >> 30, ((c >> 24) & 63) + 1, ((c >> 2) & 0x3FFFFF) + 1, c & 3
        if rank == 0:
            comp.append([i, j, k, int(t)])
        else:
            tr.append([i, j, 1 if rank == 1 else 0, int(t)])
    return comp, tr
