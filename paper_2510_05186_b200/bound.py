"""Batched branch-and-bound node lower bounds on the GPU.

The reference's depth-first branch-and-bound bounds one node at a time in Python
(``_Search._bound``, solver.py:352-383, with ``_chain_ends``, solver.py:321-350).  Here a whole
frontier of nodes is bounded in one launch of the sm_100a kernel behind
``ps_bound_batch_eval`` (one warp per node), with the same value the reference computes: the
tests pin it against bounds recorded from the reference solver itself
(tests/golden/bounds.json.gz).

A node is the state the reference bound reads: the clock, the stage free times and the committed
compute starts.  ``lower_bounds`` takes them in the reference's own form (``stage_free`` keyed by
1-based stage, ``comp_start`` keyed by ``OpId``); ``BoundEvaluator.bounds`` takes dense device
tensors.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
from .engine import _ptr, device_instance


def node_arrays(inst, nodes):
    """Dense int32 tables of reference-style nodes: clock [N], stage_free [N][P], starts
    [N][P][m][3] (-1 = not committed).  `nodes`: iterable of (clock, stage_free, comp_start)."""
    P, m = inst.num_stages, inst.num_microbatches
    nodes = list(nodes)
    clock = np.zeros(len(nodes), np.int32)
    sfree = np.zeros((len(nodes), P), np.int32)
    start = np.full((len(nodes), P, m, 3), -1, np.int32)
    for n, (t, sf, comp) in enumerate(nodes):
        clock[n] = t
        for i in range(1, P + 1):
            sfree[n, i - 1] = sf[i]
        for op, s in comp.items():
            start[n, op.stage - 1, op.microbatch - 1, int(op.kind)] = s
    return clock, sfree, start


class BoundEvaluator:
    """Lower bounds for batches of nodes of one instance on one device."""

    def __init__(self, inst, device=None):
        self.inst = inst
        self.di = device_instance(inst, device)

    def bounds(self, clock, stage_free, comp_start, out=None, stream=None):
        """Device tensors in (int32 [N], [N][P], [N][P][m][3]), device int64 [N] out; async."""
        import torch
        n = int(clock.shape[0])
        if out is None:
            out = torch.empty(n, dtype=torch.int64, device=clock.device)
        b = N.BoundBatch(n, _ptr(clock), _ptr(stage_free), _ptr(comp_start))
        N.check(self.di.lib.ps_bound_batch_eval(self.di.handle, C.byref(b), C.c_void_p(out.data_ptr()),
                                                self.di._stream(stream)))
        return out


def lower_bounds(inst, nodes, device=None) -> list[int]:
    """Reference-style nodes -> their bounds, as solver._Search._bound returns them."""
    import torch
    clock, sfree, start = node_arrays(inst, nodes)
    ev = BoundEvaluator(inst, device)
    dev = torch.device("cuda", ev.di.device)
    out = ev.bounds(torch.from_numpy(clock).to(dev), torch.from_numpy(sfree).to(dev),
                    torch.from_numpy(start).to(dev))
    return [int(x) for x in out.cpu().tolist()]
