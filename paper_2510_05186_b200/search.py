"""GPU local search over candidate structures.

One round evaluates ``neighbours`` moves of the incumbent — each decoded on the
device from Philox4x32-10 keyed by (seed, round, global index), DESIGN.md §4
— with the evaluator kernel, folds ``(makespan << 32 | index)`` of every
feasible neighbour into one int64 key with an atomic min, combines the key
across ranks with one NCCL all-reduce(MIN) of 8 bytes, and applies the winning
move in place on every rank when it strictly improves the incumbent.  The
candidate set of a round is identical at 1/2/4/8 GPUs (ranks own contiguous
index ranges) and the lowest index wins ties, so the selected schedule is
the same for every GPU count.

The winner feeds the reference solver API unchanged: ``SearchResult.schedule``
is a valid warm start for ``start_session(warm=...)`` (solver.py:543-565), and
``incumbent_events`` lists every strict improvement with its timestamp
(the IncumbentEvent stream of solver.py:81-87, 435-449).
"""

from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .engine import Base, device_instance
from .packing import decode_mask, decode_orders, encode_candidate


@dataclass(frozen=True)
class SearchConfig:
    seed: int = 0
    neighbours: int = 65536          # per round, all ranks together
    shift_permille: int = 700        # SHIFT moves; the rest toggle offload bits
    max_shift: int = 4
    share_prefix: bool = True        # resume neighbours from checkpoints of the incumbent
    dedup: bool = True               # simulate a move drawn several times in a round once
    prune: bool = False              # abandon neighbours that provably cannot improve (
                                     # same trail, measured no faster: off by default)
    # Iterated local search: after `descent_patience` rounds without improving
    # the current point, restart the descent from the best structure kicked by `kick_moves`
    # random moves.  0 = plain descent (a run then ends at convergence or its budget).
    kick_moves: int = 0
    descent_patience: int = 16


KICK_ROUND_BASE = 1 << 40            # kick k draws its moves from "round" KICK_ROUND_BASE + k
KICK_TRIES = 64                      # move draws per kick move before the kick gives up


@dataclass
class Improvement:
    round: int
    makespan: int
    timestamp: float                 # seconds since the search started
    index: int


@dataclass
class SearchResult:
    schedule: object
    makespan: int
    initial_makespan: int
    rounds: int
    evaluated: int
    elapsed: float
    improvements: list = field(default_factory=list)

    def incumbent_events(self):
        return [(imp.timestamp, imp.makespan) for imp in self.improvements]


def shard_range(total: int, rank: int, world: int):
    """Contiguous global-index range [first, first + count) owned by `rank`."""
    lo = total * rank // world
    hi = total * (rank + 1) // world
    return lo, hi - lo


def pack_key(makespan: int, index: int) -> int:
    """(makespan << 32 | index): the minimum is the best makespan, lowest index on ties."""
    return (int(makespan) << 32) | (int(index) & 0xFFFFFFFF)


def unpack_key(key: int):
    return key >> 32, key & 0xFFFFFFFF


def combine_keys(key_tensor, group=None):
    """All-reduce(MIN) of each rank's best key: one 8-byte collective per round (NCCL on GPUs)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(key_tensor, op=dist.ReduceOp.MIN, group=group)
    return key_tensor


def nccl_comm_ptr(group=None, device=None) -> int | None:
    """The ncclComm_t behind a torch.distributed NCCL process group (created on first use), for
    ps_search_round_sharded; None for other backends or when torch does not expose it."""
    import torch
    import torch.distributed as dist
    try:
        if dist.get_backend(group) != "nccl":
            return None
        pg = group if group is not None else dist.distributed_c10d._get_default_group()
        dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        warm = torch.zeros(1, dtype=torch.int64, device=dev)
        dist.all_reduce(warm, group=group)          # the communicator exists after a first collective
        torch.cuda.synchronize(dev)
        ptr = int(pg._get_backend(dev)._comm_ptr())
        return ptr or None
    except Exception:
        return None


def agree_stop(stop: bool, device, group=None) -> bool:
    """The ranks' joint stop decision: stop when ANY rank wants to.  Wall-clock budgets are read
    on each rank's own clock, so without this one rank could leave the loop while another enters
    one more round and blocks in its all-reduce.  One 4-byte all-reduce(MAX); a no-op at world 1."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1):
        return stop
    backend = dist.get_backend(group)
    dev = torch.device("cuda", device) if backend == "nccl" else torch.device("cpu")
    flag = torch.tensor([1 if stop else 0], dtype=torch.int32, device=dev)
    dist.all_reduce(flag, op=dist.ReduceOp.MAX, group=group)
    return bool(flag.item())


def improves(key: int, incumbent_makespan: int) -> bool:
    """Only strict improvements replace the incumbent (solver.py:437 convention)."""
    return key != N.BEST_NONE and unpack_key(key)[0] < incumbent_makespan


class LocalSearch:
    def __init__(self, inst, stage_orders, offloaded, config: SearchConfig = SearchConfig(),
                 device=None, group=None):
        import torch
        import torch.distributed as dist
        self.inst = inst
        self.cfg = config
        self.di = device_instance(inst, device)
        self.lib = self.di.lib
        pk = self.di.packed
        o, mk, _ = encode_candidate(pk, stage_orders, offloaded)
        dev = torch.device("cuda", self.di.device)
        self.inc_orders = torch.from_numpy(o.view(np.int16).copy()).to(dev)
        self.inc_mask = torch.from_numpy(mk.view(np.int32).copy()).to(dev)
        self.best_key = torch.empty(1, dtype=torch.int64, device=dev)
        self.group = group
        self.distributed = dist.is_available() and dist.is_initialized()
        self.rank = dist.get_rank(group) if self.distributed else 0
        self.world = dist.get_world_size(group) if self.distributed else 1
        self.first, self.count = shard_range(config.neighbours, self.rank, self.world)
        # over NCCL the round's 8-byte all-reduce(MIN) runs inside the C ABI call
        # (ps_search_round_sharded) on the torch group's communicator; other backends combine
        # the key with torch.distributed
        self.nccl_comm = nccl_comm_ptr(group, self.di.device) if self.world > 1 else None
        self.moves = N.MoveParams(config.seed & (2**64 - 1), config.shift_permille, config.max_shift)
        res = self.di.evaluate(self.inc_orders.view(1, *self.inc_orders.shape),
                               self.inc_mask.view(1, -1), peak=False)
        if not int(res.flags[0].item()) & N.FLAG_FEASIBLE:
            raise ValueError("the incumbent structure is not feasible")
        self.makespan = int(res.makespan[0].item())
        self.initial_makespan = self.makespan
        self.base = Base(self.di) if config.share_prefix else None
        if self.base is not None:
            self.base.record(self.inc_orders, self.inc_mask)
        self.round = 0
        self.evaluated = 0
        self.improvements = []
        # best structure so far (differs from the current point only after an ILS kick)
        self.best_makespan = self.makespan
        self.best_orders = self.inc_orders.clone()
        self.best_mask = self.inc_mask.clone()
        self.kicks = 0
        self.stale = 0               # rounds since the current point last improved
        # with keep_structures, (orders, mask) device copies of the best at every improvement
        self.keep_structures = False
        self.improvement_structures = []

    def _stream(self):
        import torch
        return C.c_void_p(torch.cuda.current_stream(self.di.device).cuda_stream)

    def launch_round(self, makespan_out=None):
        """Enqueue one round's generate + evaluate + argmin (no host sync)."""
        self.best_key.fill_(N.BEST_NONE)
        desc = N.SearchDesc(self.inc_orders.data_ptr(), self.inc_mask.data_ptr(), self.round,
                            self.first, self.count, self.moves, None,
                            self.base.handle if self.base is not None else None, int(self.cfg.dedup),
                            self.makespan if self.cfg.prune and makespan_out is None else 0)
        ms = C.c_void_p(makespan_out.data_ptr()) if makespan_out is not None else None
        if self.nccl_comm:
            N.check(self.lib.ps_search_round_sharded(self.di.handle, C.byref(desc), C.c_void_p(self.best_key.data_ptr()),
                                                     ms, C.c_void_p(self.nccl_comm), self._stream()))
            return
        N.check(self.lib.ps_search_round(self.di.handle, C.byref(desc), C.c_void_p(self.best_key.data_ptr()),
                                         ms, self._stream()))
        if self.world > 1:
            combine_keys(self.best_key, self.group)

    def finish_round(self, t0=None) -> bool:
        """Read the combined key (host sync) and adopt a strict improvement of the current point;
        an improvement of the best so far is recorded in `improvements`."""
        key = int(self.best_key.item())
        r = self.round
        self.round += 1
        self.evaluated += self.cfg.neighbours
        if not improves(key, self.makespan):
            self.stale += 1
            return False
        self.stale = 0
        span, idx = unpack_key(key)
        N.check(self.lib.ps_apply_move(self.di.handle, C.c_void_p(self.inc_orders.data_ptr()),
                                       C.c_void_p(self.inc_mask.data_ptr()), C.byref(self.moves),
                                       r, idx, self._stream()))
        if self.base is not None:
            self.base.record(self.inc_orders, self.inc_mask)
        self.makespan = span
        if span < self.best_makespan:
            self.best_makespan = span
            self.best_orders.copy_(self.inc_orders)
            self.best_mask.copy_(self.inc_mask)
            self.improvements.append(Improvement(r, span, (time.perf_counter() - t0) if t0 else 0.0, idx))
            if self.keep_structures:
                self.improvement_structures.append((self.best_orders.clone(), self.best_mask.clone()))
        return True

    def kick(self) -> int:
        """ILS restart: the current point becomes the best structure with up to
        `kick_moves` random moves applied — kick k applies the moves of "round"
        KICK_ROUND_BASE + k, neighbour indices 0, 1, ... in turn, keeping each one whose result is
        still feasible, until kick_moves are kept or KICK_TRIES * kick_moves were drawn.  Returns
        the current point's makespan.  Deterministic: every rank kicks identically."""
        k = self.cfg.kick_moves
        self.inc_orders.copy_(self.best_orders)
        self.inc_mask.copy_(self.best_mask)
        save_o, save_m = self.inc_orders.clone(), self.inc_mask.clone()
        span, kept, tries = self.best_makespan, 0, 0
        rnd = KICK_ROUND_BASE + self.kicks
        while kept < k and tries < KICK_TRIES * k:
            N.check(self.lib.ps_apply_move(self.di.handle, C.c_void_p(self.inc_orders.data_ptr()),
                                           C.c_void_p(self.inc_mask.data_ptr()), C.byref(self.moves),
                                           rnd, tries, self._stream()))
            tries += 1
            res = self.di.evaluate(self.inc_orders.view(1, *self.inc_orders.shape), self.inc_mask.view(1, -1),
                                   peak=False)
            if int(res.flags[0].item()) & N.FLAG_FEASIBLE:
                kept += 1
                span = int(res.makespan[0].item())
                save_o.copy_(self.inc_orders)
                save_m.copy_(self.inc_mask)
            else:
                self.inc_orders.copy_(save_o)
                self.inc_mask.copy_(save_m)
        self.kicks += 1
        self.makespan = span
        self.stale = 0
        if self.base is not None:
            self.base.record(self.inc_orders, self.inc_mask)
        return span

    def should_stop(self, local_stop: bool) -> bool:
        """Collective stop decision (agree_stop) over this search's process group."""
        return agree_stop(local_stop, self.di.device, self.group) if self.world > 1 else local_stop

    def step(self, t0=None) -> bool:
        self.launch_round()
        return self.finish_round(t0)

    def incumbent_structure(self):
        """The best structure found so far (stage orders, offloaded set)."""
        pk = self.di.packed
        o = self.best_orders.cpu().numpy().view(np.uint16)
        mk = self.best_mask.cpu().numpy().view(np.uint32)
        return decode_orders(pk, o), decode_mask(pk, mk)

    def step_ils(self, t0=None) -> bool:
        """One ILS step: a descent round, or a kick when the descent has converged."""
        if self.cfg.kick_moves > 0 and self.stale >= self.cfg.descent_patience:
            self.kick()
            return False
        return self.step(t0)

    def run(self, rounds: int | None = None, time_budget: float | None = None,
            patience: int | None = None, kicks: int | None = None) -> SearchResult:
        """Rounds until `rounds`, `time_budget` seconds, `patience` rounds without improving the
        best, or (ILS, kick_moves > 0) `kicks` restarts."""
        from .listsched import run_order
        if rounds is None and time_budget is None and patience is None and kicks is None:
            raise ValueError("need rounds, time_budget, patience or kicks")
        if kicks and self.cfg.kick_moves <= 0:
            raise ValueError("a kick budget needs SearchConfig.kick_moves > 0")
        t0 = time.perf_counter()
        since_best = 0               # steps (rounds and kicks) since the best last improved
        while True:
            if rounds is not None and self.round >= rounds:
                break
            # (a kick budget ends once the descent after the last kick has converged)
            if kicks is not None and self.kicks >= kicks and self.stale >= self.cfg.descent_patience:
                break
            if time_budget is not None and self.should_stop(time.perf_counter() - t0 >= time_budget):
                break
            best_before = self.best_makespan
            self.step_ils(t0)
            since_best = 0 if self.best_makespan < best_before else since_best + 1
            if patience is not None and since_best >= patience:
                break
        elapsed = time.perf_counter() - t0
        orders, off = self.incumbent_structure()
        sched = run_order(self.inst, orders, off, device=self.di.device)
        return SearchResult(sched, self.best_makespan, self.initial_makespan, self.round, self.evaluated,
                            elapsed, list(self.improvements))

    # -- checkpoint / resume: the search state is the incumbent, the round and the
    # improvement trail; the base recording is rebuilt from the incumbent on load
    def state_dict(self) -> dict:
        return {"inc_orders": self.inc_orders.cpu().numpy().view(np.uint16).copy(),
                "inc_mask": self.inc_mask.cpu().numpy().view(np.uint32).copy(),
                "best_orders": self.best_orders.cpu().numpy().view(np.uint16).copy(),
                "best_mask": self.best_mask.cpu().numpy().view(np.uint32).copy(),
                "round": self.round, "makespan": self.makespan, "initial_makespan": self.initial_makespan,
                "best_makespan": self.best_makespan, "kicks": self.kicks, "stale": self.stale,
                "evaluated": self.evaluated, "config": dict(self.cfg.__dict__),
                "improvements": [(i.round, i.makespan, i.timestamp, i.index) for i in self.improvements]}

    def load_state_dict(self, state: dict) -> None:
        import torch
        if dict(state["config"]) != dict(self.cfg.__dict__):
            raise ValueError("state was saved under another SearchConfig")
        self.inc_orders.copy_(torch.from_numpy(np.asarray(state["inc_orders"], np.uint16).view(np.int16)))
        self.inc_mask.copy_(torch.from_numpy(np.asarray(state["inc_mask"], np.uint32).view(np.int32)))
        self.round = int(state["round"])
        self.makespan = int(state["makespan"])
        self.initial_makespan = int(state["initial_makespan"])
        self.evaluated = int(state["evaluated"])
        self.improvements = [Improvement(r, m, t, i) for r, m, t, i in state["improvements"]]
        self.best_orders.copy_(torch.from_numpy(np.asarray(state.get("best_orders", state["inc_orders"]),
                                                           np.uint16).view(np.int16)))
        self.best_mask.copy_(torch.from_numpy(np.asarray(state.get("best_mask", state["inc_mask"]),
                                                         np.uint32).view(np.int32)))
        self.best_makespan = int(state.get("best_makespan", self.makespan))
        self.kicks = int(state.get("kicks", 0))
        self.stale = int(state.get("stale", 0))
        if self.base is not None:
            self.base.record(self.inc_orders, self.inc_mask)

    def materialize(self, first: int, count: int, rnd: int | None = None):
        """Neighbours [first, first+count) of round `rnd` as full candidate tensors (for parity)."""
        import torch
        pk = self.di.packed
        dev = self.inc_orders.device
        orders = torch.empty((count, pk.num_stages, pk.order_stride), dtype=torch.int16, device=dev)
        masks = torch.empty((count, pk.mask_words), dtype=torch.int32, device=dev)
        desc = N.SearchDesc(self.inc_orders.data_ptr(), self.inc_mask.data_ptr(),
                            self.round if rnd is None else rnd, first, count, self.moves)
        N.check(self.lib.ps_materialize_moves(self.di.handle, C.byref(desc), C.c_void_p(orders.data_ptr()),
                                              C.c_void_p(masks.data_ptr()), self._stream()))
        return orders, masks


def warm_start_search(inst, config: SearchConfig = SearchConfig(), rounds=None, time_budget=None,
                      patience=None, device=None, group=None):
    """best_feasible warm start, then GPU local search; returns SearchResult."""
    from .heuristics import best_feasible
    from .listsched import stage_order_of
    s, _ = best_feasible(inst, device=device)
    orders = {i: stage_order_of(s, i) for i in range(1, inst.num_stages + 1)}
    ls = LocalSearch(inst, orders, s.offloaded, config, device=device, group=group)
    return ls.run(rounds=rounds, time_budget=time_budget, patience=patience)


class ChannelSearch:
    """The channel-order search: the incumbent carries explicit per-channel
    transfer orders, replayed in explicit channel mode (listsched.py:233-239), and a neighbour
    shifts either one op of a stage order or one transfer — a reload or an offload — within its
    channel's order (``ps_search_round_explicit``).  Offload bits stay fixed.  Start it from a
    timed schedule (``from_schedule``): its channel orders replay it exactly.  Same selection
    rules as LocalSearch (lowest index on ties, strict improvement), no prefix sharing."""

    def __init__(self, inst, stage_orders, offloaded, channel_orders, config: SearchConfig = SearchConfig(),
                 device=None):
        import torch
        from .packing import encode_candidate
        self.inst = inst
        self.cfg = config
        self.di = device_instance(inst, device)
        self.lib = self.di.lib
        pk = self.di.packed
        o, mk, ch = encode_candidate(pk, stage_orders, offloaded, channel_orders)
        # room for every channel's transfers (2 per offloaded F of its stages)
        width = max([ch.shape[1]] + [1])
        dev = torch.device("cuda", self.di.device)
        self.chan_stride = int(width)
        self.inc_orders = torch.from_numpy(o.view(np.int16).copy()).to(dev)
        self.inc_mask = torch.from_numpy(mk.view(np.int32).copy()).to(dev)
        self.inc_chan = torch.from_numpy(np.ascontiguousarray(ch).view(np.int32).copy()).to(dev)
        self.best_key = torch.empty(1, dtype=torch.int64, device=dev)
        self.moves = N.MoveParams(config.seed & (2**64 - 1), config.shift_permille, config.max_shift)
        res = self.di.evaluate(self.inc_orders.view(1, *self.inc_orders.shape), self.inc_mask.view(1, -1),
                               self.inc_chan.view(1, *self.inc_chan.shape), peak=False)
        if not int(res.flags[0].item()) & N.FLAG_FEASIBLE:
            raise ValueError("the incumbent structure is not feasible in explicit channel mode")
        self.makespan = int(res.makespan[0].item())
        self.initial_makespan = self.makespan
        self.round = 0
        self.evaluated = 0
        self.improvements = []
        # the incumbent recorded with its channel orders: neighbours resume from its checkpoints
        self.base = None
        if config.share_prefix:
            from .engine import Base
            self.base = Base(self.di)
            self.base.record_explicit(self.inc_orders, self.inc_mask, self.inc_chan)

    @classmethod
    def from_schedule(cls, inst, schedule, config: SearchConfig = SearchConfig(), device=None):
        from .listsched import channel_order_of, stage_order_of
        orders = {i: stage_order_of(schedule, i) for i in range(1, inst.num_stages + 1)}
        chans = {g: channel_order_of(schedule, inst, g) for g in range(len(inst.topology_groups))}
        return cls(inst, orders, schedule.offloaded, chans, config, device)

    def _stream(self):
        import torch
        return C.c_void_p(torch.cuda.current_stream(self.di.device).cuda_stream)

    def launch_round(self, makespan_out=None, first=0, count=None):
        count = self.cfg.neighbours if count is None else count
        self.best_key.fill_(N.BEST_NONE)
        desc = N.SearchDesc(self.inc_orders.data_ptr(), self.inc_mask.data_ptr(), self.round, first, count,
                            self.moves, None, self.base.handle if self.base is not None else None, 0)
        N.check(self.lib.ps_search_round_explicit(
            self.di.handle, C.byref(desc), C.c_void_p(self.inc_chan.data_ptr()), self.chan_stride,
            C.c_void_p(self.best_key.data_ptr()),
            C.c_void_p(makespan_out.data_ptr()) if makespan_out is not None else None, self._stream()))

    def step(self, t0=None) -> bool:
        self.launch_round()
        key = int(self.best_key.item())
        r = self.round
        self.round += 1
        self.evaluated += self.cfg.neighbours
        if not improves(key, self.makespan):
            return False
        span, idx = unpack_key(key)
        N.check(self.lib.ps_apply_move_explicit(self.di.handle, C.c_void_p(self.inc_orders.data_ptr()),
                                                C.c_void_p(self.inc_chan.data_ptr()), self.chan_stride,
                                                C.byref(self.moves), r, idx, self._stream()))
        if self.base is not None:
            self.base.record_explicit(self.inc_orders, self.inc_mask, self.inc_chan)
        self.makespan = span
        self.improvements.append(Improvement(r, span, (time.perf_counter() - t0) if t0 else 0.0, idx))
        return True

    def materialize(self, first: int, count: int, rnd: int | None = None):
        import torch
        pk = self.di.packed
        dev = self.inc_orders.device
        orders = torch.empty((count, pk.num_stages, pk.order_stride), dtype=torch.int16, device=dev)
        masks = torch.empty((count, pk.mask_words), dtype=torch.int32, device=dev)
        chans = torch.empty((count, pk.num_channels, self.chan_stride), dtype=torch.int32, device=dev)
        desc = N.SearchDesc(self.inc_orders.data_ptr(), self.inc_mask.data_ptr(),
                            self.round if rnd is None else rnd, first, count, self.moves)
        N.check(self.lib.ps_materialize_moves_explicit(
            self.di.handle, C.byref(desc), C.c_void_p(self.inc_chan.data_ptr()), self.chan_stride,
            C.c_void_p(orders.data_ptr()), C.c_void_p(masks.data_ptr()), C.c_void_p(chans.data_ptr()),
            self._stream()))
        return orders, masks, chans

    def incumbent_structure(self):
        """(stage orders, offloaded set, channel orders) of the incumbent."""
        from .packing import decode_mask, decode_orders
        from .schedule import TransferKind
        from .instance import OpId, OpKind
        pk = self.di.packed
        ch = self.inc_chan.cpu().numpy().view(np.uint32)
        chans = {}
        for g in range(pk.num_channels):
            seq = []
            for e in ch[g]:
                if int(e) == 0xFFFFFFFF:
                    break
                e = int(e)
                seq.append((OpId(((e >> 16) & 0x7FFF) + 1, (e & 0xFFFF) + 1, OpKind.F),
                            TransferKind.RELOAD if e >> 31 else TransferKind.OFFLOAD))
            chans[g] = tuple(seq)
        return (decode_orders(pk, self.inc_orders.cpu().numpy().view(np.uint16)),
                decode_mask(pk, self.inc_mask.cpu().numpy().view(np.uint32)), chans)

    def run(self, rounds: int | None = None, time_budget: float | None = None,
            patience: int | None = None) -> SearchResult:
        from .listsched import run_order
        if rounds is None and time_budget is None and patience is None:
            raise ValueError("need rounds, time_budget or patience")
        t0 = time.perf_counter()
        stale = 0
        while True:
            if rounds is not None and self.round >= rounds:
                break
            if time_budget is not None and time.perf_counter() - t0 >= time_budget:
                break
            if self.step(t0):
                stale = 0
            else:
                stale += 1
                if patience is not None and stale >= patience:
                    break
        orders, off, chans = self.incumbent_structure()
        sched = run_order(self.inst, orders, off, chans, device=self.di.device)
        return SearchResult(sched, self.makespan, self.initial_makespan, self.round, self.evaluated,
                            time.perf_counter() - t0, list(self.improvements))
