"""Batched re-timing of cached schedule orders.

The reference cache stores solved *orders* (per-stage op orders, offloaded set,
per-channel transfer orders) and re-times them for a new instance with
``run_order`` in explicit channel-order mode, rejecting entries that deadlock
or fail STRICT validation (cache.py:224-240); ``warm_start_from_cache``
compares the adapted hit with the heuristics, the cache winning ties
(cache.py:243-259).  Here every candidate entry is re-timed in ONE kernel
launch (``run_orders(..., explicit=True)``).  Entries are read in the
reference's JSON-lines record format (CacheEntry.to_dict, cache.py:78-92);
the file store, locking and fingerprint lookup stay in the reference.
"""

from __future__ import annotations

import json
from dataclasses import dataclass

from .instance import OpId, OpKind
from .schedule import MemorySemantics, TransferKind, makespan, validate


class ShapeMismatch(Exception):
    """Entry and instance disagree on (stages, micro-batches)."""


GRID_STEP = 0.25          # the reference's default ratio grid (cache.py:30)
NO_GAMMA = -1.0           # ratio sentinel: nothing to offload (cache.py:31)


@dataclass(frozen=True)
class CachedOrder:
    num_stages: int
    num_microbatches: int
    stage_orders: tuple       # per stage (1-based position) tuple of OpId
    offloaded: frozenset
    channel_orders: tuple     # per channel tuple of (OpId, TransferKind)
    recorded_makespan_ratio: float = 0.0
    ratios: tuple = ()        # the record's fingerprint (tB/tF, tW/tF, tcomm/tF, toff/tF, limit/gamma)
    post_validation: bool = False


def entry_from_record(d: dict) -> CachedOrder:
    """One JSON-lines record of the reference cache (cache.py:78-106)."""
    order = d["order"]
    stages = tuple(tuple(OpId(i + 1, int(j), OpKind.from_letter(c)) for j, c in so)
                   for i, so in enumerate(order["stages"]))
    off = frozenset(OpId(int(i), int(j), OpKind.F) for i, j in order["offloaded"])
    chans = tuple(tuple((OpId(int(i), int(j), OpKind.from_letter(c)),
                         TransferKind.OFFLOAD if t == "O" else TransferKind.RELOAD)
                        for i, j, c, t in co) for co in order["channels"])
    return CachedOrder(int(d["key"]["P"]), int(d["key"]["m"]), stages, off, chans,
                       float(d.get("makespan_ratio", 0.0)), tuple(float(x) for x in d["key"].get("ratios", ())),
                       bool(d["key"].get("post_validation", False)))


def load_entries(path) -> list:
    out = []
    with open(path, encoding="utf-8") as fh:
        for line in fh:
            if line.strip():
                out.append(entry_from_record(json.loads(line)))
    return out


def _shape(entry):
    key = getattr(entry, "key", None)
    if key is not None:
        return key.num_stages, key.num_microbatches
    return entry.num_stages, entry.num_microbatches


def adapt_batch(entries, inst, device=None) -> list:
    """Re-time every entry for `inst` in one launch: a Schedule, or None when the order deadlocks
    or the result fails STRICT validation (cache.py:224-240)."""
    from .listsched import OrderInfeasible, run_orders
    for e in entries:
        if _shape(e) != (inst.num_stages, inst.num_microbatches):
            raise ShapeMismatch(f"entry is {_shape(e)[0]}x{_shape(e)[1]}, instance is "
                                f"{inst.num_stages}x{inst.num_microbatches}")
    cands, slots = [], []
    for e in entries:
        orders = {i + 1: tuple(e.stage_orders[i]) for i in range(len(e.stage_orders))}
        chans = {g: tuple(e.channel_orders[g]) for g in range(len(e.channel_orders))}
        # an entry recorded under another topology (the cache key ignores topology_groups) is
        # not adaptable here: ChannelMismatch, DESIGN.md §7
        if _channels_match(inst, chans):
            slots.append(len(cands))
            cands.append((orders, frozenset(e.offloaded), chans))
        else:
            slots.append(None)
    res = run_orders(inst, cands, explicit=True, device=device) if cands else []
    out = []
    for k in slots:
        r = None if k is None else res[k]
        if r is None or isinstance(r, OrderInfeasible) or not validate(r, inst, MemorySemantics.STRICT).ok:
            out.append(None)
        else:
            out.append(r)
    return out


def _channels_match(inst, chans) -> bool:
    """Every listed transfer belongs to a stage the instance serves on that channel."""
    n = len(inst.topology_groups)
    for g, seq in chans.items():
        if g >= n:
            continue                     # channels the instance lacks are never read (listsched.py:233)
        for op, _kind in seq:
            if not (1 <= op[0] <= inst.num_stages) or inst.stage_channel(op[0]) != g:
                return False
    return True


def adapt(entry, inst, device=None):
    return adapt_batch([entry], inst, device)[0]


def best_adapted(entries, inst, device=None):
    """(schedule, index) of the minimum-makespan adaptable entry, first wins ties; or (None, None)."""
    best = (None, None, None)
    for k, s in enumerate(adapt_batch(entries, inst, device)):
        if s is None:
            continue
        span = makespan(s, inst)
        if best[0] is None or span < best[0]:
            best = (span, s, k)
    return best[1], best[2]


def warm_start_from_entries(entries, inst, params=None, device=None):
    """Best of the adapted entries and the heuristics; the cache wins ties (cache.py:243-259)."""
    from .heuristics import AdaParams, best_feasible
    adapted, _ = best_adapted(entries, inst, device)
    fallback, name = best_feasible(inst, params or AdaParams(), device=device)
    if adapted is not None and makespan(adapted, inst) <= makespan(fallback, inst):
        return adapted, "cache"
    return fallback, name


# -- every entry within the lookup radius ---------------------------------
# The reference's lookup returns the ONE nearest same-shape entry within a grid step and adapts it
# (cache.py:207-221, 243-259); here every entry within that radius is re-timed in one launch and
# the best adaptable one is kept.

def _mean(vals):
    vals = list(vals)
    return sum(vals) / len(vals) if vals else 0.0


def _snap(value, step):
    return round(round(value / step) * step, 9)


def fingerprint(inst, grid_step: float = GRID_STEP):
    """(P, m, ratios, post_validation): the reference's discretize (cache.py:111-131)."""
    if grid_step <= 0:
        raise ValueError("grid_step must be positive")
    ops = list(inst.ops())           # (kinds compared by value: reference instances carry their own OpKind)
    tf = _mean(inst.proc_time[op] for op in ops if int(op[2]) == 0)
    if tf <= 0:
        raise ValueError("mean forward time is zero")
    tb = _mean(inst.proc_time[op] for op in ops if int(op[2]) == 1)
    tw = _mean(inst.proc_time[op] for op in ops if int(op[2]) == 2)
    gammas = [inst.act_size[x] for x in inst.offloadable_ops()]
    mem = _snap(_mean(inst.mem_limit.values()) / _mean(gammas), grid_step) if gammas else NO_GAMMA
    ratios = (_snap(tb / tf, grid_step), _snap(tw / tf, grid_step), _snap(inst.comm_time / tf, grid_step),
              _snap(inst.offload_time / tf, grid_step), mem)
    return inst.num_stages, inst.num_microbatches, ratios, bool(inst.post_validation)


def _entry_key(e):
    key = getattr(e, "key", None)
    if key is not None:                  # a reference CacheEntry
        return key.num_stages, key.num_microbatches, tuple(key.ratios), bool(key.post_validation)
    return e.num_stages, e.num_microbatches, tuple(e.ratios), bool(e.post_validation)


def _ratio_distance(a, b) -> float:
    """The reference's _distance (cache.py:198-204): max abs difference, inf across NO_GAMMA."""
    worst = 0.0
    for x, y in zip(a, b):
        if (x == NO_GAMMA) != (y == NO_GAMMA):
            return float("inf")
        worst = max(worst, abs(x - y))
    return worst


def within_radius(entries, inst, grid_step: float = GRID_STEP) -> list:
    """Indices of the entries the reference's lookup would consider (same shape and post-validation
    flag, ratio distance within one grid step), ranked as lookup ranks them: (distance, recorded
    makespan ratio), first wins ties.  lookup's hit is the first of them."""
    P, m, ratios, post = fingerprint(inst, grid_step)
    ranked = []
    for k, e in enumerate(entries):
        eP, em, er, epost = _entry_key(e)
        if (eP, em, epost) != (P, m, post):
            continue
        d = _ratio_distance(er, ratios)
        if d > grid_step + 1e-9:
            continue
        ranked.append((d, e.recorded_makespan_ratio, k))
    ranked.sort(key=lambda t: t[:2])       # stable: equal ranks keep file order, as lookup's strict <
    return [k for _, _, k in ranked]


def adapt_radius(entries, inst, grid_step: float = GRID_STEP, device=None):
    """Re-time every entry within the lookup radius in ONE launch.  Returns (best schedule or None,
    its entry index or None, [(index, schedule or None) in lookup rank order]); the best is the
    minimum makespan, the better-ranked entry on ties."""
    idx = within_radius(entries, inst, grid_step)
    adapted = adapt_batch([entries[k] for k in idx], inst, device) if idx else []
    best = (None, None, None)
    for k, s in zip(idx, adapted):
        if s is None:
            continue
        span = makespan(s, inst)
        if best[0] is None or span < best[0]:
            best = (span, s, k)
    return best[1], best[2], list(zip(idx, adapted))


def warm_start_from_radius(entries, inst, params=None, grid_step: float = GRID_STEP, device=None):
    """warm_start_from_cache (cache.py:243-259) over every entry within the radius: the best
    adapted entry against the heuristics, the cache winning ties."""
    from .heuristics import AdaParams, best_feasible
    adapted, _, _ = adapt_radius(entries, inst, grid_step, device)
    fallback, name = best_feasible(inst, params or AdaParams(), device=device)
    if adapted is not None and makespan(adapted, inst) <= makespan(fallback, inst):
        return adapted, "cache"
    return fallback, name
