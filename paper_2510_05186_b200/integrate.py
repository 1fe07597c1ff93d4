"""Bind the B200 evaluator into an unmodified reference ``pipesched`` package.

The reference calls ``run_order`` from four places — the generators
(heuristics.py:61, 81, 104, 176) and the cache (cache.py:235) — through
module-level names imported from ``pipesched.listsched``.  ``install`` points
those names at a wrapper that evaluates on the GPU and answers in the
reference's own types: it returns ``pipesched.schedule.Schedule`` objects
(events in commit order, so ``==`` against the CPU path holds) and raises the
reference's ``OrderInfeasible`` with the same ``stages`` tuple.

    import pipesched
    from paper_2510_05186_b200 import integrate
    integrate.install(pipesched)          # pipesched.best_feasible etc. now time on the GPU
    integrate.uninstall(pipesched)        # back to the CPU path
"""

from __future__ import annotations

import importlib
import time
from dataclasses import dataclass

import numpy as np

from . import listsched as _ours
from .packing import decode_mask, decode_orders
from .search import SearchConfig
from .packing import ChannelMismatch

_SITES = ("listsched", "heuristics", "cache")
_saved: dict = {}


def gpu_run_order_for(ref_pkg):
    """A run_order with the reference signature that evaluates on the GPU."""
    ref_sched = importlib.import_module(ref_pkg.__name__ + ".schedule")
    ref_ls = importlib.import_module(ref_pkg.__name__ + ".listsched")

    def run_order(inst, stage_orders, offloaded, channel_orders=None):
        try:
            return _ours.run_order(inst, stage_orders, offloaded, channel_orders, types=ref_sched)
        except _ours.OrderInfeasible as e:
            raise ref_ls.OrderInfeasible(str(e), e.stages) from None
        except ChannelMismatch as e:
            # an explicit channel order from another topology: not replayable here;
            # the reference's callers (cache.adapt) treat it as not adaptable
            raise ref_ls.OrderInfeasible(str(e), ()) from None

    run_order.__doc__ = "GPU-evaluated drop-in for pipesched.listsched.run_order (listsched.py:167)."
    return run_order


_GENERATORS = ("ada_offload", "pipeoffload_like", "one_f_one_b", "sequential_schedule", "best_feasible")
_GEN_SITES = ("heuristics", "cache", "online")


def gpu_generators_for(ref_pkg, originals: dict):
    """The reference's generators (heuristics.py:50-210) with the whole AdaOffload back-off
    sequence and the other three structures timed in one batched launch (heuristics.generate_all),
    answers decoded into the reference's own Schedule type.  A generator whose structure is
    infeasible defers to the reference's own function (through the GPU run_order), which raises
    its own InfeasibleSchedule with its own message."""
    from . import heuristics as _heur
    ref_h = importlib.import_module(ref_pkg.__name__ + ".heuristics")
    ref_sched = importlib.import_module(ref_pkg.__name__ + ".schedule")
    names = {"ada_offload": "ada", "pipeoffload_like": "pipeoffload", "one_f_one_b": "1f1b",
             "sequential_schedule": "sequential"}

    def _all(inst, params):
        spans: dict = {}
        out = _heur.generate_all(inst, _heur.AdaParams(tolerance=params.tolerance), types=ref_sched, spans=spans)
        return out, spans

    def single(fn_name, takes_params):
        key = names[fn_name]

        def gen(inst, params=ref_h.AdaParams()):
            out, _ = _all(inst, params)
            if isinstance(out[key], Exception):
                return originals[fn_name](inst, params) if takes_params else originals[fn_name](inst)
            return out[key]
        if not takes_params:
            def gen_noparams(inst):
                return gen(inst)
            gen_noparams.__doc__ = f"GPU-batched drop-in for pipesched.heuristics.{fn_name}."
            return gen_noparams
        gen.__doc__ = f"GPU-batched drop-in for pipesched.heuristics.{fn_name}."
        return gen

    def best_feasible(inst, params=ref_h.AdaParams()):
        out, spans = _all(inst, params)
        best = None
        for key in ("ada", "pipeoffload", "1f1b", "sequential"):        # _GENERATORS order, first wins ties
            if isinstance(out[key], Exception):
                continue
            if best is None or spans[key] < best[0]:
                best = (spans[key], out[key], key)
        if best is None:
            raise ref_h.NoFeasibleSchedule("all generators failed on this instance")
        return best[1], best[2]

    best_feasible.__doc__ = "GPU-batched drop-in for pipesched.heuristics.best_feasible (heuristics.py:196)."
    return {"ada_offload": single("ada_offload", True), "pipeoffload_like": single("pipeoffload_like", False),
            "one_f_one_b": single("one_f_one_b", False), "sequential_schedule": single("sequential_schedule", False),
            "best_feasible": best_feasible}


@dataclass(frozen=True)
class WarmSearch:
    """How the GPU local search improves a warm start before the reference solver sees it."""

    config: SearchConfig = SearchConfig()
    rounds: int | None = None
    time_budget: float | None = None
    patience: int | None = 16          # steps in a row without improving the best that end the search
    kicks: int | None = None           # ILS restarts (config.kick_moves > 0)
    device: int | None = None


def search_warm_start(ref_pkg, inst, warm=None, search: WarmSearch = WarmSearch()):
    """Run the GPU local search on a reference instance and return ``(schedule, events)``.

    ``warm`` (a reference ``Schedule``) is the start; by default the reference's own
    ``best_feasible`` (heuristics.py:196-210 — GPU-timed when installed).  ``schedule`` is the
    winner as a reference ``Schedule`` (commit-ordered events, STRICT-valid), ready for
    ``pipesched.start_session(warm=...)`` (solver.py:543-565); ``events`` are the strict
    improvements as reference ``IncumbentEvent`` objects with the search's timestamps
    (solver.py:81-87, 435-449), the warm start first at 0.0."""
    from .search import LocalSearch
    ref_solver = importlib.import_module(ref_pkg.__name__ + ".solver")
    ref_sched = importlib.import_module(ref_pkg.__name__ + ".schedule")
    ref_ls = importlib.import_module(ref_pkg.__name__ + ".listsched")
    if warm is None:
        warm, _ = ref_pkg.best_feasible(inst, ref_pkg.AdaParams())
    span0 = ref_sched.makespan(warm, inst)
    orders = {i: ref_ls.stage_order_of(warm, i) for i in range(1, inst.num_stages + 1)}
    ls = LocalSearch(inst, orders, warm.offloaded, search.config, device=search.device)
    if ls.makespan != span0:
        raise RuntimeError("warm start re-timed to a different makespan")
    rounds = search.rounds
    if rounds is None and search.time_budget is None and search.patience is None and search.kicks is None:
        rounds = 64
    ls.keep_structures = True
    res = ls.run(rounds=rounds, time_budget=search.time_budget, patience=search.patience, kicks=search.kicks)
    # every strict improvement of the best as a reference Schedule, all timed in one launch
    pk = ls.di.packed
    structures = [(decode_orders(pk, o.cpu().numpy().view(np.uint16)), decode_mask(pk, mk.cpu().numpy().view(np.uint32)))
                  for o, mk in ls.improvement_structures]
    scheds = _ours.run_orders(inst, structures, device=ls.di.device, types=ref_sched) if structures else []
    from .solver import lower_bound
    lb = lower_bound(inst, inst.post_validation, device=ls.di.device)
    events = [ref_solver.IncumbentEvent(warm, span0, min(lb, span0), 0.0)]
    for imp, sched in zip(res.improvements, scheds):
        if ref_sched.makespan(sched, inst) != imp.makespan:
            raise RuntimeError("replayed incumbent re-timed to a different makespan")
        events.append(ref_solver.IncumbentEvent(sched, imp.makespan, min(lb, imp.makespan), imp.timestamp))
    return events[-1].schedule, events


def search_fed_start_session(ref_pkg, search: WarmSearch = WarmSearch()):
    """A ``start_session`` with the reference signature (solver.py:543-565) whose warm start is
    first improved by the GPU local search; the reference branch-and-bound then runs unchanged
    from the search's winner.  The returned reference ``SolveSession`` streams the search's
    improvements (their timestamps) followed by the solver's (shifted by the search's time)."""
    ref_solver = importlib.import_module(ref_pkg.__name__ + ".solver")
    original = _saved.get((ref_pkg.__name__, "solver.start_session"), ref_solver.start_session)

    def start_session(inst, budget=None, warm=None, symmetry=True, post_validation=None, auto_warm=True):
        if warm is None and not auto_warm:
            return original(inst, budget, warm=None, symmetry=symmetry, post_validation=post_validation,
                            auto_warm=False)
        t0 = time.monotonic()
        try:
            best, events = search_warm_start(ref_pkg, inst, warm, search)
        except ref_pkg.NoFeasibleSchedule:
            return original(inst, budget, warm=None, symmetry=symmetry, post_validation=post_validation,
                            auto_warm=False)
        spent = time.monotonic() - t0
        session = original(inst, budget, warm=best, symmetry=symmetry, post_validation=post_validation,
                           auto_warm=False)
        # the search's improvements, then the solver's stream (its first event is the winner again,
        # re-stamped by the solver at its own clock 0)
        merged = events[:-1]
        for ev in session.stream():
            merged.append(ref_solver.IncumbentEvent(ev.schedule, ev.makespan, ev.lower_bound,
                                                    ev.timestamp + spent, ev.status))
        return ref_solver.SolveSession(session.outcome, merged)

    start_session.__doc__ = "GPU-search-fed drop-in for pipesched.solver.start_session (solver.py:543)."
    return start_session


def install(ref_pkg, search: WarmSearch | None = None, generators: bool = True) -> None:
    """Point the reference's run_order call sites at the GPU evaluator; with ``generators``, also
    its generators and ``best_feasible`` at the batched GPU versions (one launch for the whole
    AdaOffload back-off sequence); with ``search``, also let its ``start_session`` (and so
    ``solve`` and ``online_sim``) start from the GPU local search's winner."""
    fn = gpu_run_order_for(ref_pkg)
    for site in _SITES:
        mod = importlib.import_module(f"{ref_pkg.__name__}.{site}")
        if hasattr(mod, "run_order"):
            _saved.setdefault((ref_pkg.__name__, site), mod.run_order)
            mod.run_order = fn
    ref_pkg.run_order = fn
    if generators:
        ref_h = importlib.import_module(ref_pkg.__name__ + ".heuristics")
        originals = {name: _saved.get((ref_pkg.__name__, f"heuristics.{name}"), getattr(ref_h, name))
                     for name in _GENERATORS}
        gens = gpu_generators_for(ref_pkg, originals)
        for site in _GEN_SITES + ("",):
            mod = importlib.import_module(f"{ref_pkg.__name__}.{site}") if site else ref_pkg
            for name in _GENERATORS:
                if hasattr(mod, name):
                    _saved.setdefault((ref_pkg.__name__, f"{site or 'pkg'}.{name}"), getattr(mod, name))
                    setattr(mod, name, gens[name])
    if search is not None:
        ref_solver = importlib.import_module(ref_pkg.__name__ + ".solver")
        ref_online = importlib.import_module(ref_pkg.__name__ + ".online")
        _saved.setdefault((ref_pkg.__name__, "solver.start_session"), ref_solver.start_session)
        _saved.setdefault((ref_pkg.__name__, "online.start_session"), ref_online.start_session)
        fed = search_fed_start_session(ref_pkg, search)
        ref_solver.start_session = fed
        ref_online.start_session = fed
        ref_pkg.start_session = fed


def uninstall(ref_pkg) -> None:
    for site in _GEN_SITES + ("",):
        mod = importlib.import_module(f"{ref_pkg.__name__}.{site}") if site else ref_pkg
        for name in _GENERATORS:
            key = (ref_pkg.__name__, f"{site or 'pkg'}.{name}")
            if key in _saved:
                setattr(mod, name, _saved.pop(key))
    for site in _SITES:
        key = (ref_pkg.__name__, site)
        if key in _saved:
            mod = importlib.import_module(f"{ref_pkg.__name__}.{site}")
            mod.run_order = _saved.pop(key)
    ref_pkg.run_order = importlib.import_module(ref_pkg.__name__ + ".listsched").run_order
    for site in ("solver", "online"):
        key = (ref_pkg.__name__, f"{site}.start_session")
        if key in _saved:
            mod = importlib.import_module(f"{ref_pkg.__name__}.{site}")
            mod.start_session = _saved.pop(key)
    ref_pkg.start_session = importlib.import_module(ref_pkg.__name__ + ".solver").start_session
