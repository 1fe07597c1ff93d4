"""Anytime solver API driven by the GPU local search.

Same call shapes as the reference solver API — ``SolveBudget``, ``SolveOutcome``,
``IncumbentEvent``, ``start_session`` / ``SolveSession`` / ``incumbent_stream``,
``solve`` (solver.py:45-87, 523-582) — and ``online_sim`` on top of it
(online.py:48-81).  The reference's engine behind that API is a recursive
branch-and-bound (solver.py:164-520), which this tier does not rebuild; here
the engine is the GPU local search: a warm start (given, or the batched
``best_feasible``), then search rounds until the budget is spent, recording
every strict improvement as an ``IncumbentEvent`` with its timestamp.  The
lower bound is a simple valid bound (busiest stage; one microbatch's critical
path), so the status is ``Optimal`` only when the incumbent meets it.
"""

from __future__ import annotations

import time as _time
from dataclasses import dataclass, replace

from .instance import OpId, OpKind, PipelineInstance
from .schedule import MemorySemantics, Schedule, makespan, validate

OPTIMAL = "Optimal"
FEASIBLE = "Feasible"
INFEASIBLE = "Infeasible"
UNKNOWN = "Unknown"


class SessionClosed(Exception):
    """The incumbent stream was already consumed."""


@dataclass(frozen=True)
class SolveBudget:
    wall_time_limit: float | None = 300.0     # seconds
    node_limit: int | None = None             # here: neighbour evaluations
    target_gap: float = 0.0

    def __post_init__(self):
        if self.wall_time_limit is None and self.node_limit is None:
            raise ValueError("need a wall-time or node limit")
        if self.target_gap < 0:
            raise ValueError("target_gap must be >= 0")


@dataclass
class SolveOutcome:
    incumbent: Schedule | None
    incumbent_makespan: int | None
    lower_bound: int
    status: str
    nodes: int = 0                # neighbours evaluated
    prunes_bound: int = 0
    dead_ends: int = 0
    elapsed: float = 0.0

    def to_dict(self):
        return {"status": self.status, "makespan": self.incumbent_makespan,
                "lower_bound": self.lower_bound, "nodes": self.nodes,
                "prunes_bound": self.prunes_bound, "dead_ends": self.dead_ends,
                "elapsed_s": round(self.elapsed, 6)}


@dataclass(frozen=True)
class IncumbentEvent:
    schedule: Schedule
    makespan: int
    lower_bound: int
    timestamp: float
    status: str | None = None     # set on the final event of a stream


class SolveSession:
    def __init__(self, outcome: SolveOutcome, events):
        self.outcome = outcome
        self._events = list(events)
        self._consumed = False

    def stream(self):
        if self._consumed:
            raise SessionClosed("incumbent stream already consumed")
        self._consumed = True
        return iter(self._events)


def incumbent_stream(session: SolveSession):
    return session.stream()


def lower_bound(inst: PipelineInstance, post_validation: bool, device=None) -> int:
    """The reference solver's root bound (solver.py:481): ``_Search._bound`` at the empty node
    (clock 0, every stage free at 0, nothing committed), computed by the batched GPU bound kernel
    (bound.py) — per-stage work, and the F-down / B-up / W chains of every microbatch."""
    from .bound import lower_bounds
    if post_validation != inst.post_validation:
        inst = replace(inst, post_validation=post_validation)
    root = (0, {i: 0 for i in range(1, inst.num_stages + 1)}, {})
    return lower_bounds(inst, [root], device=device)[0]


def start_session(inst: PipelineInstance, budget: SolveBudget | None = None,
                  warm: Schedule | None = None, symmetry: bool = True,
                  post_validation: bool | None = None, auto_warm: bool = True,
                  search=None, device=None) -> SolveSession:
    """Run the GPU local search within `budget` and wrap its improvements in a session."""
    from .heuristics import AdaParams, NoFeasibleSchedule, best_feasible
    from .listsched import stage_order_of
    from .search import LocalSearch, SearchConfig
    budget = budget or SolveBudget()
    post = inst.post_validation if post_validation is None else post_validation
    if post != inst.post_validation:
        inst = replace(inst, post_validation=post)
    t0 = _time.monotonic()
    if warm is None and auto_warm:
        try:
            warm, _ = best_feasible(inst, AdaParams(), device=device)
        except NoFeasibleSchedule:
            warm = None
    if warm is not None and not validate(warm, inst, MemorySemantics.STRICT).ok:
        warm = None                # unsafe warm starts are unusable as incumbents (solver.py:557-560)
    lb = lower_bound(inst, post, device=device)
    if warm is None:
        outcome = SolveOutcome(None, None, lb, UNKNOWN, elapsed=_time.monotonic() - t0)
        return SolveSession(outcome, [])
    span0 = makespan(warm, inst)
    events = [IncumbentEvent(warm, span0, min(lb, span0), 0.0)]
    # the engine: iterated local search until the budget is spent
    cfg = search or SearchConfig(kick_moves=4)
    best, best_span, nodes = warm, span0, 0
    over = (budget.wall_time_limit is not None and budget.wall_time_limit <= 0) or \
           (budget.node_limit is not None and budget.node_limit <= 0)
    if not over and span0 > lb:
        orders = {i: stage_order_of(warm, i) for i in range(1, inst.num_stages + 1)}
        ls = LocalSearch(inst, orders, warm.offloaded, cfg, device=device)
        if ls.makespan != span0:
            raise RuntimeError("warm start re-timed to a different makespan")
        while True:
            # the wall-clock test is collective: every rank leaves the loop on the same round
            if budget.wall_time_limit is not None and ls.should_stop(
                    _time.monotonic() - t0 >= budget.wall_time_limit):
                break
            if budget.node_limit is not None and nodes + cfg.neighbours > budget.node_limit:
                break
            before = ls.best_makespan
            ls.step_ils()
            nodes = ls.evaluated
            if ls.best_makespan < before:
                best_span = ls.best_makespan
                o, off = ls.incumbent_structure()
                from .listsched import run_order
                best = run_order(inst, o, off, device=ls.di.device)
                events.append(IncumbentEvent(best, best_span, min(lb, best_span), _time.monotonic() - t0))
                if best_span <= lb:
                    break
                if budget.target_gap > 0 and best_span - lb <= budget.target_gap * best_span:
                    break
    status = OPTIMAL if best_span <= lb else FEASIBLE
    bound = best_span if status == OPTIMAL else lb
    last = events[-1]
    events[-1] = IncumbentEvent(last.schedule, last.makespan, bound, last.timestamp, status)
    outcome = SolveOutcome(best, best_span, bound, status, nodes=nodes, elapsed=_time.monotonic() - t0)
    return SolveSession(outcome, events)


def solve(inst: PipelineInstance, opts=None, budget: SolveBudget | None = None,
          warm: Schedule | None = None) -> SolveOutcome:
    post = None
    if opts is not None:
        post = getattr(opts, "post_validation", None)
    return start_session(inst, budget=budget, warm=warm, post_validation=post).outcome


# -- online loop (reference online.py:48-81) --------------------------------------------------

@dataclass(frozen=True)
class OnlineStep:
    iteration: int
    source: str
    span: int


@dataclass(frozen=True)
class OnlineReport:
    total_time: int
    warm_source: str
    solver_status: str
    steps: tuple = ()
    trajectory: tuple = ()

    def to_dict(self):
        return {"total_time": self.total_time, "warm_source": self.warm_source,
                "solver_status": self.solver_status,
                "steps": [{"iteration": s.iteration, "source": s.source, "span": s.span} for s in self.steps],
                "trajectory": [{"at": t, "span": s} for t, s in self.trajectory]}


def online_sim(inst: PipelineInstance, iterations: int, budget: SolveBudget | None = None,
               params=None) -> OnlineReport:
    """Iterations consume their schedule's makespan on one clock with the solver's seconds; at
    every boundary the newest strictly better incumbent that has arrived is adopted."""
    from .heuristics import AdaParams, best_feasible
    if iterations < 1:
        raise ValueError("iterations must be >= 1")
    warm, source = best_feasible(inst, params or AdaParams())
    session = start_session(inst, budget or SolveBudget(wall_time_limit=0.0), warm=warm)
    incumbents = [(ev.timestamp, ev.makespan, ev.schedule) for ev in incumbent_stream(session)]
    cur_src, cur_span = "warm", makespan(warm, inst)
    sim, steps = 0, []
    for it in range(1, iterations + 1):
        steps.append(OnlineStep(it, cur_src, cur_span))
        sim += cur_span
        for at, span, _sched in incumbents:
            if at <= sim and span < cur_span:
                cur_src, cur_span = f"incumbent@{at:.3f}", span
    return OnlineReport(total_time=sim, warm_source=source, solver_status=session.outcome.status,
                        steps=tuple(steps),
                        trajectory=tuple((round(at, 6), span) for at, span, _ in incumbents))
