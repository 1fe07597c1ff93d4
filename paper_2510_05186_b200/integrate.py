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

from . import listsched as _ours
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


def install(ref_pkg) -> None:
    fn = gpu_run_order_for(ref_pkg)
    for site in _SITES:
        mod = importlib.import_module(f"{ref_pkg.__name__}.{site}")
        if hasattr(mod, "run_order"):
            _saved.setdefault((ref_pkg.__name__, site), mod.run_order)
            mod.run_order = fn
    ref_pkg.run_order = fn


def uninstall(ref_pkg) -> None:
    for site in _SITES:
        key = (ref_pkg.__name__, site)
        if key in _saved:
            mod = importlib.import_module(f"{ref_pkg.__name__}.{site}")
            mod.run_order = _saved.pop(key)
    ref_pkg.run_order = importlib.import_module(ref_pkg.__name__ + ".listsched").run_order
