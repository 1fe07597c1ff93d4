"""B200-native candidate-schedule evaluation and local search for OptPipe.

Drop-in for the reference ``pipesched`` hot path: the names
below mirror the reference package root (pkg/src/pipesched/__init__.py:4-30)
for everything on the path — instance model, schedule model, ``run_order``
and the warm-start generators — with the timing computed by hand-written
sm_100a kernels behind the C ABI in ``include/pipesched_b200.h``.
"""

from .instance import (InvariantViolation, OpId, OpKind, ParseError, PipelineInstance,
                       instance_from_dict, instance_to_dict, load_instance, make_uniform_instance,
                       random_instance, save_instance)
from .schedule import (ComputeEvent, EvalMetrics, IncompleteSchedule, InvalidSchedule,
                       MemorySemantics, MemoryTrace, NegativeUsage, Schedule, TransferEvent,
                       TransferKind, ValidationReport, Violation, bubble_ratio, check_structure,
                       load_schedule, makespan, memory_trace, save_schedule, schedule_from_dict,
                       schedule_to_dict, validate)
from .listsched import OrderInfeasible, channel_order_of, run_order, run_orders, stage_order_of
from .heuristics import (AdaParams, InfeasibleSchedule, NoFeasibleSchedule, ada_offload,
                         best_feasible, fill_profile, one_f_one_b, pipeoffload_like,
                         sequential_schedule)

__version__ = "0.1.0"
