"""yasmin-b200: B200-native (sm_100a) core of the yasmin conflict-driven ASP solver.

The reference-facing API lives in :mod:`paper_1909_01786_b200.aspine`; it is a
thin ctypes mirror of the C-ABI in ``include/yasmin_b200.h``.
"""
from .aspine import (  # noqa: F401
    ConflictTrace, DeviceError, Fleet, GroundProgram, HeuristicConfig, HeuristicKind, LearnMode, LogicError, Model,
    NogoodStore, ParseError, PropagationOutcome, Propagator, RestartPolicy, SolveResult, SolveStats, SolveStatus,
    SolverConfig, StatsContext, StoreCapacityError, VerificationError, device_count, dump_nogoods, emit_stats,
    cubes, parse_file, parse_program, print_program, solve, stats_csv_header, store_csv, tp_step, validate, verify_model,
)
