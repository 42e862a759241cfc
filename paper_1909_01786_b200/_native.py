"""Loader for the in-tree C-ABI library ``_lib/libyasmin_b200.so``.

The product has exactly one implementation: the sm_100a engine behind the
C-ABI in ``include/yasmin_b200.h``. If the library is missing this module
raises instead of falling back to anything else.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# YAS_LIBRARY: developer A/B of an alternative build of the same library (default: the in-tree one)
LIB_PATH = os.environ.get("YAS_LIBRARY") or os.path.join(_HERE, "_lib", "libyasmin_b200.so")

# every symbol include/yasmin_b200.h declares (checked by tests/test_abi.py)
EXPORTS = [
    "yas_version", "yas_device_count", "yas_device_name",
    "yas_program_parse", "yas_program_parse_file", "yas_program_free", "yas_program_atom_count",
    "yas_program_rule_count", "yas_program_constraint_count", "yas_program_atom_name", "yas_program_find",
    "yas_program_rule", "yas_program_print", "yas_program_dump_nogoods", "yas_program_store_csv",
    "yas_program_diagnostics", "yas_program_rule_aux", "yas_program_total_atoms", "yas_program_census",
    "yas_program_tp_step", "yas_program_cubes", "yas_verify_model",
    "yas_config_default", "yas_solve", "yas_result_status", "yas_result_model_count", "yas_result_model",
    "yas_result_model_cube", "yas_result_models_flat", "yas_result_stats", "yas_result_free", "yas_stats_csv_header", "yas_emit_stats",
    "yas_store_build", "yas_store_free", "yas_store_size", "yas_store_total_atoms", "yas_store_dump_csv",
    "yas_store_units", "yas_store_unit_ids", "yas_store_bounds", "yas_store_occurrences", "yas_store_planted",
    "yas_free_ints",
    "yas_propagator_create", "yas_propagator_free", "yas_propagator_reset", "yas_propagator_initial",
    "yas_propagator_propagate", "yas_propagator_push_decision", "yas_propagator_assign", "yas_propagator_seed",
    "yas_propagator_add_learned", "yas_propagator_count_literals", "yas_propagator_atoms", "yas_propagator_cells", "yas_propagator_reasons",
    "yas_propagator_deps", "yas_propagator_trail", "yas_propagator_conflicts", "yas_propagator_frontier",
    "yas_propagator_level", "yas_propagator_profile", "yas_propagator_flush", "yas_propagator_pass_trace",
    "yas_propagator_last_error",
    "yas_fleet_unique_id", "yas_fleet_create_nccl", "yas_fleet_create", "yas_fleet_free", "yas_fleet_info",
    "yas_fleet_allreduce", "yas_program_create", "yas_program_intern", "yas_program_add_rule", "yas_store_nogood",
    "yas_propagator_clear_frontier", "yas_propagator_transfers",
]


class yas_trace(C.Structure):
    _fields_ = [("mode", C.c_int), ("conflict_id", C.c_int32), ("learned_length", C.c_uint64),
                ("backjump_level", C.c_uint32)]


TRACE_FN = C.CFUNCTYPE(None, C.POINTER(yas_trace), C.c_void_p)
ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.POINTER(C.c_uint64), C.c_size_t, C.c_int, C.c_void_p)
BROADCAST_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_size_t, C.c_int, C.c_void_p)


class yas_config(C.Structure):
    _fields_ = [
        ("mode", C.c_int), ("heuristic", C.c_int), ("activity_decay", C.c_double), ("workers", C.c_uint),
        ("restarts_enabled", C.c_int), ("restart_base", C.c_uint64), ("restart_factor", C.c_double),
        ("max_models", C.c_uint64), ("deps_words", C.c_uint32), ("conflict_fanout", C.c_uint32),
        ("seed", C.c_uint64), ("verify", C.c_int), ("debug_validate", C.c_int),
        ("learned_capacity", C.c_uint64), ("trace", TRACE_FN), ("trace_user", C.c_void_p),
        ("device", C.c_int), ("engine", C.c_int), ("cube_atoms", C.c_uint32), ("cube_depth", C.c_uint32),
        ("slots", C.c_uint32),
        ("rank", C.c_int), ("world", C.c_int), ("portfolio", C.c_uint32), ("count_lits", C.c_uint32),
        ("n_devices", C.c_uint32), ("devices", C.POINTER(C.c_int)), ("reference_order", C.c_int),
        ("fleet", C.c_void_p),
    ]


class yas_stats(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in (
        "decisions", "propagations", "conflicts", "learned_count", "learned_length_sum", "restarts", "models")] + [
        ("wall_ms", C.c_double)] + [(n, C.c_uint64) for n in (
        "passes", "watch_replacements", "duplicate_learned", "blocking_nogoods", "res_learned", "fwd_learned",
        "fwd_fallbacks", "uip_check_failures", "fwd_decision_only_failures", "asserting_failures", "checks",
        "searches", "launches")] + [("device_ms", C.c_double), ("cubes", C.c_uint64), ("checked_lits", C.c_uint64),
                                              ("portfolio_variant", C.c_int64), ("fleet_models", C.c_uint64),
                                              ("devices", C.c_uint32), ("fleet_ranks", C.c_uint32),
                                              ("fleet_winner", C.c_int32), ("pad", C.c_uint32)]


class yas_outcome(C.Structure):
    _fields_ = [("violated", C.c_int), ("propagations", C.c_uint64), ("passes", C.c_uint64),
                ("checks", C.c_uint64), ("checked_lits", C.c_uint64), ("n_conflicts", C.c_uint32),
                ("device_ms", C.c_float)]


_lib = None


def lib() -> C.CDLL:
    """Load the library (once). Raises FileNotFoundError when it was not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise FileNotFoundError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(yasmin-b200 has no fallback implementation)")
    L = C.CDLL(LIB_PATH)
    P, U32, U64, I32, SZ = C.c_void_p, C.c_uint32, C.c_uint64, C.c_int32, C.c_size_t
    pI32, pU32, pU64, pU8 = C.POINTER(C.c_int32), C.POINTER(C.c_uint32), C.POINTER(C.c_uint64), C.POINTER(C.c_uint8)
    sig = {
        "yas_version": (C.c_char_p, []),
        "yas_device_count": (C.c_int, []),
        "yas_device_name": (C.c_int, [C.c_int, C.c_char_p, SZ]),
        "yas_program_parse": (C.c_int, [C.c_char_p, SZ, C.POINTER(P), C.POINTER(C.c_int), C.c_char_p, SZ]),
        "yas_program_parse_file": (C.c_int, [C.c_char_p, C.POINTER(P), C.POINTER(C.c_int), C.c_char_p, SZ]),
        "yas_program_free": (None, [P]),
        "yas_program_atom_count": (U32, [P]),
        "yas_program_rule_count": (U32, [P]),
        "yas_program_constraint_count": (U32, [P]),
        "yas_program_atom_name": (C.c_char_p, [P, U32]),
        "yas_program_find": (U32, [P, C.c_char_p]),
        "yas_program_rule": (C.c_int, [P, U32, pU32, C.POINTER(pU32), pU32, C.POINTER(pU32), pU32]),
        "yas_program_print": (SZ, [P, C.c_char_p, SZ]),
        "yas_program_dump_nogoods": (SZ, [P, C.c_char_p, SZ]),
        "yas_program_store_csv": (SZ, [P, C.c_char_p, SZ]),
        "yas_program_diagnostics": (SZ, [P, C.c_char_p, SZ]),
        "yas_program_rule_aux": (C.c_int, [P, U32, pU32]),
        "yas_program_total_atoms": (U32, [P]),
        "yas_program_census": (C.c_int, [P, pU64, pU64]),
        "yas_program_tp_step": (SZ, [P, pU32, SZ, pU32, SZ]),
        "yas_program_cubes": (SZ, [P, U32, U32, U32, C.c_int, C.c_int, pI32, SZ, pU32]),
        "yas_verify_model": (C.c_int, [P, pU32, SZ]),
        "yas_config_default": (None, [C.POINTER(yas_config)]),
        "yas_solve": (C.c_int, [P, C.POINTER(yas_config), C.POINTER(P), C.c_char_p, SZ]),
        "yas_result_status": (C.c_int, [P]),
        "yas_result_model_count": (U64, [P]),
        "yas_result_model": (pU32, [P, U64, pU32]),
        "yas_result_model_cube": (U32, [P, U64]),
        "yas_result_models_flat": (SZ, [P, pU32, SZ, pU64, pU32]),
        "yas_result_stats": (None, [P, C.POINTER(yas_stats)]),
        "yas_result_free": (None, [P]),
        "yas_stats_csv_header": (SZ, [C.c_char_p, SZ]),
        "yas_emit_stats": (SZ, [C.POINTER(yas_stats), C.c_char_p, C.c_char_p, C.c_char_p, C.c_uint, C.c_int,
                                U64, C.c_int, C.c_char_p, SZ]),
        "yas_store_build": (C.c_int, [pI32, pU32, SZ, pU32, pU8, U32, C.POINTER(P), C.c_char_p, SZ]),
        "yas_store_free": (None, [P]),
        "yas_store_size": (U32, [P]),
        "yas_store_total_atoms": (U32, [P]),
        "yas_store_dump_csv": (SZ, [P, C.c_char_p, SZ]),
        "yas_store_units": (SZ, [P, pI32, SZ]),
        "yas_store_unit_ids": (SZ, [P, pI32, SZ]),
        "yas_store_bounds": (None, [P, pU32]),
        "yas_store_occurrences": (SZ, [P, I32, U32, pI32, SZ]),
        "yas_store_planted": (C.c_int, [U32, U64, U32, U64, C.POINTER(P), C.POINTER(pI32), C.POINTER(SZ), pI32]),
        "yas_free_ints": (None, [pI32]),
        "yas_propagator_create": (C.c_int, [P, U32, C.c_int, C.c_int, C.POINTER(P), C.c_char_p, SZ]),
        "yas_propagator_free": (None, [P]),
        "yas_propagator_reset": (C.c_int, [P]),
        "yas_propagator_initial": (C.c_int, [P, C.POINTER(yas_outcome)]),
        "yas_propagator_propagate": (C.c_int, [P, U32, C.POINTER(yas_outcome)]),
        "yas_propagator_push_decision": (C.c_int, [P, I32]),
        "yas_propagator_assign": (C.c_int, [P, pI32, SZ, U32, pU64, U32, C.c_int, I32]),
        "yas_propagator_seed": (C.c_int, [P, pI32, SZ]),
        "yas_propagator_add_learned": (I32, [P, pI32, SZ]),
        "yas_propagator_count_literals": (C.c_int, [P, C.c_int]),
        "yas_propagator_atoms": (U32, [P]),
        "yas_propagator_cells": (C.c_int, [P, pI32]),
        "yas_propagator_reasons": (C.c_int, [P, pI32]),
        "yas_propagator_deps": (C.c_int, [P, U32, pU64, pU8]),
        "yas_propagator_trail": (SZ, [P, pI32, SZ]),
        "yas_propagator_conflicts": (SZ, [P, pI32, SZ]),
        "yas_propagator_frontier": (SZ, [P, pI32, SZ]),
        "yas_propagator_level": (U32, [P]),
        "yas_propagator_profile": (C.c_int, [P, C.POINTER(C.c_uint64)]),
        "yas_propagator_flush": (C.c_int, [P]),
        "yas_propagator_pass_trace": (C.c_int, [P, C.c_int, C.POINTER(C.c_uint64), C.c_size_t, C.POINTER(U32)]),
        "yas_propagator_last_error": (SZ, [P, C.c_char_p, SZ]),
        "yas_propagator_clear_frontier": (C.c_int, [P]),
        "yas_propagator_transfers": (C.c_int, [P, pU64, pU64]),
        "yas_program_create": (P, []),
        "yas_program_intern": (U32, [P, C.c_char_p]),
        "yas_program_add_rule": (C.c_int, [P, U32, pU32, SZ, pU32, SZ]),
        "yas_store_nogood": (SZ, [P, U32, pI32, SZ, pU32, pU8]),
        "yas_fleet_unique_id": (C.c_int, [C.POINTER(C.c_uint8), C.c_char_p, SZ]),
        "yas_fleet_create_nccl": (C.c_int, [C.POINTER(C.c_uint8), C.c_int, C.c_int, C.c_int, C.POINTER(P),
                                            C.c_char_p, SZ]),
        "yas_fleet_create": (C.c_int, [C.c_int, C.c_int, C.c_int, ALLREDUCE_FN, BROADCAST_FN, P, C.POINTER(P),
                                       C.c_char_p, SZ]),
        "yas_fleet_free": (None, [P]),
        "yas_fleet_info": (C.c_int, [P, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int),
                                     C.POINTER(C.c_int)]),
        "yas_fleet_allreduce": (C.c_int, [P, pU64, SZ, C.c_int, C.c_char_p, SZ]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L
