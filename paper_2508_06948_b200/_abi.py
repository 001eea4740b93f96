"""ctypes binding of the C ABI in include/kairos_b200.h.

This is plumbing for tests and the benchmark: every computation happens in
the CUDA kernels of libkairos_b200.so. Loading fails loudly when the library
has not been built (there is no CPU fallback).
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "_lib" / "libkairos_b200.so"
HEADER_PATH = _PKG.parent / "include" / "kairos_b200.h"

KX_OK = 0
KX_ERR_INVALID = 1
KX_ERR_LOGIC = 2
KX_ERR_RUNTIME = 3
KX_ERR_CUDA = 4
KX_ERR_CAPACITY = 5
KX_ERR_LIVELOCK = 6

KX_MEM_HOST = 0
KX_MEM_DEVICE = 1
KX_MEM_HOST_MAPPED = 2  # kx_queue_upload: pinned host columns read in place (see kairos_b200.h)

SCHED = {"kairos": 0, "fcfs": 1, "topo_depth": 2, "oracle": 3}
DISPATCH = {"time_slot": 0, "round_robin": 1, "static_threshold": 2}


class KxError(RuntimeError):
    """Raised for a non-zero kx status; `code` maps to the reference's
    exception type (1 invalid_argument, 2 logic_error, 3 runtime_error)."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"[kx status {code}] {msg}")
        self.code = code


class kx_workflow_sizes(C.Structure):
    _fields_ = [("n_edges", C.c_int64), ("n_diagnostics", C.c_int64), ("instances", C.c_int64)]


class kx_instance(C.Structure):
    _fields_ = [("id", C.c_int32), ("pool", C.c_int32), ("capacity_tokens", C.c_double),
                ("decode_rate", C.c_double), ("prefill_rate", C.c_double),
                ("max_batch", C.c_int32), ("_pad", C.c_int32)]


class kx_dispatcher_config(C.Structure):
    _fields_ = [("policy", C.c_int32), ("oracle_expected_time", C.c_int32),
                ("slot_len", C.c_double), ("resume_watermark", C.c_double),
                ("static_threshold", C.c_double), ("default_expected_time", C.c_double)]


class kx_sched_config(C.Structure):
    _fields_ = [("n_pools", C.c_int32), ("n_instances", C.c_int32),
                ("instances", C.POINTER(kx_instance)), ("dispatcher", kx_dispatcher_config),
                ("queue_capacity", C.c_int64), ("max_agents", C.c_int32),
                ("slot_ring", C.c_int32), ("device", C.c_int32),
                ("log_capacity_per_pool", C.c_int32)]


class kx_queue_view(C.Structure):
    _fields_ = [("agent", C.c_void_p), ("prompt_tokens", C.c_void_p), ("app_start", C.c_void_p),
                ("queue_enter", C.c_void_p), ("msg_key", C.c_void_p), ("uid", C.c_void_p),
                ("kept_tokens", C.c_void_p), ("pure_exec", C.c_void_p)]


class kx_decision(C.Structure):
    _fields_ = [("time", C.c_double), ("predicted_peak", C.c_double), ("uid", C.c_uint64),
                ("queue_index", C.c_int64), ("agent", C.c_int32), ("target", C.c_int32),
                ("pool", C.c_int32), ("admitted", C.c_int32)]


class kx_engine_config(C.Structure):
    _fields_ = [("n_instances", C.c_int32), ("scheduler", C.c_int32),
                ("instances", C.POINTER(kx_instance)), ("dispatcher", kx_dispatcher_config),
                ("n_agents", C.c_int32), ("slot_ring", C.c_int32), ("topo_depth", C.c_void_p),
                ("dispatch_period", C.c_double), ("recompute_fraction", C.c_double),
                ("heap_capacity", C.c_int32), ("device", C.c_int32), ("max_events", C.c_uint64),
                ("warmup_seconds", C.c_double), ("agent_order", C.c_void_p),
                ("kairos_rebuild_interval", C.c_uint64)]


class kx_replica_batch(C.Structure):
    _fields_ = [("n_replicas", C.c_int32), ("_pad", C.c_int32)] + [
        (n, C.c_void_p) for n in ["wf_base", "arrival", "wf_offsets", "agent", "parent",
                                  "prompt_tokens", "target_tokens", "pure_exec", "remaining", "uid"]]


class kx_replica_results(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in [
        "call_order", "exec_start", "exec_end", "instance", "first_enqueue", "queue_seconds",
        "episodes", "preemptions", "wf_order", "wf_finish", "wf_output_tokens", "wf_calls",
        "scalars", "counts", "metrics", "histogram", "priority_keys", "table_versions"]]


class kx_convergence_config(C.Structure):
    _fields_ = [("min_samples", C.c_uint64), ("relative_threshold", C.c_double), ("window_cap", C.c_int64)]


class kx_phase_stat(C.Structure):
    _fields_ = [("name", C.c_char * 32), ("total_ms", C.c_double), ("launches", C.c_int64),
                ("alg_bytes", C.c_double)]


class kx_length_spec(C.Structure):
    _fields_ = [("kind", C.c_int32), ("_pad", C.c_int32), ("a", C.c_double), ("b", C.c_double),
                ("min_tokens", C.c_int64), ("max_tokens", C.c_int64)]


class kx_agent_spec(C.Structure):
    _fields_ = [("prompt_len", kx_length_spec), ("output_len", kx_length_spec),
                ("n_choice", C.c_int32), ("n_parallel", C.c_int32), ("choice_to", C.c_void_p),
                ("choice_p", C.c_void_p), ("parallel_to", C.c_void_p), ("feedback_target", C.c_int32),
                ("feedback_max_iterations", C.c_int32), ("feedback_probability", C.c_double)]


class kx_app_spec(C.Structure):
    _fields_ = [("entry", C.c_int32), ("n_members", C.c_int32), ("members", C.c_void_p),
                ("weight", C.c_double)]


class kx_workload_config(C.Structure):
    _fields_ = [("n_agents", C.c_int32), ("n_apps", C.c_int32), ("agents", C.POINTER(kx_agent_spec)),
                ("apps", C.POINTER(kx_app_spec)), ("arrival_kind", C.c_int32),
                ("entry_selection", C.c_int32), ("rate", C.c_double), ("n_trace", C.c_int64),
                ("trace", C.c_void_p), ("trace_scale", C.c_double), ("duration", C.c_double)]


# name -> (restype, argtypes)
_P = C.c_void_p
SIGNATURES = {
    "kx_abi_version": (C.c_int, []),
    "kx_last_error": (C.c_char_p, []),
    "kx_device_available": (C.c_int, []),
    "kx_sched_create": (C.c_int, [C.POINTER(kx_sched_config), C.POINTER(_P)]),
    "kx_sched_destroy": (C.c_int, [_P]),
    "kx_sched_stream": (C.c_int, [_P, C.POINTER(_P)]),
    "kx_sched_synchronize": (C.c_int, [_P]),
    "kx_set_scheduler": (C.c_int, [_P, C.c_int32]),
    "kx_set_agent_tables": (C.c_int, [_P, C.c_int32, _P, _P, _P, _P, C.c_uint64]),
    "kx_set_remaining_table": (C.c_int, [_P, C.c_uint64, C.c_int64, _P, _P, C.c_int32]),
    "kx_queue_upload": (C.c_int, [_P, C.c_int64, C.POINTER(kx_queue_view), C.c_int32]),
    "kx_queue_enqueue": (C.c_int, [_P, C.c_int64, C.POINTER(kx_queue_view), C.c_int32]),
    "kx_graph_release": (C.c_int, [_P]),
    "kx_queue_size": (C.c_int, [_P, C.POINTER(C.c_int64)]),
    "kx_queue_remove_admitted": (C.c_int, [_P]),
    "kx_score": (C.c_int, [_P, _P, _P, _P, C.c_int32]),
    "kx_order": (C.c_int, [_P]),
    "kx_order_fetch": (C.c_int, [_P, _P, _P, C.c_int32]),
    "kx_dispatch_round": (C.c_int, [_P, C.c_double]),
    "kx_dispatch_fetch": (C.c_int, [_P, _P, _P, _P, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "kx_tick": (C.c_int, [_P, C.c_double]),
    "kx_waiting_reserve": (C.c_int, [_P, C.c_int64]),
    "kx_waiting_upload": (C.c_int, [_P, C.c_int64, _P, C.POINTER(kx_queue_view)]),
    "kx_waiting_fetch": (C.c_int, [_P, C.c_int32, C.c_int64, _P, C.POINTER(C.c_int64)]),
    "kx_admissions_fetch": (C.c_int, [_P, _P, _P, C.POINTER(C.c_int64)]),
    "kx_rr_next": (C.c_int, [_P, _P, _P]),
    "kx_instances_set_live": (C.c_int, [_P, _P, _P, _P]),
    "kx_instances_get_live": (C.c_int, [_P, _P, _P, _P, _P]),
    "kx_ledger_try_place": (C.c_int, [_P, C.c_int32, C.c_double, C.c_double, C.c_double, C.c_double,
                                      C.POINTER(C.c_int32), C.POINTER(C.c_double),
                                      C.POINTER(C.c_int64)]),
    "kx_ledger_commit": (C.c_int, [_P, C.c_int32, C.c_uint64, C.c_double, C.c_double, C.c_double,
                                   C.c_double]),
    "kx_ledger_commit_batch": (C.c_int, [_P, C.c_int64, _P, _P, _P, _P, _P, _P, _P]),
    "kx_on_request_finished": (C.c_int, [_P, C.c_int32, C.c_uint64, C.c_double]),
    "kx_on_overload": (C.c_int, [_P, C.c_int32]),
    "kx_on_live_usage": (C.c_int, [_P, C.c_int32, C.c_double]),
    "kx_gc": (C.c_int, [_P, C.c_double]),
    "kx_ledger_read": (C.c_int, [_P, C.c_int32, C.POINTER(C.c_int64), _P, _P, C.POINTER(C.c_int32)]),
    "kx_state_checkpoint": (C.c_int, [_P]),
    "kx_state_restore": (C.c_int, [_P]),
    "kx_profile_enable": (C.c_int, [_P, C.c_int32]),
    "kx_profile_read": (C.c_int, [_P, C.POINTER(kx_phase_stat), C.c_int32, C.POINTER(C.c_int32)]),
    "kx_launch_count": (C.c_int64, []),
    "kx_replicas_run": (C.c_int, [C.POINTER(kx_engine_config), C.POINTER(kx_replica_batch),
                                  C.POINTER(kx_replica_results), C.POINTER(C.c_double)]),
    "kx_sorting_accuracy": (C.c_int, [C.c_int64, _P, _P, _P, C.c_int32, C.POINTER(C.c_uint64),
                                      C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "kx_aggregate_metrics": (C.c_int, [C.c_int32, _P, _P]),
    "kx_w1_matrix": (C.c_int, [C.c_int32, _P, _P, _P]),
    "kx_profiler_create": (C.c_int, [C.c_int32, C.POINTER(kx_convergence_config),
                                     C.POINTER(kx_convergence_config), C.c_int64, C.c_int32, C.POINTER(_P)]),
    "kx_profiler_destroy": (C.c_int, [_P]),
    "kx_profiler_record_execution": (C.c_int, [_P, C.c_int64, _P, _P]),
    "kx_profiler_record_remaining": (C.c_int, [_P, C.c_int64, _P, _P, _P, _P, _P]),
    "kx_profiler_read": (C.c_int, [_P, C.c_int32, C.c_int32, C.c_int64, _P, C.POINTER(C.c_int64),
                                   C.POINTER(C.c_uint64), C.POINTER(C.c_int32), C.POINTER(C.c_double)]),
    "kx_graph_capture_begin": (C.c_int, [_P]),
    "kx_graph_capture_end": (C.c_int, [_P]),
    "kx_graph_launch": (C.c_int, [_P]),
    "kx_builtin_agent_name": (C.c_char_p, [C.c_int32]),
    "kx_expected_exec_times": (C.c_int, [C.c_int32, C.c_void_p, C.c_void_p, C.c_int64, C.c_double, C.c_void_p]),
    "kx_realize_builtin": (C.c_int, [C.c_uint32, C.c_double, C.c_double, C.c_uint64, C.c_double,
                                     C.c_double, C.POINTER(_P)]),
    "kx_realize": (C.c_int, [C.POINTER(kx_workload_config), C.c_uint64, C.c_double, C.c_double,
                             C.POINTER(_P)]),
    "kx_realization_sizes": (C.c_int, [_P, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "kx_realization_copy": (C.c_int, [_P] + [_P] * 10),
    "kx_realization_free": (None, [_P]),
    "kx_orchestrator_dp": (C.c_int, [C.c_int64, _P, _P, _P, _P, C.c_double, C.c_double, C.c_uint64,
                                     _P, _P, _P, C.c_int32]),
    "kx_record_remaining": (C.c_int, [C.c_int64, _P, _P, _P, _P, _P, C.c_int32]),
    "kx_trace_parse": (C.c_int, [C.c_char_p, C.c_int64, C.c_int32, C.POINTER(_P)]),
    "kx_trace_free": (None, [_P]),
    "kx_trace_sizes": (C.c_int, [_P, C.POINTER(C.c_int64), C.POINTER(C.c_int32), C.POINTER(C.c_int64),
                                 C.POINTER(C.c_int64)]),
    "kx_trace_agents": (C.c_int, [_P, _P, _P]),
    "kx_trace_columns": (C.c_int, [_P] + [_P] * 8),
    "kx_trace_msg_id": (C.c_int, [_P, C.c_int64, _P, C.c_int64, C.POINTER(C.c_int64)]),
    "kx_trace_msg_spans": (C.c_int, [_P, C.c_int64, _P, _P, _P]),
    "kx_trace_format": (C.c_int, [_P, _P, C.c_int64, C.POINTER(C.c_int64)]),
    "kx_workflow_reconstruct": (C.c_int, [_P, C.POINTER(kx_workflow_sizes)]),
    "kx_workflow_fetch": (C.c_int, [_P] + [_P] * 10),
}

_lib = None


def load(path: str | os.PathLike | None = None) -> C.CDLL:
    """Load libkairos_b200.so (raises if it is missing: no fallback)."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path else LIB_PATH
    if not p.exists():
        raise RuntimeError(
            f"{p} is missing: build the CUDA library first (`make` or __graft_entry__.build()). "
            "The kairos_b200 scheduling path has no CPU fallback.")
    lib = C.CDLL(str(p))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.kx_abi_version() != 1:
        raise RuntimeError("ABI version mismatch")
    if path is None:
        _lib = lib
    return lib


def check(status: int) -> None:
    if status != KX_OK:
        msg = _lib.kx_last_error().decode() if _lib is not None else ""
        raise KxError(status, msg)


def ptr(a) -> int | None:
    """Address of a numpy array or torch tensor (None passes through)."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    return a.ctypes.data
