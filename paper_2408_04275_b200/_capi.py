"""ctypes mirror of include/disttrain_b200.h.

One `Library` class binds any shared object exporting that ABI under a
prefix: the product (`libdisttrain_b200.so`, prefix ``dtb_``) and — in tests
only — the oracles under ``oracle/`` (``mmref_`` / ``mmport_``).  No
fallback: a missing symbol or library raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

c_i32, c_i64, c_f64, c_u8 = C.c_int32, C.c_int64, C.c_double, C.c_uint8
P = C.POINTER


class Arch(C.Structure):
    _fields_ = [("layers", c_i32), ("heads", c_i32), ("groups", c_i32),
                ("reserved", c_i32), ("hidden", c_i64), ("ffn_hidden", c_i64)]


class ModuleMemory(C.Structure):
    _fields_ = [("param_grad_bytes", c_f64), ("optimizer_bytes", c_f64),
                ("activation_bytes_per_mb", c_f64)]


class ModuleSpec(C.Structure):
    _fields_ = [("arch", Arch), ("mem", ModuleMemory), ("frozen", c_i32),
                ("reserved", c_i32)]


class ModelSpec(C.Structure):
    _fields_ = [("unit", ModuleSpec * 3), ("seq_len", c_i64),
                ("frozen_backward_factor", c_f64), ("dp_sync_seconds", c_f64)]


class ClusterSpec(C.Structure):
    _fields_ = [("total_gpus", c_i32), ("gpus_per_node", c_i32),
                ("peak_flops", c_f64), ("gpu_mem_bytes", c_f64),
                ("intra_node_bw", c_f64), ("inter_node_bw", c_f64)]


class ProfileRow(C.Structure):
    _fields_ = [("module", c_i32), ("tp", c_i32), ("has_bwd", c_i32),
                ("reserved", c_i32), ("token_load", c_f64), ("fwd_s", c_f64),
                ("bwd_s", c_f64)]


class CostBook(C.Structure):
    _fields_ = [("rows", P(ProfileRow)), ("n_rows", c_i64),
                ("analytic_efficiency", c_f64),
                ("analytic_bwd_fwd_ratio", c_f64)]


class Parallelism(C.Structure):
    _fields_ = [("tp", c_i32), ("dp", c_i32), ("pp", c_i32)]


class Plan(C.Structure):
    _fields_ = [("unit", Parallelism * 3), ("vpp", c_i32),
                ("global_batch", c_i64)]


class WorkloadStats(C.Structure):
    _fields_ = [("seq_len", c_i64), ("mean_encoder_tokens", c_f64),
                ("mean_generator_tokens", c_f64)]


class Samples(C.Structure):
    _fields_ = [("n", c_i64), ("text_tokens", P(c_i32)),
                ("image_offsets", P(c_i32)), ("image_tokens", P(c_i32)),
                ("audio_offsets", P(c_i32)), ("audio_tokens", P(c_i32))]


class Microbatches(C.Structure):
    _fields_ = [("n", c_i64), ("encoder_tokens", P(c_i64)),
                ("generator_tokens", P(c_i64)), ("sample_count", P(c_i32))]


class ReorderMode(C.Structure):
    _fields_ = [("intra", c_i32), ("inter", c_i32), ("sort_order", c_i32)]


class Tuple(C.Structure):
    _fields_ = [("tp_me", c_i32), ("dp_me", c_i32), ("tp_lm", c_i32),
                ("dp_lm", c_i32), ("tp_mg", c_i32), ("dp_mg", c_i32)]


class PredictedTimes(C.Structure):
    _fields_ = [("t_warm", c_f64), ("t_steady", c_f64), ("t_iter", c_f64)]


class Candidate(C.Structure):
    _fields_ = [("tuple", Tuple), ("feasible", c_i32), ("reason", c_i32),
                ("plan", Plan), ("times", PredictedTimes), ("cont_x", c_f64),
                ("cont_y", c_f64), ("cont_z", c_f64), ("cont_t_iter", c_f64)]


class OrchestrationResult(C.Structure):
    _fields_ = [("best", Plan), ("times", PredictedTimes),
                ("candidates_evaluated", c_i64), ("solve_seconds", c_f64)]


class MemoryReport(C.Structure):
    _fields_ = [("bytes_per_gpu", c_f64 * 3), ("fits", c_i32 * 3),
                ("pass_", c_i32), ("capacity_bytes", c_f64)]


class TraceCsr(C.Structure):
    _fields_ = [("cap_samples", C.c_int64), ("cap_image", C.c_int64), ("cap_audio", C.c_int64),
                ("text_tokens", C.c_void_p), ("image_offsets", C.c_void_p),
                ("image_tokens", C.c_void_p), ("audio_offsets", C.c_void_p),
                ("audio_tokens", C.c_void_p)]


class TraceResult(C.Structure):
    _fields_ = [("n_samples", C.c_int64), ("n_image", C.c_int64), ("n_audio", C.c_int64),
                ("n_lines", C.c_int64), ("error_kind", C.c_int32), ("error_line", C.c_int32),
                ("error_reason", C.c_int32), ("reserved", C.c_int32)]


class ReorderReport(C.Structure):
    _fields_ = [("output_order", P(c_i32)), ("group_load_before", P(c_f64)),
                ("group_load_after", P(c_f64)), ("t_iter_before", c_f64),
                ("t_iter_after", c_f64)]


class PeerHandle(C.Structure):
    _fields_ = [("bytes", C.c_ubyte * 64)]


VP = C.c_void_p
_SIGS = {
    "last_error": (C.c_char_p, []),
    "abi_version": (C.c_int, []),
    "context_create": (c_i32, [c_i32, P(VP)]),
    "warnings_enable": (c_i32, [VP, c_i32]),
    "warnings_count": (c_i64, [VP]),
    "warning_at": (C.c_char_p, [VP, c_i64]),
    "warnings_clear": (c_i32, [VP]),
    "context_destroy": (c_i32, [VP]),
    "cost_model_create": (c_i32, [VP, P(ModelSpec), P(ClusterSpec),
                                  P(CostBook), P(VP)]),
    "cost_model_destroy": (c_i32, [VP]),
    "cost_sizes": (c_i32, [VP, P(Samples), P(c_i64)]),
    "unit_times": (c_i32, [VP, VP, c_i32, c_i32, c_i64, P(c_f64), P(c_f64),
                           P(c_f64)]),
    "memory_check": (c_i32, [VP, VP, P(Plan), P(MemoryReport)]),
    "build_stage_times": (c_i32, [VP, VP, P(Plan), P(Microbatches), P(c_f64),
                                  P(c_f64)]),
    "microbatch_fwd_keys": (c_i32, [VP, VP, P(Plan), P(Microbatches),
                                    P(c_f64)]),
    "compute_stats": (c_i32, [VP, P(Samples), c_i64, P(WorkloadStats)]),
    "intra_partition": (c_i32, [VP, P(c_f64), c_i64, c_i32, c_i32, c_i32,
                                P(c_i32), P(c_i64)]),
    "block_group_loads": (c_i32, [VP, P(c_f64), P(c_i32), c_i64, c_i32,
                                  P(c_f64)]),
    "select_min": (c_i32, [VP, P(c_f64), c_i64, P(c_i32), c_i64, c_i32,
                           P(c_i32)]),
    "select_closest": (c_i32, [VP, P(c_f64), c_i64, P(c_i32), c_i64, c_i32,
                               c_f64, P(c_i32)]),
    "schedule": (c_i32, [VP, P(c_f64), P(c_f64), c_i32, c_i32, c_i32,
                         P(c_i32), P(c_i32), P(c_i32), P(c_i32), P(c_f64),
                         P(c_f64), P(c_f64), P(c_f64)]),
    "get_intervals": (c_i32, [VP, c_i64, P(c_i32), P(c_i32), P(c_i32),
                              P(c_i32), P(c_f64), P(c_f64), P(c_i64),
                              P(c_f64), P(c_f64), P(c_i64), P(c_i32)]),
    "interval_windows": (c_i32, [VP, P(c_f64), P(c_f64), c_i32, c_i32,
                                 P(c_f64)]),
    "exhaustive_order": (c_i32, [VP, P(c_f64), P(c_f64), c_i32, c_i32, c_i32, P(c_f64),
                                 P(c_i32), P(c_f64)]),
    "schedule_batch": (c_i32, [VP, c_i64, P(c_f64), P(c_f64), c_i32, c_i32,
                               c_i32, P(c_f64), P(c_f64)]),
    "schedule_batch_dev": (c_i32, [VP, c_i64, VP, VP, c_i32, c_i32, c_i32,
                                   VP, VP, VP]),
    "simulate_iteration": (c_i32, [VP, VP, P(Plan), c_i32, P(c_i64),
                                   P(Microbatches), P(c_f64), P(c_f64),
                                   P(c_i32), P(c_f64), P(c_f64)]),
    "inter_reorder": (c_i32, [VP, P(c_f64), P(c_f64), c_i32, c_i32,
                              P(c_f64), c_i32, P(c_i32)]),
    "inter_reorder_batch": (c_i32, [VP, c_i64, P(c_f64), P(c_f64), c_i32,
                                    c_i32, P(c_f64), c_i32, P(c_i32)]),
    "inter_reorder_batch_dev": (c_i32, [VP, c_i64, VP, VP, c_i32, c_i32, VP,
                                        c_i32, VP, VP]),
    "disaggregated_reorder": (c_i32, [VP, VP, P(Plan), P(ReorderMode),
                                      P(Samples), P(ReorderReport)]),
    "reorder_stream": (c_i32, [VP, VP, P(Plan), P(ReorderMode), P(Samples),
                               c_i64, P(c_i32), P(c_f64), P(c_f64), P(c_f64),
                               P(c_f64), P(c_u8)]),
    "reorder_stream_dev": (c_i32, [VP, VP, P(Plan), P(ReorderMode),
                                   P(Samples), c_i64, VP, VP, VP, VP, VP, VP,
                                   VP]),
    "intra_stream_dev": (c_i32, [VP, c_i64, c_i32, c_i32, P(Samples), c_i64, VP, VP, VP, VP,
                                 VP]),
    "predict_times": (c_i32, [VP, VP, P(WorkloadStats), P(Plan), c_i64,
                              P(PredictedTimes)]),
    "enumerate_parallelism": (c_i32, [VP, P(ClusterSpec), c_i64, P(c_i64),
                                      P(Tuple), c_i64]),
    "solve_subproblem": (c_i32, [VP, VP, P(WorkloadStats), P(Tuple), c_i64,
                                 c_i64, c_i32, P(Candidate)]),
    "brute_force_oracle": (c_i32, [VP, VP, P(WorkloadStats), c_i64, c_i32, c_i32,
                                   P(OrchestrationResult)]),
    "rigid_baseline": (c_i32, [VP, VP, P(WorkloadStats), c_i64, c_i32, P(Plan)]),
    "ingest_trace": (c_i32, [VP, C.c_char_p, c_i64, c_i64, P(TraceCsr), P(TraceResult)]),
    "ingest_trace_dev": (c_i32, [VP, VP, c_i64, c_i64, P(TraceCsr), P(TraceResult)]),
    "model_orchestration": (c_i32, [VP, VP, P(WorkloadStats), c_i64, c_i32,
                                    P(OrchestrationResult), P(Candidate),
                                    c_i64]),
    "orchestration_shard_dev": (c_i32, [VP, VP, P(WorkloadStats), c_i64,
                                        c_i32, c_i64, c_i64, VP, VP, VP]),
    "best_reduce_dev": (c_i32, [VP, VP, c_i64, VP, VP]),
    "peer_buffer_create": (c_i32, [VP, c_i64, P(VP), P(PeerHandle)]),
    "peer_buffer_destroy": (c_i32, [VP, VP]),
    "peer_group_open": (c_i32, [VP, c_i32, c_i32, VP, c_i64, P(PeerHandle), P(VP)]),
    "peer_group_close": (c_i32, [VP]),
    "shard_range": (c_i32, [c_i64, c_i32, c_i32, P(c_i64), P(c_i64)]),
    "reorder_stream_shard_dev": (c_i32, [VP, VP, P(Plan), P(ReorderMode), P(Samples), c_i64, VP,
                                         VP, VP, VP, VP, VP, VP]),
    "reorder_stream_graph_create": (c_i32, [VP, VP, P(Plan), P(ReorderMode), P(Samples), c_i64,
                                            VP, VP, VP, VP, VP, VP, VP, P(VP)]),
    "graph_launch": (c_i32, [VP, VP]),
    "graph_destroy": (c_i32, [VP]),
    # oracle-only extras (CPU baselines)
    "set_threads": (None, [C.c_int]),
    "stream_prepare": (c_i32, [P(Samples), c_i64, P(VP)]),
    "stream_destroy": (c_i32, [VP]),
    "stream_run": (c_i32, [VP, VP, P(Plan), P(ReorderMode), c_i64, c_i64,
                           P(c_i32), P(c_f64), P(c_f64), P(c_f64), P(c_f64)]),
    "model_orchestration_mt": (c_i32, [VP, VP, P(WorkloadStats), c_i64,
                                       c_i32, P(OrchestrationResult)]),
}

STATUS_NAMES = {
    0: "OK", 1: "InternalError", 2: "KTooLargeError", 3: "IndivisibleVppError",
    4: "BatchSizeMismatchError", 5: "ConfigError", 6: "EmptyProfileError",
    7: "InfeasibleError", 8: "CapExceededError", 9: "TraceError", 100: "InvalidArgument",
    101: "CudaError",
}


class Library:
    """Binds every ABI function present in `path` under `prefix`."""

    def __init__(self, path: str, prefix: str):
        if not os.path.exists(path):
            raise FileNotFoundError(f"native library not built: {path}")
        self.path = path
        self.prefix = prefix
        self.lib = C.CDLL(path, mode=C.RTLD_LOCAL)
        self.fns = {}
        for name, (res, args) in _SIGS.items():
            try:
                fn = getattr(self.lib, prefix + name)
            except AttributeError:
                continue
            fn.restype = res
            fn.argtypes = args
            self.fns[name] = fn

    def has(self, name: str) -> bool:
        return name in self.fns

    def __getattr__(self, name):
        fns = self.__dict__.get("fns")
        if fns is not None and name in fns:
            return fns[name]
        raise AttributeError(f"{self.prefix}{name} not exported by {self.__dict__.get('path')}")


def ptr(a: np.ndarray | None, ctype):
    """Pointer to a contiguous numpy array (None -> NULL)."""
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"], "array must be contiguous"
    return a.ctypes.data_as(P(ctype))
