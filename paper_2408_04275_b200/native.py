"""Loads the sm_100a product library (libdisttrain_b200.so, built in-tree).

No fallback of any kind: a missing library, a missing symbol or a missing
GPU raises immediately.
"""
from __future__ import annotations

import os

from . import _capi
from .api import Planner

HERE = os.path.dirname(os.path.abspath(__file__))
# DTB_LIB_PATH: an experiment build (build.py with DTB_DEFINES) for tools/
LIB_PATH = os.environ.get("DTB_LIB_PATH") or os.path.join(HERE, "libdisttrain_b200.so")
_lib = None


def library() -> _capi.Library:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise FileNotFoundError(
                f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
        _lib = _capi.Library(LIB_PATH, "dtb_")
        missing = [n for n in REQUIRED if not _lib.has(n)]
        if missing:
            raise ImportError(f"libdisttrain_b200.so lacks {missing}")
    return _lib


REQUIRED = [
    "last_error", "abi_version", "context_create", "context_destroy", "cost_model_create",
    "cost_model_destroy", "cost_sizes", "unit_times", "memory_check", "build_stage_times",
    "microbatch_fwd_keys", "compute_stats", "intra_partition", "block_group_loads",
    "select_min", "select_closest", "schedule", "get_intervals", "interval_windows",
    "schedule_batch", "schedule_batch_dev", "exhaustive_order", "brute_force_oracle",
    "rigid_baseline", "simulate_iteration", "inter_reorder",
    "inter_reorder_batch", "inter_reorder_batch_dev", "disaggregated_reorder", "reorder_stream",
    "reorder_stream_dev", "intra_stream_dev", "predict_times", "enumerate_parallelism", "solve_subproblem",
    "model_orchestration", "orchestration_shard_dev", "best_reduce_dev",
    "peer_buffer_create", "peer_buffer_destroy", "peer_group_open", "peer_group_close",
    "shard_range", "reorder_stream_shard_dev", "reorder_stream_graph_create", "graph_launch",
    "graph_destroy", "warnings_enable", "warnings_count", "warning_at", "warnings_clear",
]


def planner(device: int = 0) -> Planner:
    return Planner(library(), device)
