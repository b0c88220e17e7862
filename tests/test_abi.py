"""The C-ABI library loads and exports every symbol include/*.h declares
(no compute calls: runs without a GPU)."""
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "disttrain_b200.h")).read()
    return sorted(set(re.findall(r"\b(dtb_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_hot_path():
    syms = declared_symbols()
    for must in ("dtb_intra_partition", "dtb_inter_reorder", "dtb_disaggregated_reorder",
                 "dtb_model_orchestration", "dtb_reorder_stream_dev", "dtb_schedule"):
        assert must in syms


def test_library_exports_every_declared_symbol():
    import ctypes
    from paper_2408_04275_b200 import native
    if not os.path.exists(native.LIB_PATH):
        import __graft_entry__
        __graft_entry__.build()
    lib = ctypes.CDLL(native.LIB_PATH)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    assert lib.dtb_abi_version() == 1


def test_oracles_export_the_same_abi(ref, port):
    names = [s[len("dtb_"):] for s in declared_symbols()]
    device_only = {"schedule_batch_dev", "inter_reorder_batch_dev", "reorder_stream_dev",
                   "orchestration_shard_dev", "best_reduce_dev", "infeasible_reason_text",
                   "intra_stream_dev", "ingest_trace_dev",
                   # multi-GPU plumbing (CUDA IPC peer groups)
                   "peer_buffer_create", "peer_buffer_destroy", "peer_group_open",
                   "peer_group_close", "shard_range", "reorder_stream_shard_dev",
                   # CUDA graphs of a device call
                   "reorder_stream_graph_create", "graph_launch", "graph_destroy"}
    # trace ingest is pinned by the compiled reference and nlohmann itself
    # (tests/test_ingest.py); the C port does not restate a JSON library
    ref_only = {"ingest_trace",
                # warning log: the compiled reference's own sink; the C port
                # restates arithmetic, not the string log
                "warnings_enable", "warnings_count", "warning_at", "warnings_clear"}
    for name in names:
        if name in device_only:
            continue
        assert ref.lib.has(name), "mmref_" + name
        if name not in ref_only:
            assert port.lib.has(name), "mmport_" + name


def test_product_path_fails_loudly_without_the_library(tmp_path, monkeypatch):
    """No CPU fallback: a missing libdisttrain_b200.so is an error."""
    from paper_2408_04275_b200 import native
    monkeypatch.setattr(native, "LIB_PATH", str(tmp_path / "missing.so"))
    monkeypatch.setattr(native, "_lib", None)
    with pytest.raises(FileNotFoundError):
        native.library()
