"""ctypes binding of libsemisort_b200.so (the C ABI in include/semisort_b200.h).

The library is built in-tree by ``_build.build()`` (``__graft_entry__.build``).
There is no fallback: if the shared library is missing, every entry point
raises ``RuntimeError`` naming the build command.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

from .errors import ConfigurationError, ContractError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsemisort_b200.so")

SS_OK, SS_ERR_CONFIG, SS_ERR_CONTRACT, SS_ERR_RESOURCE, SS_ERR_COMM = range(5)
SS_MODE_EQ, SS_MODE_LT = 0, 1
SS_AGG_COUNT, SS_AGG_SUM64 = 0, 1

u64, u32, i32, vp = C.c_uint64, C.c_uint32, C.c_int, C.c_void_p


class SSParams(C.Structure):
    _fields_ = [("input_size", u64), ("light_buckets", u32), ("light_bits", u32),
                ("subarray_len", u64), ("base_case_cutoff", u64), ("max_heavy", u32),
                ("sample_factor", u32), ("seed", u64), ("sample_count", u64),
                ("heavy_threshold_int", u64), ("heavy_threshold", C.c_double)]


class SSTelemetry(C.Structure):
    _fields_ = [("max_depth", u64), ("nodes", u64), ("scratch_allocations", u64),
                ("scratch_moves", u64), ("bucket_assignments", u64),
                ("matrix_cells_by_level", u64 * 65), ("kernel_launches", u64), ("levels", u64),
                ("leaves_smem", u64), ("leaves_global", u64), ("nodes_folded", u64), ("fold_records", u64), ("timing", C.c_int32),
                ("reserved", C.c_int32), ("phase_ms", C.c_double * 8)]


PHASES = ("sample", "count", "scan", "distribute", "copy_back", "children", "leaves", "other")

_SIGS = {
    "ss_last_error": (C.c_char_p, []),
    "ss_version": (i32, []),
    "ss_semisort_workspace_bytes": (u64, [u64, u32, u32, C.POINTER(SSParams)]),
    "ss_semisort": (i32, [vp, vp, u64, u32, u32, i32, i32, C.POINTER(SSParams), vp, u64,
                          C.POINTER(SSTelemetry), vp]),
    "ss_local_refine": (i32, [vp, vp, vp, vp, u64, u32, u32, i32, i32, C.POINTER(SSParams),
                              C.POINTER(C.c_int64), u32, i32, u32, vp, u64, C.POINTER(SSTelemetry), vp]),
    "ss_aggregate_workspace_bytes": (u64, [u64, u32, u32, C.POINTER(SSParams)]),
    "ss_collect_reduce": (i32, [vp, vp, u64, u32, u32, i32, i32, C.POINTER(SSParams), vp, u64,
                                C.POINTER(u64), C.POINTER(SSTelemetry), vp]),
    "ss_histogram": (i32, [vp, u64, u32, i32, C.POINTER(SSParams), vp, u64, C.POINTER(u64),
                           C.POINTER(SSTelemetry), vp]),
    "ss_result_copy": (i32, [vp, u64, u32, u32, C.POINTER(SSParams), vp, vp, u64, vp]),
    "ss_phase_workspace_bytes": (u64, [u64, u32, u32, C.POINTER(SSParams)]),
    "ss_sample_heavy": (i32, [vp, u64, u32, C.POINTER(SSParams), u64, vp, C.POINTER(u32), vp, u64, vp]),
    "ss_assign_bucket_ids": (i32, [vp, u64, u32, i32, C.POINTER(SSParams), u32, vp, u32, vp, vp, u64, vp]),
    "ss_count_matrix": (i32, [vp, vp, u64, u32, i32, C.POINTER(SSParams), u32, vp, u32, u32, vp, vp, u64, vp]),
    "ss_column_scan": (i32, [vp, u64, u32, vp, vp, vp, u64, vp]),
    "ss_distribute": (i32, [vp, vp, vp, vp, vp, u64, u32, u32, i32, C.POINTER(SSParams), u32, vp, u32, u32,
                            vp, vp, u64, vp]),
    "ss_base_case": (i32, [vp, vp, u64, u32, u32, i32, i32, vp, u64, vp]),
    "ss_base_case_workspace_bytes": (u64, [u64, u32, u32]),
    "ss_partition": (i32, [vp, vp, u64, u32, u32, u32, vp, vp, C.POINTER(u64), vp, u64, vp]),
    "ss_partition_workspace_bytes": (u64, [u64, u32]),
    "ss_generate": (i32, [i32, C.c_double, u64, u64, u64, u32, u64, i32, vp, vp, u32, i32, u32, vp]),
    "ss_validate_indexed": (i32, [vp, vp, vp, u64, u32, u32, u64, vp, u64, C.POINTER(C.c_int32), vp]),
    "ss_validate_workspace_bytes": (u64, [u64]),
    "ss_count_distinct": (i32, [vp, u64, u32, vp, u64, C.POINTER(u64), vp]),
    "ss_count_distinct_workspace_bytes": (u64, [u64]),
    "ss_csr_workspace_bytes": (u64, [u64, u64, C.POINTER(SSParams)]),
    "ss_graph_transpose": (i32, [u64, u64, vp, vp, vp, vp, C.POINTER(SSParams), vp, u64,
                                 C.POINTER(SSTelemetry), vp]),
    "ss_csr_from_edges": (i32, [u64, u64, vp, vp, vp, vp, C.POINTER(SSParams), vp, u64,
                                C.POINTER(SSTelemetry), vp]),
    "ss_records_unpack": (i32, [vp, u64, u32, u32, vp, vp, vp]),
    "ss_records_pack": (i32, [vp, vp, u64, u32, u32, vp, vp]),
    "ss_bytes_hash": (i32, [vp, u64, vp, u64, vp, vp, vp]),
    "ss_bytes_chunk": (i32, [vp, vp, u64, u64, vp, vp]),
    "ss_bytes_equal": (i32, [vp, vp, vp, u64, vp, C.POINTER(C.c_uint64), vp]),
    "ss_partition_pairs": (i32, [vp, vp, u64, u32, u32, vp, C.POINTER(u64), vp, u64, vp]),
    "ss_partition_pairs_workspace_bytes": (u64, [u64, u32]),
    "ss_semisort_pairs": (i32, [vp, u64, u32, i32, i32, C.POINTER(SSParams), vp, vp, u64,
                                C.POINTER(SSTelemetry), vp]),
    "ss_semisort_pairs_workspace_bytes": (u64, [u64, u32, C.POINTER(SSParams), i32]),
    "ss_params_for_input": (i32, [u64, C.POINTER(SSParams), C.POINTER(SSParams)]),
    "ss_nccl_unique_id": (i32, [C.c_char_p]),
    "ss_nccl_comm_init": (i32, [C.c_char_p, i32, i32, C.POINTER(vp)]),
    "ss_nccl_comm_destroy": (i32, [vp]),
    "ss_dist_semisort": (i32, [vp, u32, u32, vp, vp, u64, u32, i32, i32, C.POINTER(SSParams), vp, vp, u64, vp,
                               u64, C.POINTER(u64), C.POINTER(SSTelemetry), vp]),
    "ss_dist_semisort_workspace_bytes": (u64, [u64, u32, u32, C.POINTER(SSParams)]),
    "ss_validate_shard": (i32, [i32, C.c_double, u64, u64, i32, vp, vp, u64, u32, u32, u32, vp, u64,
                                C.POINTER(u64), vp]),
    "ss_index_fingerprint": (i32, [u64, u64, vp, u64, C.POINTER(u64), vp]),
}

EXPORTS = tuple(_SIGS)

_lock = threading.Lock()
_lib = None


def lib():
    """The loaded library (loads once; raises if it was never built)."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise RuntimeError(
                        f"{LIB_PATH} is missing: build it with `python -m paper_2304_10078_b200._build` "
                        "(or __graft_entry__.build()); there is no CPU fallback")
                handle = C.CDLL(LIB_PATH)
                for name, (res, args) in _SIGS.items():
                    fn = getattr(handle, name)
                    fn.restype = res
                    fn.argtypes = args
                _lib = handle
    return _lib


def check(rc: int) -> None:
    """Map a C status to the reference's exception types (errors.py:4-13)."""
    if rc == SS_OK:
        return
    msg = lib().ss_last_error().decode("utf-8", "replace")
    if rc == SS_ERR_CONFIG:
        raise ConfigurationError(msg)
    if rc == SS_ERR_CONTRACT:
        raise ContractError(msg)
    if rc == SS_ERR_RESOURCE:
        if "out of memory" in msg or "workspace too small" in msg:
            raise MemoryError(msg)
        raise RuntimeError(msg)
    raise RuntimeError(f"collective failure: {msg}")
