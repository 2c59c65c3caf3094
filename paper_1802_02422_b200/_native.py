"""ctypes binding of the C ABI in include/givf_b200.h.

The library is built in-tree (`make`, or `__graft_entry__.build()`) into
`paper_1802_02422_b200/_lib/libgivf_b200.so`.  There is no fallback: if the
library is missing or no CUDA device is present, the calls raise.
"""

from __future__ import annotations

import ctypes
import os

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib", "libgivf_b200.so")

GIVF_OK, GIVF_EINVAL, GIVF_ECUDA, GIVF_ENOMEM, GIVF_EINVARIANT = 0, 1, 2, 3, 4

# every symbol include/givf_b200.h declares
EXPORTS = (
    "givf_last_error",
    "givf_version",
    "givf_index_create",
    "givf_index_destroy",
    "givf_index_device_bytes",
    "givf_index_counters",
    "givf_search_topk",
    "givf_search_full",
    "givf_probe_scores",
    "givf_probe",
    "givf_merge_topk",
    "givf_plan_capacity",
    "givf_plan",
    "givf_search_planned",
    "givf_kernel_launches",
    "givf_profile_enable",
    "givf_profile_read",
    # include/givf_build.h
    "givf_assign_nearest",
    "givf_encode_rows",
    "givf_knn_exact",
)

STAGES = ("probe_gemm", "probe_select", "probe_recheck", "probe_full", "plan", "scan",
          "finish", "merge", "lut", "probe_sample", "plan_scores")


class IndexDesc(ctypes.Structure):
    _fields_ = [
        ("k", ctypes.c_int32),
        ("dim", ctypes.c_int32),
        ("groups", ctypes.c_int32),
        ("m", ctypes.c_int32),
        ("grouping", ctypes.c_int32),
        ("n", ctypes.c_int64),
        ("centroids", ctypes.c_void_p),
        ("alphas", ctypes.c_void_p),
        ("neighbor_ids", ctypes.c_void_p),
        ("norm_terms", ctypes.c_void_p),
        ("group_sizes", ctypes.c_void_p),
        ("region_offsets", ctypes.c_void_p),
        ("local_sizes", ctypes.c_void_p),
        ("local_lo", ctypes.c_void_p),
        ("point_ids", ctypes.c_void_p),
        ("codes", ctypes.c_void_p),
        ("const_bytes", ctypes.c_void_p),
        ("codewords", ctypes.c_void_p),
        ("rotation", ctypes.c_void_p),
        ("const_lo", ctypes.c_double),
        ("const_hi", ctypes.c_double),
    ]


class SearchParamsC(ctypes.Structure):
    _fields_ = [
        ("nprobe", ctypes.c_int32),
        ("tau", ctypes.c_double),
        ("candidates", ctypes.c_int64),
        ("ef_search", ctypes.c_int32),
        ("rerank", ctypes.c_int32),
        ("prune", ctypes.c_int32),
    ]


class SearchStatsC(ctypes.Structure):
    _fields_ = [
        ("regions_visited", ctypes.c_int64),
        ("subregions_visited", ctypes.c_int64),
        ("subregions_pruned", ctypes.c_int64),
        ("codes_scanned", ctypes.c_int64),
    ]


class EncodeDesc(ctypes.Structure):
    """givf_encode_desc (include/givf_build.h)."""

    _fields_ = [
        ("x", ctypes.c_void_p),
        ("order", ctypes.c_void_p),
        ("seg", ctypes.c_void_p),
        ("seg_region", ctypes.c_void_p),
        ("nseg", ctypes.c_int64),
        ("dim", ctypes.c_int32),
        ("l", ctypes.c_int32),
        ("m", ctypes.c_int32),
        ("grouping", ctypes.c_int32),
        ("centroids", ctypes.c_void_p),
        ("neighbor_ids", ctypes.c_void_p),
        ("alphas", ctypes.c_void_p),
        ("c_sq", ctypes.c_void_p),
        ("codewords", ctypes.c_void_p),
        ("cw_sq", ctypes.c_void_p),
        ("const_lo", ctypes.c_double),
        ("const_step", ctypes.c_double),
        ("pick", ctypes.c_void_p),
        ("codes", ctypes.c_void_p),
        ("const_bytes", ctypes.c_void_p),
        ("consts", ctypes.c_void_p),
    ]


class PlanItemC(ctypes.Structure):
    """givf_plan_item: one begun group of a plan in its global form."""

    _fields_ = [("group", ctypes.c_int32), ("len", ctypes.c_int32), ("base", ctypes.c_double)]


_lib = None


def load(path: str = LIB_PATH):
    """Load the native library once; raises if it is not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(
            f"givf_b200 native library not found at {path}; build it with `make` "
            "(or __graft_entry__.build()) -- there is no CPU fallback"
        )
    lib = ctypes.CDLL(path)
    vp, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
    lib.givf_last_error.restype = ctypes.c_char_p
    lib.givf_version.restype = ctypes.c_char_p
    lib.givf_index_create.argtypes = [ctypes.POINTER(IndexDesc), ctypes.c_int, ctypes.POINTER(vp)]
    lib.givf_index_destroy.argtypes = [vp]
    lib.givf_index_device_bytes.argtypes = [vp]
    lib.givf_index_device_bytes.restype = i64
    lib.givf_index_counters.argtypes = [vp, vp, i32]
    lib.givf_search_topk.argtypes = [vp, vp, i64, ctypes.POINTER(SearchParamsC), i32, vp, vp, vp, vp]
    lib.givf_search_full.argtypes = [vp, vp, i64, ctypes.POINTER(SearchParamsC), i64, vp, vp, vp, vp]
    lib.givf_probe.argtypes = [vp, vp, i64, i32, vp, vp, vp]
    lib.givf_probe_scores.argtypes = [vp, vp, i64, vp, vp, vp]
    lib.givf_merge_topk.argtypes = [vp, vp, i32, i64, i32, vp, vp, ctypes.c_int, vp]
    lib.givf_plan_capacity.argtypes = [vp, ctypes.POINTER(SearchParamsC), ctypes.POINTER(i64)]
    lib.givf_plan.argtypes = [vp, vp, i64, ctypes.POINTER(SearchParamsC), i64, vp, vp, vp, vp]
    lib.givf_search_planned.argtypes = [vp, vp, i64, ctypes.POINTER(SearchParamsC), vp, vp, i32,
                                        vp, vp, vp]
    lib.givf_kernel_launches.restype = i64
    lib.givf_profile_enable.argtypes = [ctypes.c_int]
    lib.givf_profile_read.argtypes = [vp, vp, i32]
    lib.givf_assign_nearest.argtypes = [vp, i64, vp, i32, i32, vp, vp, vp]
    lib.givf_encode_rows.argtypes = [ctypes.POINTER(EncodeDesc), vp]
    lib.givf_knn_exact.argtypes = [vp, i64, vp, i64, i32, i32, vp, vp, vp]
    _lib = lib
    return lib


def check(rc: int) -> None:
    """Map a status code to the reference's exception types."""
    if rc == GIVF_OK:
        return
    msg = _lib.givf_last_error().decode()
    if rc == GIVF_EINVAL:
        raise ValueError(msg)
    if rc == GIVF_EINVARIANT:
        from .errors import InvariantError

        raise InvariantError(msg)
    if rc == GIVF_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(f"givf_b200 CUDA error: {msg}")


def kernel_launches() -> int:
    return int(load().givf_kernel_launches())


def profile_enable(on: bool = True) -> None:
    load().givf_profile_enable(1 if on else 0)


def profile_read() -> dict:
    """{stage: (ms, launches)} since the last read (synchronises)."""
    import numpy as np

    ms = np.zeros(len(STAGES), np.float64)
    cnt = np.zeros(len(STAGES), np.int64)
    check(load().givf_profile_read(ms.ctypes.data, cnt.ctypes.data, len(STAGES)))
    return {name: (float(ms[i]), int(cnt[i])) for i, name in enumerate(STAGES)}
