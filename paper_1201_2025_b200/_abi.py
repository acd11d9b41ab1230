"""ctypes binding of the C-ABI in include/hsad_gpu.h (libhsad_b200.so).

This is the binding a Python caller (tests, bench.py) uses; the C++ drop-in for
the reference's own C++ API lives in include/hsad/hsad_b200.hpp. There is no CPU
fallback: importing this module without the built library raises.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

PKG = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("HSAD_B200_LIB", PKG / "libhsad_b200.so"))

HSAD_OK = 0
HSAD_E_INVALID_VALUE = 2
HSAD_E_SIZE_MISMATCH = 3
HSAD_E_NON_FINITE_VALUE = 4
HSAD_E_OUT_OF_BOUNDS = 5
HSAD_E_UNSUPPORTED_ORDER = 6
HSAD_E_TOO_SHORT = 8
HSAD_E_TARGET_TOO_LARGE = 10
HSAD_E_TOO_FEW_SAMPLES = 12
HSAD_E_SINGULAR_AFTER_RIDGE = 13
HSAD_E_CONFIG_MISMATCH = 16
HSAD_E_DIMENSION_MISMATCH = 19
HSAD_E_DEGENERATE_TRUTH = 20
HSAD_E_CUDA = 64
HSAD_E_UNSUPPORTED = 65
HSAD_E_NCCL = 66

HSAD_LRX, HSAD_DWRX, HSAD_DWEST = 0, 1, 2
WINDOW_SINGLE, WINDOW_DUAL = 0, 1

# symbols include/hsad_gpu.h declares (checked by tests/test_abi.py)
EXPORTED = [
    "hsad_abi_version", "hsad_status_name", "hsad_last_error_message", "hsad_get_limits",
    "hsad_device_check", "hsad_mirror_index", "hsad_window_validate", "hsad_daubechies_filters",
    "hsad_reduce", "hsad_detect", "hsad_detect_multi", "hsad_strip_rows", "hsad_row_quantum",
    "hsad_decode_status", "hsad_pipeline_host", "hsad_reduce_detect",
    "hsad_read_cube", "hsad_reduce_raw", "hsad_pipeline_raw", "hsad_pipeline_sharded", "hsad_roc", "hsad_top_k", "hsad_adaptive_threshold", "hsad_render_pgm",
    "hsad_strip_plan", "hsad_gather_maps", "hsad_nccl_available", "hsad_nccl_unique_id",
    "hsad_nccl_comm_init_rank", "hsad_nccl_comm_init_all", "hsad_nccl_comm_destroy",
    "hsad_last_reduce_detect_fused", "hsad_dwest_pairs", "hsad_dual_window_samples",
    "hsad_encode_score_map",
]

HSAD_BSQ, HSAD_BIL, HSAD_BIP = 0, 1, 2


class Window(C.Structure):
    _fields_ = [("mode", C.c_int32), ("single_size", C.c_int32), ("inner_size", C.c_int32),
                ("outer_size", C.c_int32)]


class Request(C.Structure):
    _fields_ = [("algorithm", C.c_int32), ("window", Window), ("guard", C.c_int32),
                ("ridge", C.c_double), ("eigen_fraction", C.c_double),
                ("d_scores", C.c_void_p), ("score_bytes", C.c_int32),
                ("d_eigcount", C.c_void_p)]


class PixelError(C.Structure):
    _fields_ = [("code", C.c_int32), ("row", C.c_int64), ("col", C.c_int64)]


class CubeHeader(C.Structure):  # hsad_cube_header
    _fields_ = [("samples", C.c_int32), ("lines", C.c_int32), ("bands", C.c_int32),
                ("interleave", C.c_int32), ("data_type_code", C.c_int32), ("byte_order", C.c_int32)]


class RocSummary(C.Structure):  # hsad_roc_summary
    _fields_ = [("positives", C.c_uint64), ("negatives", C.c_uint64),
                ("auc_twice_num", C.c_uint64), ("auc", C.c_double), ("distinct", C.c_uint64)]


class MapDesc(C.Structure):  # hsad_map_desc
    _fields_ = [("d_strip", C.c_void_p), ("d_full", C.c_void_p), ("elem_bytes", C.c_int32)]


class Limits(C.Structure):
    _fields_ = [("max_detect_bands", C.c_int32), ("max_window", C.c_int32),
                ("max_reduce_bands", C.c_int32)]


def load(path: Path | str = LIB_PATH) -> C.CDLL:
    path = Path(path)
    if not path.exists():
        raise ImportError(
            f"{path} is missing: build it with `make -C paper_1201_2025_b200` "
            "(or __graft_entry__.build()); there is no CPU fallback")
    lib = C.CDLL(str(path))
    I32, I64, VP, D = C.c_int32, C.c_int64, C.c_void_p, C.c_double
    P = C.POINTER
    sig = {
        "hsad_abi_version": (I32, []),
        "hsad_status_name": (C.c_char_p, [I32]),
        "hsad_last_error_message": (C.c_char_p, []),
        "hsad_get_limits": (None, [P(Limits)]),
        "hsad_device_check": (I32, []),
        "hsad_mirror_index": (I32, [I32, I32]),
        "hsad_window_validate": (I32, [P(Window)]),
        "hsad_daubechies_filters": (I32, [I32, P(D), P(D), P(I32)]),
        "hsad_reduce": (I32, [VP, I32, I64, I64, I32, I32, I32, VP, I32, VP]),
        "hsad_detect": (I32, [VP, I32, I64, I64, I32, P(Request), P(PixelError), VP]),
        "hsad_detect_multi": (I32, [VP, I32, I64, I64, I32, I64, I64, I64, I64, P(Request), I32,
                                    VP, P(PixelError), VP]),
        "hsad_reduce_detect": (I32, [VP, I64, I64, I32, I32, I32, I64, I64, I64, I64, VP,
                                     P(Request), I32, VP, P(PixelError), VP]),
        "hsad_strip_rows": (I32, [I64, I64, I64, P(Request), I32, P(I64), P(I64)]),
        "hsad_row_quantum": (I64, [I64, I64]),
        "hsad_decode_status": (I32, [C.c_uint64, I64, P(PixelError)]),
        "hsad_pipeline_host": (I32, [VP, I64, I64, I32, I32, I32, P(Request), I32,
                                     P(PixelError), VP]),
        "hsad_read_cube": (I32, [VP, I64, P(CubeHeader), VP, I32, VP]),
        "hsad_reduce_raw": (I32, [VP, I64, P(CubeHeader), I32, I32, VP, I32, VP]),
        "hsad_pipeline_raw": (I32, [VP, I64, P(CubeHeader), I32, I32, P(Request), I32,
                                    P(PixelError), VP]),
        "hsad_pipeline_sharded": (I32, [VP, I64, I64, I32, I32, I32, P(Request), I32, I32,
                                        P(PixelError)]),
        "hsad_roc": (I32, [VP, I32, VP, I64, P(RocSummary), VP, VP, I64, VP]),
        "hsad_top_k": (I32, [VP, I32, I64, I64, VP, P(D), VP]),
        "hsad_adaptive_threshold": (I32, [VP, I32, I64, D, P(D), VP, VP]),
        "hsad_render_pgm": (I32, [VP, I32, I64, VP, VP]),
        "hsad_strip_plan": (I32, [I64, I64, I32, I32, P(I64), P(I64), P(I64)]),
        "hsad_gather_maps": (I32, [VP, I32, I32, I32, I64, I64, P(MapDesc), I32, VP]),
        "hsad_nccl_available": (I32, []),
        "hsad_nccl_unique_id": (I32, [VP]),
        "hsad_nccl_comm_init_rank": (I32, [P(VP), I32, VP, I32]),
        "hsad_nccl_comm_init_all": (I32, [P(VP), I32]),
        "hsad_nccl_comm_destroy": (I32, [VP]),
        "hsad_last_reduce_detect_fused": (I32, []),
        "hsad_dwest_pairs": (I32, [VP, VP, I64, D, VP, VP, VP, VP]),
        "hsad_dual_window_samples": (I32, [VP, I32, I64, I64, I32, I64, I64, P(Window), VP, VP, VP]),
        "hsad_encode_score_map": (I32, [VP, I32, I64, VP, VP]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


_lib: C.CDLL | None = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        _lib = load()
    return _lib
