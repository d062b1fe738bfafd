"""ctypes binding of the C ABI in include/knn_b200.h.

The shared library is built in-tree (``make`` at the repo root or
``__graft_entry__.build()``) into ``paper_0906_0231_b200/lib/libknn_b200.so``.
Loading fails loudly when it is missing: there is no CPU fallback.
"""
from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

# KNN_B200_LIB: an alternative in-tree build of the same library (tuning
# experiments); the default is the library `make` builds.
LIB_PATH = Path(os.environ.get("KNN_B200_LIB") or Path(__file__).resolve().parent / "lib" / "libknn_b200.so")

# Every exported symbol of include/knn_b200.h (checked by the CPU test suite).
EXPORTS = (
    "knn_b200_abi_version",
    "knn_b200_last_error",
    "knn_b200_device_count",
    "knn_b200_create",
    "knn_b200_destroy",
    "knn_b200_solve",
    "knn_b200_solve_f64",
    "knn_b200_solve_multi_f64",
    "knn_b200_knnv_header",
    "knn_b200_load_knnv_device",
    "knn_b200_debug_tc_dots",
    "knn_b200_tri_unit_plan",
    "knn_b200_comm_unique_id",
    "knn_b200_comm_init",
    "knn_b200_comm_broadcast",
    "knn_b200_solve_sharded_device",
    "knn_b200_debug_solve_sharded_loopback",
    "knn_b200_solve_rows_device",
    "knn_b200_solve_multi",
    "knn_b200_generate_device",
)

ABI_VERSION = 2

OK, ERR_CONFIG, ERR_VALIDATION, ERR_INTERNAL, ERR_IO = 0, 2, 3, 4, 5
METRIC_HELLINGER, METRIC_SQEUCLIDEAN, METRIC_COSINE, METRIC_EUCLIDEAN = 0, 1, 2, 3
METRIC_MANHATTAN, METRIC_ROOT_SQUARES = 4, 5
ARITH_AUTO, ARITH_EXACT, ARITH_TENSOR = 0, 1, 2
ARITH_NAMES = {"auto": ARITH_AUTO, "exact": ARITH_EXACT, "tensor": ARITH_TENSOR}


class Stats(ctypes.Structure):
    """knn_b200_stats."""

    _fields_ = [
        ("pair_evaluations", ctypes.c_uint64),
        ("distance_evals", ctypes.c_uint64),
        ("rescored", ctypes.c_uint64),
        ("fallback_rows", ctypes.c_uint32),
        ("kernel_launches", ctypes.c_uint32),
        ("arith_used", ctypes.c_int32),
        ("n_devices", ctypes.c_int32),
        ("seconds", ctypes.c_double),
        ("h2d_ms", ctypes.c_double),
        ("kernel_ms", ctypes.c_double),
        ("d2h_ms", ctypes.c_double),
        ("sweep_ms", ctypes.c_double),
        ("exact_rows", ctypes.c_uint32),
        ("reserved", ctypes.c_uint32),
    ]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


_u32p = ctypes.POINTER(ctypes.c_uint32)
_f32p = ctypes.POINTER(ctypes.c_float)

_lock = threading.Lock()
_lib = None


def load() -> ctypes.CDLL:
    """Load and type the library once; raise if it was not built."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH} is missing: the B200 CUDA library was not built "
                "(run `make` or __graft_entry__.build()); there is no CPU fallback")
        lib = ctypes.CDLL(str(LIB_PATH))
        lib.knn_b200_abi_version.restype = ctypes.c_int
        lib.knn_b200_last_error.restype = ctypes.c_char_p
        lib.knn_b200_device_count.argtypes = [ctypes.POINTER(ctypes.c_int)]
        lib.knn_b200_create.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)]
        lib.knn_b200_destroy.argtypes = [ctypes.c_void_p]
        lib.knn_b200_destroy.restype = None
        lib.knn_b200_solve.argtypes = [
            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32,
            ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(Stats)]
        lib.knn_b200_solve_f64.argtypes = [
            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32,
            ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(Stats)]
        lib.knn_b200_solve_multi_f64.argtypes = [
            ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_int,
            ctypes.c_uint32, ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(Stats)]
        lib.knn_b200_solve_rows_device.argtypes = [
            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32,
            ctypes.c_int, ctypes.c_int, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_void_p,
            ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(Stats)]
        lib.knn_b200_solve_multi.argtypes = [
            ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_int,
            ctypes.c_int, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(Stats)]
        lib.knn_b200_generate_device.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64,
                                                 ctypes.c_uint64, ctypes.c_void_p]
        lib.knn_b200_knnv_header.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_uint32),
                                             ctypes.POINTER(ctypes.c_uint32)]
        lib.knn_b200_load_knnv_device.argtypes = [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_void_p, ctypes.c_uint64,
                                                  ctypes.POINTER(ctypes.c_uint32), ctypes.POINTER(ctypes.c_uint32),
                                                  ctypes.c_void_p]
        lib.knn_b200_debug_tc_dots.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint32, ctypes.c_void_p,
                                               ctypes.c_uint32, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_void_p]
        lib.knn_b200_tri_unit_plan.argtypes = [ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_void_p,
                                               ctypes.c_void_p]
        lib.knn_b200_comm_unique_id.argtypes = [ctypes.c_void_p]
        lib.knn_b200_comm_init.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
        lib.knn_b200_comm_broadcast.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int,
                                                ctypes.c_void_p]
        lib.knn_b200_solve_sharded_device.argtypes = [
            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_int,
            ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(Stats)]
        lib.knn_b200_debug_solve_sharded_loopback.argtypes = [
            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_int,
            ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(Stats),
            ctypes.c_void_p, ctypes.c_void_p]
        if lib.knn_b200_abi_version() != ABI_VERSION:
            raise RuntimeError(f"{LIB_PATH}: ABI version {lib.knn_b200_abi_version()} != {ABI_VERSION}")
        _lib = lib
        return lib


def last_error() -> str:
    return load().knn_b200_last_error().decode(errors="replace")
