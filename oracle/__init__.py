"""Parity checkers for the B200 k-NN engine -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference`` arm) may import this package.
The product package ``paper_0906_0231_b200`` never imports it and has no CPU
fallback.

Two checkers live here:

* :class:`CRestatement` -- ``libknn_oracle.so``, the plain-C restatement of the
  reference algorithm (``knn_oracle.c``; each function cites the reference
  file:line it follows).
* :class:`Reference` -- ``_ref/libtknn_ref_capi.so``, the UNMODIFIED reference
  library compiled from ``/root/reference/proj/src`` (``Makefile``), reached
  through the ``ref_capi.cpp`` shim.  Absent when the reference was not
  available at build time; callers must skip, not substitute.
"""
from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
C_ORACLE_PATH = HERE / "libknn_oracle.so"
REF_CAPI_PATH = HERE / "_ref" / "libtknn_ref_capi.so"

METRICS = {"hellinger": 0, "sqeuclidean": 1, "cosine": 2, "manhattan": 3, "root_of_squares": 4}

_u32p = ctypes.POINTER(ctypes.c_uint32)
_f32p = ctypes.POINTER(ctypes.c_float)
_u64p = ctypes.POINTER(ctypes.c_uint64)
_f64p = ctypes.POINTER(ctypes.c_double)
REF_F64_CAPI_PATH = HERE / "_ref" / "f64" / "libtknn_ref_capi.so"


def _ptr(a: np.ndarray, t):
    return a.ctypes.data_as(t)


def metric_id(metric) -> int:
    return metric if isinstance(metric, int) else METRICS[metric]


class CRestatement:
    """ctypes view of ``libknn_oracle.so``."""

    def __init__(self, path: Path = C_ORACLE_PATH):
        if not path.exists():
            raise FileNotFoundError(f"{path} not built; run `make -C oracle`")
        lib = ctypes.CDLL(str(path))
        lib.ko_splitmix64_next.argtypes = [_u64p]
        lib.ko_splitmix64_next.restype = ctypes.c_uint64
        lib.ko_next_unit_float.argtypes = [_u64p]
        lib.ko_next_unit_float.restype = ctypes.c_float
        lib.ko_generate.argtypes = [ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint64, _f32p]
        lib.ko_generate_at.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, _f32p]
        lib.ko_fold.argtypes = [ctypes.c_int, _f32p, _f32p, ctypes.c_uint32]
        lib.ko_fold.restype = ctypes.c_float
        lib.ko_heap_stream.argtypes = [ctypes.c_uint32, _f32p, _u32p, ctypes.c_uint32, _f32p, _u32p]
        lib.ko_heap_stream.restype = ctypes.c_uint32
        lib.ko_brute_force.argtypes = [_f32p, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32,
                                       ctypes.c_int, _u32p, _f32p, _u64p]
        lib.ko_rows_topk.argtypes = [_f32p, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32,
                                     ctypes.c_int, _u32p, ctypes.c_uint32, ctypes.c_uint32,
                                     _u32p, _f32p]
        lib.ko_fold_f64.argtypes = [ctypes.c_int, _f32p, _f32p, ctypes.c_uint32]
        lib.ko_fold_f64.restype = ctypes.c_double
        lib.ko_brute_force_f64.argtypes = [_f32p, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32,
                                           ctypes.c_int, _u32p, _f64p]
        lib.ko_rows_topk_f64.argtypes = [_f32p, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32,
                                         ctypes.c_int, _u32p, ctypes.c_uint32, _u32p, _f64p]
        self.lib = lib

    def rows_topk_f64(self, x: np.ndarray, k: int, metric, rows):
        """The double build's lists for the query rows ``rows`` (single thread)."""
        x = np.ascontiguousarray(x, dtype=np.float32)
        rows = np.ascontiguousarray(rows, dtype=np.uint32)
        n, d = x.shape
        cap = min(k, n - 1)
        idx = np.empty((rows.size, cap), dtype=np.uint32)
        dist = np.empty((rows.size, cap), dtype=np.float64)
        rc = self.lib.ko_rows_topk_f64(_ptr(x, _f32p), n, d, k, metric_id(metric), _ptr(rows, _u32p), rows.size,
                                       _ptr(idx, _u32p), _ptr(dist, _f64p))
        if rc != 0:
            raise ValueError(f"ko_rows_topk_f64 failed with code {rc}")
        return idx, dist

    def brute_force_f64(self, x: np.ndarray, k: int, metric):
        """brute_force_knn of the KNN_DOUBLE_ACCUM build: float64 distances."""
        x = np.ascontiguousarray(x, dtype=np.float32)
        n, d = x.shape
        cap = min(k, n - 1)
        idx = np.empty((n, cap), dtype=np.uint32)
        dist = np.empty((n, cap), dtype=np.float64)
        rc = self.lib.ko_brute_force_f64(_ptr(x, _f32p), n, d, k, metric_id(metric),
                                         _ptr(idx, _u32p), _ptr(dist, _f64p))
        if rc != 0:
            raise ValueError(f"ko_brute_force_f64 failed with code {rc}")
        return idx, dist

    def splitmix64(self, seed: int, count: int) -> list[int]:
        s = ctypes.c_uint64(seed)
        return [self.lib.ko_splitmix64_next(ctypes.byref(s)) for _ in range(count)]

    def unit_floats(self, seed: int, count: int) -> list[float]:
        s = ctypes.c_uint64(seed)
        return [self.lib.ko_next_unit_float(ctypes.byref(s)) for _ in range(count)]

    def generate(self, n: int, d: int, seed: int) -> np.ndarray:
        out = np.empty((n, d), dtype=np.float32)
        self.lib.ko_generate(n, d, seed, _ptr(out, _f32p))
        return out

    def generate_at(self, seed: int, first: int, count: int) -> np.ndarray:
        """Elements [first, first + count) of generate_dataset's row-major
        stream (Weyl jump, knn_oracle.c ko_generate_at)."""
        out = np.empty(count, dtype=np.float32)
        self.lib.ko_generate_at(seed, first, count, _ptr(out, _f32p))
        return out

    def fold(self, metric, u: np.ndarray, v: np.ndarray) -> np.float32:
        u = np.ascontiguousarray(u, dtype=np.float32)
        v = np.ascontiguousarray(v, dtype=np.float32)
        return np.float32(self.lib.ko_fold(metric_id(metric), _ptr(u, _f32p), _ptr(v, _f32p), u.size))

    def heap_stream(self, capacity: int, dist: np.ndarray, index: np.ndarray):
        dist = np.ascontiguousarray(dist, dtype=np.float32)
        index = np.ascontiguousarray(index, dtype=np.uint32)
        od = np.empty(capacity, dtype=np.float32)
        oi = np.empty(capacity, dtype=np.uint32)
        m = self.lib.ko_heap_stream(capacity, _ptr(dist, _f32p), _ptr(index, _u32p), dist.size,
                                    _ptr(od, _f32p), _ptr(oi, _u32p))
        return oi[:m], od[:m]

    def brute_force(self, x: np.ndarray, k: int, metric):
        x = np.ascontiguousarray(x, dtype=np.float32)
        n, d = x.shape
        cap = min(k, n - 1)
        idx = np.empty((n, cap), dtype=np.uint32)
        dist = np.empty((n, cap), dtype=np.float32)
        pairs = ctypes.c_uint64(0)
        rc = self.lib.ko_brute_force(_ptr(x, _f32p), n, d, k, metric_id(metric),
                                     _ptr(idx, _u32p), _ptr(dist, _f32p), ctypes.byref(pairs))
        if rc != 0:
            raise ValueError(f"ko_brute_force failed with code {rc}")
        return idx, dist, pairs.value

    def rows_topk(self, x: np.ndarray, k: int, metric, rows, threads: int | None = None):
        x = np.ascontiguousarray(x, dtype=np.float32)
        rows = np.ascontiguousarray(rows, dtype=np.uint32)
        n, d = x.shape
        cap = min(k, n - 1)
        idx = np.empty((rows.size, cap), dtype=np.uint32)
        dist = np.empty((rows.size, cap), dtype=np.float32)
        threads = threads or os.cpu_count() or 1
        rc = self.lib.ko_rows_topk(_ptr(x, _f32p), n, d, k, metric_id(metric), _ptr(rows, _u32p),
                                   rows.size, threads, _ptr(idx, _u32p), _ptr(dist, _f32p))
        if rc != 0:
            raise ValueError(f"ko_rows_topk failed with code {rc}")
        return idx, dist


class Reference:
    """ctypes view of the compiled, unmodified reference library."""

    def __init__(self, path: Path = REF_CAPI_PATH):
        if not path.exists():
            raise FileNotFoundError(f"{path} not built (needs /root/reference at build time)")
        lib = ctypes.CDLL(str(path))
        lib.ref_last_error.restype = ctypes.c_char_p
        lib.ref_generate.argtypes = [ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint64, _f32p]
        lib.ref_brute_force.argtypes = [_f32p, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32,
                                        ctypes.c_int, _u32p, _f32p, _u64p,
                                        ctypes.POINTER(ctypes.c_double)]
        lib.ref_solve_knn.argtypes = [_f32p, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32,
                                      ctypes.c_int, ctypes.c_uint32, ctypes.c_uint32, _u32p, _f32p,
                                      _u64p, ctypes.POINTER(ctypes.c_double)]
        lib.ref_rows_topk.argtypes = [_f32p, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32,
                                      ctypes.c_int, _u32p, ctypes.c_uint32, ctypes.c_uint32,
                                      _u32p, _f32p]
        self.lib = lib

    def _check(self, rc: int, what: str):
        if rc != 0:
            raise RuntimeError(f"{what} failed ({rc}): {self.lib.ref_last_error().decode()}")

    def generate(self, n: int, d: int, seed: int) -> np.ndarray:
        out = np.empty((n, d), dtype=np.float32)
        self._check(self.lib.ref_generate(n, d, seed, _ptr(out, _f32p)), "ref_generate")
        return out

    def brute_force(self, x: np.ndarray, k: int, metric):
        x = np.ascontiguousarray(x, dtype=np.float32)
        n, d = x.shape
        cap = min(k, n - 1)
        idx = np.empty((n, cap), dtype=np.uint32)
        dist = np.empty((n, cap), dtype=np.float32)
        pairs = ctypes.c_uint64(0)
        secs = ctypes.c_double(0)
        self._check(self.lib.ref_brute_force(_ptr(x, _f32p), n, d, k, metric_id(metric),
                                             _ptr(idx, _u32p), _ptr(dist, _f32p),
                                             ctypes.byref(pairs), ctypes.byref(secs)),
                    "ref_brute_force")
        return idx, dist, pairs.value, secs.value

    def solve_knn(self, x: np.ndarray, k: int, metric, n_lanes: int = 1, gsize: int = 0,
                  want_lists: bool = True):
        x = np.ascontiguousarray(x, dtype=np.float32)
        n, d = x.shape
        cap = min(k, n - 1)
        idx = np.empty((n, cap), dtype=np.uint32) if want_lists else None
        dist = np.empty((n, cap), dtype=np.float32) if want_lists else None
        pairs = ctypes.c_uint64(0)
        secs = ctypes.c_double(0)
        self._check(self.lib.ref_solve_knn(_ptr(x, _f32p), n, d, k, metric_id(metric), n_lanes,
                                           gsize, _ptr(idx, _u32p) if want_lists else None,
                                           _ptr(dist, _f32p) if want_lists else None,
                                           ctypes.byref(pairs), ctypes.byref(secs)),
                    "ref_solve_knn")
        return idx, dist, pairs.value, secs.value

    def rows_topk(self, x: np.ndarray, k: int, metric, rows, threads: int | None = None):
        x = np.ascontiguousarray(x, dtype=np.float32)
        rows = np.ascontiguousarray(rows, dtype=np.uint32)
        n, d = x.shape
        cap = min(k, n - 1)
        idx = np.empty((rows.size, cap), dtype=np.uint32)
        dist = np.empty((rows.size, cap), dtype=np.float32)
        self._check(self.lib.ref_rows_topk(_ptr(x, _f32p), n, d, k, metric_id(metric),
                                           _ptr(rows, _u32p), rows.size,
                                           threads or os.cpu_count() or 1, _ptr(idx, _u32p),
                                           _ptr(dist, _f32p)),
                    "ref_rows_topk")
        return idx, dist


def c_oracle() -> CRestatement:
    return CRestatement()


def reference() -> Reference | None:
    """The compiled reference, or None when it was not built here."""
    return Reference() if REF_CAPI_PATH.exists() else None


def normalize_rows(x: np.ndarray) -> np.ndarray:
    """SURVEY §8(d) cosine inputs: L2-normalise rows in double, store f32."""
    x64 = x.astype(np.float64)
    nrm = np.sqrt((x64 * x64).sum(axis=1, keepdims=True))
    nrm[nrm == 0] = 1.0
    return (x64 / nrm).astype(np.float32)


class ReferenceF64:
    """The compiled reference in its KNN_DOUBLE_ACCUM build
    (``_ref/f64/libtknn_ref_capi.so``): brute_force_knn with double distances."""

    def __init__(self, path: Path = REF_F64_CAPI_PATH):
        if not path.exists():
            raise FileNotFoundError(f"{path} not built (needs /root/reference at build time)")
        lib = ctypes.CDLL(str(path))
        lib.ref_last_error.restype = ctypes.c_char_p
        lib.ref_brute_force_f64.argtypes = [_f32p, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32,
                                            ctypes.c_int, _u32p, _f64p]
        self.lib = lib

    def brute_force(self, x: np.ndarray, k: int, metric):
        x = np.ascontiguousarray(x, dtype=np.float32)
        n, d = x.shape
        cap = min(k, n - 1)
        idx = np.empty((n, cap), dtype=np.uint32)
        dist = np.empty((n, cap), dtype=np.float64)
        rc = self.lib.ref_brute_force_f64(_ptr(x, _f32p), n, d, k, metric_id(metric),
                                          _ptr(idx, _u32p), _ptr(dist, _f64p))
        if rc != 0:
            raise ValueError(self.lib.ref_last_error().decode())
        return idx, dist
