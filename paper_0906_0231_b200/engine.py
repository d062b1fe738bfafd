"""Python mirror of the reference's engine interface, running on the B200 C ABI.

Same names, argument meaning and error behaviour as the reference C++ API
(paths relative to /root/reference/proj):

=====================  ===================================================
``Dataset``            include/knn/dataset.hpp:12-34, src/dataset.cpp:11-30
``CumulativeDistance`` include/knn/distance.hpp:26-33 (+ ``hellinger()``,
                       ``squared_euclidean()`` src/distance.cpp:12-34,
                       ``distance_by_name`` :152-165)
``GridPlan``,          include/knn/schedule.hpp:13-26,
``make_plan``,         src/schedule.cpp:10-38
``auto_gsize``
``EngineOptions``,     include/knn/engine.hpp:14-31
``EngineResult``
``solve_knn``          include/knn/engine.hpp:37-38, src/engine.cpp:13-68
``ConfigError`` ...    include/knn/errors.hpp:8-31
=====================  ===================================================

``solve_knn`` validates options and plans exactly like engine.cpp:15-23, then
hands the whole computation to ``knn_b200_solve_multi`` (one host thread per
GPU, ``n_lanes`` -> GPUs).  Results come back as flat arrays
(``EngineResult.index`` / ``.distance``, n x min(k, n-1)); ``.lists`` builds
the reference's ``NeighborList`` objects lazily for small n.
"""
from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass, field
from typing import NamedTuple

import numpy as np

from . import _lib

# --------------------------------------------------------------------------
# errors.hpp:8-31


class ConfigError(RuntimeError):
    """Invalid parameter or parameter combination (CLI exit code 2)."""


class ValidationError(RuntimeError):
    """Rejected input data, e.g. non-finite or out-of-domain (exit code 3)."""


class IoError(RuntimeError):
    """Unreadable or malformed file (io.cpp; CLI exit code 3)."""


class ConsistencyError(RuntimeError):
    """Broken internal invariant; always a bug (exit code 4)."""


class EngineError(RuntimeError):
    """CUDA / internal failure inside the B200 engine (exit code 4)."""


def raise_for_status(rc: int) -> None:
    if rc == _lib.OK:
        return
    msg = _lib.last_error()
    if rc == _lib.ERR_CONFIG:
        raise ConfigError(msg)
    if rc == _lib.ERR_VALIDATION:
        raise ValidationError(msg)
    if rc == _lib.ERR_IO:
        raise IoError(msg)
    raise EngineError(msg)


# --------------------------------------------------------------------------
# dataset.hpp / dataset.cpp


class Dataset:
    """n vectors of dimension d, dense row-major float32, immutable.

    Rejects n < 2, d < 1, a wrongly sized buffer and non-finite coordinates
    with ValidationError, like dataset.cpp:13-29.
    """

    def __init__(self, n: int, d: int, values):
        if n < 2:
            raise ValidationError(f"dataset needs at least 2 vectors, got {n}")
        if d < 1:
            raise ValidationError("dataset dimension must be at least 1")
        arr = np.ascontiguousarray(np.asarray(values, dtype=np.float32)).reshape(-1)
        if arr.size != n * d:
            raise ValidationError(f"dataset value buffer holds {arr.size} floats, expected {n * d}")
        finite = np.isfinite(arr)
        if not finite.all():
            i = int(np.argmin(finite))
            raise ValidationError(f"non-finite coordinate {i % d} in vector {i // d}")
        arr = arr.reshape(n, d)
        arr.setflags(write=False)
        self._values = arr

    @classmethod
    def from_array(cls, x) -> "Dataset":
        x = np.asarray(x, dtype=np.float32)
        return cls(x.shape[0], x.shape[1], x)

    def size(self) -> int:
        return self._values.shape[0]

    def dim(self) -> int:
        return self._values.shape[1]

    def row(self, i: int) -> np.ndarray:
        return self._values[i]

    def values(self) -> np.ndarray:
        return self._values


# --------------------------------------------------------------------------
# distance.hpp:19-33, distance.cpp:12-34, 152-165


class MetricKind:
    hellinger = 0
    sqeuclidean = 1
    custom = 2


@dataclass(frozen=True)
class CumulativeDistance:
    """A registered distance.  Only the GPU-known folds exist here: the
    reference's custom functors are host function pointers, which cannot run
    on the device; ``cosine`` is the custom fold of SURVEY §8(d)."""

    name: str
    kind: int
    metric_id: int
    nonnegative_domain: bool = False


def hellinger() -> CumulativeDistance:
    return CumulativeDistance("hellinger", MetricKind.hellinger, _lib.METRIC_HELLINGER, True)


def squared_euclidean() -> CumulativeDistance:
    return CumulativeDistance("sqeuclidean", MetricKind.sqeuclidean, _lib.METRIC_SQEUCLIDEAN)


def cosine() -> CumulativeDistance:
    """step acc + u*v, finalize 1 - acc (callers L2-normalise rows)."""
    return CumulativeDistance("cosine", MetricKind.custom, _lib.METRIC_COSINE)


def euclidean() -> CumulativeDistance:
    """The BASELINE configs' "Euclidean": sqeuclidean fold, sqrtf at output
    (SURVEY §8(d) metric mapping)."""
    return CumulativeDistance("euclidean", MetricKind.custom, _lib.METRIC_EUCLIDEAN)


def manhattan() -> CumulativeDistance:
    """The reference test suite's custom functor: step acc + |u - v|
    (test_distance.cpp:134-145).  EXACT policy."""
    return CumulativeDistance("manhattan", MetricKind.custom, _lib.METRIC_MANHATTAN)


def root_of_squares() -> CumulativeDistance:
    """The reference test suite's custom functor: the sqeuclidean step with
    finalize sqrt, ranked by the finalized distance (test_distance.cpp:166-178).
    EXACT policy."""
    return CumulativeDistance("root_of_squares", MetricKind.custom, _lib.METRIC_ROOT_SQUARES)


_REGISTRY = {"hellinger": hellinger, "sqeuclidean": squared_euclidean, "cosine": cosine, "euclidean": euclidean,
             "manhattan": manhattan, "root_of_squares": root_of_squares}


def distance_by_name(name: str) -> CumulativeDistance:
    try:
        return _REGISTRY[name]()
    except KeyError:
        raise ConfigError(f"unknown distance '{name}'; registered: {', '.join(sorted(_REGISTRY))}") from None


def distance_names() -> list[str]:
    return sorted(_REGISTRY)


# --------------------------------------------------------------------------
# schedule.hpp:13-26, schedule.cpp:10-38

kDefaultBsize = 64
kDefaultC1 = 32
kDefaultC2 = 32
kDefaultBufSize = 16


@dataclass(frozen=True)
class GridPlan:
    n: int = 0
    gsize: int = 0
    bsize: int = 0
    c1: int = 0
    c2: int = 0
    n_lanes: int = 0
    n_grids: int = 0


def make_plan(n: int, gsize: int, bsize: int, c1: int, c2: int, n_lanes: int) -> GridPlan:
    if n < 2:
        raise ConfigError(f"n must be at least 2, got {n}")
    if gsize < 1:
        raise ConfigError("gsize must be at least 1")
    if bsize < 1:
        raise ConfigError("bsize must be at least 1")
    if bsize > gsize:
        raise ConfigError(f"bsize ({bsize}) must not exceed gsize ({gsize})")
    if c1 < 1:
        raise ConfigError("c1 must be at least 1")
    if c2 < 1:
        raise ConfigError("c2 must be at least 1")
    if n_lanes < 1:
        raise ConfigError("n_lanes must be at least 1")
    return GridPlan(n, gsize, bsize, c1, c2, n_lanes, (n - 1) // gsize + 1)


def auto_gsize(n: int, bsize: int) -> int:
    rounded = (n + bsize - 1) // bsize * bsize
    return max(min(rounded, 4096), bsize)


# --------------------------------------------------------------------------
# heap.hpp:16-27, 62-67 ; select.hpp:49-60 ; engine.hpp:14-31


class Neighbor(NamedTuple):
    distance: float
    index: int


class NeighborList(NamedTuple):
    query: int
    neighbors: list


@dataclass
class SelectStats:
    offered: int = 0
    buffered: int = 0
    flush_pushes: int = 0


@dataclass
class EngineOptions:
    k: int = 100
    n_lanes: int = 1
    gsize: int = 0
    bsize: int = kDefaultBsize
    c1: int = kDefaultC1
    c2: int = kDefaultC2
    buf_size: int = kDefaultBufSize
    workers: int = 1


@dataclass
class EngineResult:
    index: np.ndarray            # n x min(k, n-1) uint32
    distance: np.ndarray         # n x min(k, n-1) float32
    plan: GridPlan
    pair_evaluations: int
    select_stats: SelectStats
    seconds: float
    gpu_stats: dict = field(default_factory=dict)

    @property
    def lists(self) -> list[NeighborList]:
        return [NeighborList(i, [Neighbor(float(dd), int(j)) for dd, j in zip(self.distance[i], self.index[i])])
                for i in range(self.index.shape[0])]


def arith_from_env() -> int:
    v = os.environ.get("KNN_B200_ARITH", "auto") or "auto"
    if v not in _lib.ARITH_NAMES:
        raise ConfigError(f"KNN_B200_ARITH must be auto, exact or tensor, got '{v}'")
    return _lib.ARITH_NAMES[v]


def solve_knn(ds: Dataset, f: CumulativeDistance, opt: EngineOptions, arith: int | str | None = None) -> EngineResult:
    """Exact all-pairs k-NN of ``ds`` under ``f`` on the GPU(s).

    Option checks, plan and validation order follow engine.cpp:15-23; the
    result is bit-identical to the reference's brute_force_knn.
    """
    if opt.k < 1:
        raise ConfigError("k must be at least 1")
    if opt.buf_size < 1:
        raise ConfigError("buf_size must be at least 1")
    if opt.workers < 1:
        raise ConfigError("workers must be at least 1")
    gsize = opt.gsize if opt.gsize != 0 else auto_gsize(ds.size(), opt.bsize)
    plan = make_plan(ds.size(), gsize, opt.bsize, opt.c1, opt.c2, opt.n_lanes)
    if f.nonnegative_domain:  # validate_dataset (distance.cpp:36-59), before any compute
        v = ds.values()
        bad = ~(v >= 0)
        if bad.any():
            i = int(np.argmax(bad.reshape(-1)))
            d = ds.dim()
            raise ValidationError(f"coordinate {i % d} of vector {i // d} (value {v.reshape(-1)[i]:.6f}) "
                                  f"is outside the domain of {f.name}")
    if arith is None:
        arith = arith_from_env()
    elif isinstance(arith, str):
        arith = _lib.ARITH_NAMES[arith]
    lib = _lib.load()
    n, d = ds.size(), ds.dim()
    klist = min(opt.k, n - 1)
    index = np.empty((n, klist), dtype=np.uint32)
    distance = np.empty((n, klist), dtype=np.float32)
    st = _lib.Stats()
    x = ds.values()
    rc = lib.knn_b200_solve_multi(x.ctypes.data, n, d, opt.k, f.metric_id, arith, plan.n_lanes,
                                  index.ctypes.data, distance.ctypes.data, ctypes.byref(st))
    raise_for_status(rc)
    pairs = int(st.pair_evaluations)
    return EngineResult(index, distance, plan, pairs, SelectStats(offered=2 * pairs), float(st.seconds),
                        st.as_dict())


# --------------------------------------------------------------------------
# Device-resident API (one context per device), used by the multi-GPU
# driver and bench.py.


class Context:
    """A knn_b200_ctx bound to one CUDA device."""

    def __init__(self, device: int = 0):
        lib = _lib.load()
        h = ctypes.c_void_p()
        raise_for_status(lib.knn_b200_create(device, ctypes.byref(h)))
        self._h = h
        self.device = device

    def close(self):
        if self._h:
            _lib.load().knn_b200_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def solve(self, x: np.ndarray, k: int, metric: CumulativeDistance, arith: int = _lib.ARITH_AUTO,
              out: tuple[np.ndarray, np.ndarray] | None = None):
        """Host arrays in, host arrays out (knn_b200_solve).  ``out``: optional
        caller-owned (index uint32, distance float32) arrays of shape
        n x min(k, n-1), e.g. views of pinned memory."""
        x = np.ascontiguousarray(x, dtype=np.float32)
        n, d = x.shape
        klist = min(k, n - 1) if n >= 2 else 0
        if out is not None:
            index, distance = out
            if (index.shape != (n, max(klist, 0)) or distance.shape != index.shape or index.dtype != np.uint32
                    or distance.dtype != np.float32 or not index.flags.c_contiguous
                    or not distance.flags.c_contiguous):
                raise ConfigError("out must be C-contiguous (uint32, float32) arrays of shape n x min(k, n-1)")
        else:
            index = np.empty((n, max(klist, 0)), dtype=np.uint32)
            distance = np.empty((n, max(klist, 0)), dtype=np.float32)
        st = _lib.Stats()
        rc = _lib.load().knn_b200_solve(self._h, x.ctypes.data, n, d, k, metric.metric_id, arith,
                                        index.ctypes.data, distance.ctypes.data, ctypes.byref(st))
        raise_for_status(rc)
        return index, distance, st.as_dict()

    def solve_f64(self, x: np.ndarray, k: int, metric: CumulativeDistance):
        """The reference's KNN_DOUBLE_ACCUM build (types.hpp:9-13): float
        coordinates, double accumulation and distances (knn_b200_solve_f64,
        EXACT policy).  Returns float64 distances."""
        x = np.ascontiguousarray(x, dtype=np.float32)
        n, d = x.shape
        klist = min(k, n - 1) if n >= 2 else 0
        index = np.empty((n, max(klist, 0)), dtype=np.uint32)
        distance = np.empty((n, max(klist, 0)), dtype=np.float64)
        st = _lib.Stats()
        rc = _lib.load().knn_b200_solve_f64(self._h, x.ctypes.data, n, d, k, metric.metric_id,
                                            index.ctypes.data, distance.ctypes.data, ctypes.byref(st))
        raise_for_status(rc)
        return index, distance, st.as_dict()

    def solve_rows_device(self, x_ptr: int, n: int, d: int, k: int, metric: CumulativeDistance,
                          row_begin: int, row_end: int, out_index_ptr: int, out_dist_ptr: int,
                          stream_ptr: int = 0, arith: int = _lib.ARITH_AUTO, want_stats: bool = False):
        st = _lib.Stats() if want_stats else None
        rc = _lib.load().knn_b200_solve_rows_device(
            self._h, x_ptr, n, d, k, metric.metric_id, arith, row_begin, row_end, out_index_ptr,
            out_dist_ptr, stream_ptr, ctypes.byref(st) if st is not None else None)
        raise_for_status(rc)
        return st.as_dict() if st is not None else None


def comm_unique_id() -> bytes:
    """128 opaque bytes (an ncclUniqueId) for Context.comm_init."""
    buf = ctypes.create_string_buffer(128)
    raise_for_status(_lib.load().knn_b200_comm_unique_id(buf))
    return buf.raw


def comm_init(ctx: Context, uid: bytes, rank: int, world: int) -> None:
    """Bind an NCCL communicator of `world` ranks to ctx (collective)."""
    buf = ctypes.create_string_buffer(bytes(uid), 128)
    raise_for_status(_lib.load().knn_b200_comm_init(ctx._h, buf, rank, world))


def comm_broadcast_torch(ctx: Context, t, root: int = 0) -> None:
    """In-place NCCL broadcast of a CUDA tensor over ctx's communicator."""
    import torch
    stream = torch.cuda.current_stream(t.device).cuda_stream
    raise_for_status(_lib.load().knn_b200_comm_broadcast(ctx._h, t.data_ptr(), t.numel() * t.element_size(), root,
                                                         stream))


def shard_rows(n: int, rank: int, world: int) -> tuple[int, int]:
    """Rows of rank `rank` in a sharded solve: [R r, min(R (r+1), n)), R = ceil(n / world)."""
    rr = -(-n // world)
    b = min(rr * rank, n)
    return b, min(b + rr, n)


def solve_sharded_torch(ctx: Context, x, k: int, metric: CumulativeDistance, arith: int = _lib.ARITH_AUTO,
                        rank: int = 0, world: int = 1, want_stats: bool = False):
    """This rank's contiguous shard of the whole problem's lists
    (knn_b200_solve_sharded_device, collective over ctx's communicator).
    Returns (index int32, distance float32, stats)."""
    import torch
    if not (x.is_cuda and x.dtype == torch.float32 and x.is_contiguous() and x.dim() == 2):
        raise ConfigError("x must be a contiguous 2-D float32 CUDA tensor")
    n, d = x.shape
    klist = min(k, n - 1)
    b, e = shard_rows(n, rank, world)
    idx = torch.empty((max(e - b, 1), klist), dtype=torch.int32, device=x.device)
    dist = torch.empty((max(e - b, 1), klist), dtype=torch.float32, device=x.device)
    st = _lib.Stats() if want_stats else None
    stream = torch.cuda.current_stream(x.device).cuda_stream
    raise_for_status(_lib.load().knn_b200_solve_sharded_device(
        ctx._h, x.data_ptr(), n, d, k, metric.metric_id, arith, idx.data_ptr(), dist.data_ptr(), stream,
        ctypes.byref(st) if st is not None else None))
    return idx[: e - b], dist[: e - b], (st.as_dict() if st is not None else None)


def solve_sharded_loopback_torch(ctx: Context, x, k: int, metric: CumulativeDistance, world: int):
    """Test hook: all `world` rank programs of the sharded triangle on x's
    device, one after another (knn_b200_debug_solve_sharded_loopback).
    Returns (index, distance, stats, rank_ms (world x 4), sent bytes (world))."""
    import numpy as np
    import torch
    n, d = x.shape
    klist = min(k, n - 1)
    idx = torch.empty((n, klist), dtype=torch.int32, device=x.device)
    dist = torch.empty((n, klist), dtype=torch.float32, device=x.device)
    st = _lib.Stats()
    rank_ms = np.zeros((world, 4), dtype=np.float32)
    xbytes = np.zeros(world, dtype=np.uint64)
    stream = torch.cuda.current_stream(x.device).cuda_stream
    raise_for_status(_lib.load().knn_b200_debug_solve_sharded_loopback(
        ctx._h, x.data_ptr(), n, d, k, metric.metric_id, world, idx.data_ptr(), dist.data_ptr(), stream,
        ctypes.byref(st), rank_ms.ctypes.data, xbytes.ctypes.data))
    return idx, dist, st.as_dict(), rank_ms, xbytes


def solve_rows_torch(ctx: Context, x, k: int, metric: CumulativeDistance, row_begin: int, row_end: int,
                     arith: int = _lib.ARITH_AUTO, out=None, want_stats: bool = False):
    """Rows [row_begin, row_end) of a CUDA float32 tensor ``x`` (n x d) against
    all n rows, on torch's current stream.  Returns (index, distance) tensors
    (int32 view of the uint32 indices, float32)."""
    import torch

    if not (x.is_cuda and x.dtype == torch.float32 and x.is_contiguous() and x.dim() == 2):
        raise ConfigError("x must be a contiguous 2-D float32 CUDA tensor")
    n, d = x.shape
    klist = min(k, n - 1)
    rows = row_end - row_begin
    if out is None:
        idx = torch.empty((rows, klist), dtype=torch.int32, device=x.device)
        dist = torch.empty((rows, klist), dtype=torch.float32, device=x.device)
    else:
        idx, dist = out
        for t, dt in ((idx, torch.int32), (dist, torch.float32)):
            if (t.shape != (rows, klist) or t.dtype != dt or not t.is_contiguous() or t.device != x.device):
                raise ConfigError(f"out must be contiguous (int32, float32) tensors of shape ({rows}, {klist}) "
                                  f"on {x.device}")
    if not (0 <= row_begin <= row_end <= n):
        raise ConfigError(f"row range [{row_begin}, {row_end}) outside [0, {n})")
    stream = torch.cuda.current_stream(x.device).cuda_stream
    st = ctx.solve_rows_device(x.data_ptr(), n, d, k, metric, row_begin, row_end, idx.data_ptr(),
                               dist.data_ptr(), stream, arith, want_stats)
    return idx, dist, st


def knnv_header(path) -> tuple[int, int]:
    """(n, d) of a KNNV dataset file, checked like load_dataset (io.cpp:64-88)."""
    n, d = ctypes.c_uint32(0), ctypes.c_uint32(0)
    raise_for_status(_lib.load().knn_b200_knnv_header(os.fsencode(path), ctypes.byref(n), ctypes.byref(d)))
    return n.value, d.value


def load_knnv_torch(ctx: Context, path, device=None):
    """load_dataset (io.cpp:64-97) straight into a CUDA tensor: the payload is
    read in parallel through pinned staging and checked on the device."""
    import torch

    n, d = knnv_header(path)
    x = torch.empty((n, d), dtype=torch.float32, device=device or f"cuda:{ctx.device}")
    on, od = ctypes.c_uint32(0), ctypes.c_uint32(0)
    stream = torch.cuda.current_stream(x.device).cuda_stream
    raise_for_status(_lib.load().knn_b200_load_knnv_device(ctx._h, os.fsencode(path), x.data_ptr(), n * d,
                                                           ctypes.byref(on), ctypes.byref(od), stream))
    return x


def generate_torch(ctx: Context, n: int, d: int, seed: int, device=None):
    """generate_dataset(n, d, seed) (src/io.cpp:57-62) produced on the device."""
    import torch

    x = torch.empty((n, d), dtype=torch.float32, device=device or f"cuda:{ctx.device}")
    stream = torch.cuda.current_stream(x.device).cuda_stream
    raise_for_status(_lib.load().knn_b200_generate_device(ctx._h, x.data_ptr(), n * d, seed, stream))
    return x


def device_count() -> int:
    c = ctypes.c_int(0)
    raise_for_status(_lib.load().knn_b200_device_count(ctypes.byref(c)))
    return c.value
