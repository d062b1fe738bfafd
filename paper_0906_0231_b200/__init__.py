"""B200-native exact all-pairs k-NN (Kato & Hosino, arXiv 0906.0231).

Hot path: Phase 1 (all-pairs distances) fused with Phase 2 (per-query top-k)
in sm_100a CUDA kernels behind the C ABI ``include/knn_b200.h``; this package
is the Python mirror of the reference's ``knn::solve_knn`` interface on top of
that ABI.  See DESIGN.md.
"""
from .engine import (  # noqa: F401
    ConfigError,
    ConsistencyError,
    Context,
    CumulativeDistance,
    Dataset,
    EngineError,
    EngineOptions,
    EngineResult,
    GridPlan,
    MetricKind,
    Neighbor,
    NeighborList,
    SelectStats,
    ValidationError,
    auto_gsize,
    cosine,
    device_count,
    distance_by_name,
    distance_names,
    euclidean,
    generate_torch,
    IoError,
    hellinger,
    knnv_header,
    load_knnv_torch,
    make_plan,
    manhattan,
    root_of_squares,
    solve_knn,
    comm_broadcast_torch,
    comm_init,
    comm_unique_id,
    shard_rows,
    solve_rows_torch,
    solve_sharded_loopback_torch,
    solve_sharded_torch,
    squared_euclidean,
)

__version__ = "0.1.0"
