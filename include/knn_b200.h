/*
 * knn_b200.h -- C ABI of the B200-native exact all-pairs k-NN engine.
 *
 * This is the drop-in boundary for the hot path of the reference tknn
 * library (paths relative to /root/reference/proj):
 *
 *   knn::solve_knn(const Dataset&, const CumulativeDistance&,
 *                  const EngineOptions&) -> EngineResult
 *     declared include/knn/engine.hpp:37-38, defined src/engine.cpp:13-68
 *
 * The C++ translation unit paper_0906_0231_b200/host/engine_b200.cpp defines
 * exactly that function on top of this ABI (it replaces src/engine.cpp at
 * link time); INTEGRATION.md shows the link line and a ctypes binding.
 *
 * Conventions
 *   - Plain C types only.  Nothing here allocates caller-visible memory; the
 *     caller owns every input and output buffer.
 *   - Every entry point returns a knn_b200_status.  Codes mirror the exit
 *     codes of the reference CLI (tools/main.cpp:225-240): 2 = ConfigError,
 *     3 = ValidationError, 4 = internal/CUDA error.  knn_b200_last_error()
 *     returns the message of the last failure on the calling thread.
 *   - Output rows are ascending by (distance, index), self excluded, of length
 *     min(k, n-1) for any k >= 1, exactly as NeighborList
 *     (include/knn/heap.hpp:62-67, src/heap.cpp:69).  Lists longer than 256
 *     run the sort-based EXACT path.  Results are bit-identical to the reference's
 *     brute_force_knn for every arithmetic policy.
 *   - There is no CPU fallback: without a usable sm_100 device every compute
 *     entry point fails with KNN_B200_ERR_INTERNAL.
 */
#ifndef KNN_B200_H
#define KNN_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KNN_B200_ABI_VERSION 2

#if defined(__GNUC__)
#define KNN_B200_API __attribute__((visibility("default")))
#else
#define KNN_B200_API
#endif

typedef enum {
    KNN_B200_OK = 0,
    KNN_B200_ERR_CONFIG = 2,     /* knn::ConfigError     (engine.cpp:15-17)  */
    KNN_B200_ERR_VALIDATION = 3, /* knn::ValidationError (distance.cpp:36-59, dataset.cpp:13-29) */
    KNN_B200_ERR_INTERNAL = 4,   /* std::runtime_error / CUDA failure        */
    KNN_B200_ERR_IO = 5          /* knn::IoError (io.cpp; CLI exit code 3)   */
} knn_b200_status;

/* Metric ids.  HELLINGER and SQEUCLIDEAN are the reference built-ins
 * (src/distance.cpp:12-34, MetricKind include/knn/distance.hpp:19); COSINE is
 * the custom fold "cosine" (step acc + u*v, finalize 1 - acc) of SURVEY §8(d).
 * Other custom functors cannot run on the GPU and are rejected by the C++
 * drop-in with ConfigError. */
typedef enum {
    KNN_B200_METRIC_HELLINGER = 0,
    KNN_B200_METRIC_SQEUCLIDEAN = 1,
    KNN_B200_METRIC_COSINE = 2,
    /* "Euclidean" of the BASELINE configs: selection on the
     * sqeuclidean fold, reported distance = IEEE sqrtf of it at output. */
    KNN_B200_METRIC_EUCLIDEAN = 3,
    /* Custom folds of the reference's registry (distance.hpp:68-77) the
     * device restates, EXACT policy: manhattan = acc + |u - v|
     * (test_distance.cpp:134-145); root-of-squares = the sqeuclidean fold
     * with finalize sqrt, ranked by the finalized distance
     * (test_distance.cpp:166-178). */
    KNN_B200_METRIC_MANHATTAN = 4,
    KNN_B200_METRIC_ROOT_SQUARES = 5
} knn_b200_metric;

/* Arithmetic policy for Phase 1 (EngineOptions has no field for it; the C++
 * drop-in reads KNN_B200_ARITH=auto|exact|tensor).
 *   EXACT  : SIMT FP32 fold, coordinate order 0..d-1, FSUB/FMUL/FADD with no
 *            contraction -- every distance bit-identical to fold_distance.
 *   TENSOR : tcgen05 FP16 filter (||a||^2+||b||^2-2ab, FP32 accumulate in
 *            TMEM) keeping a per-row candidate list with a proven error band,
 *            then an exact re-score; rows whose band is not proven are
 *            recomputed by the EXACT kernel.  Output equals EXACT bit for bit.
 *   AUTO   : TENSOR where supported, else EXACT. */
typedef enum {
    KNN_B200_ARITH_AUTO = 0,
    KNN_B200_ARITH_EXACT = 1,
    KNN_B200_ARITH_TENSOR = 2
} knn_b200_arith;

typedef struct {
    uint64_t pair_evaluations; /* semantic count: unordered pairs covered, n(n-1)/2 for a full solve
                                  (EngineResult::pair_evaluations, engine.hpp:28) */
    uint64_t distance_evals;   /* ordered (query, reference) distances the kernels executed */
    uint64_t rescored;         /* candidates re-scored by the exact fold (TENSOR) */
    uint32_t fallback_rows;    /* rows without a first-pass proof, finished by the band-capture pass (TENSOR) */
    uint32_t kernel_launches;  /* device kernels launched by this call */
    int32_t arith_used;        /* knn_b200_arith actually run */
    int32_t n_devices;         /* GPUs used */
    double seconds;            /* whole call, host clock (validation excluded for host API) */
    double h2d_ms;             /* host->device copy, CUDA events */
    double kernel_ms;          /* all kernels, CUDA events */
    double d2h_ms;             /* device->host copy, CUDA events */
    double sweep_ms;           /* the dominant distance+top-k kernel alone, CUDA events */
    uint32_t exact_rows;       /* rows recomputed by the EXACT kernel (TENSOR: capture overflow) */
    uint32_t reserved;
} knn_b200_stats;

typedef struct knn_b200_ctx knn_b200_ctx;

KNN_B200_API int knn_b200_abi_version(void);
KNN_B200_API const char *knn_b200_last_error(void);

/* Number of visible CUDA devices with compute capability 10.x. */
KNN_B200_API int knn_b200_device_count(int *out_count);

/* A context owns one device's streams and grow-only workspace; reuse it
 * across calls (the reference CLI bench calls solve_knn twice,
 * tools/main.cpp:163-164).  Calls on one context are serialised by a mutex,
 * and each call's device work is ordered after the previous call's (an
 * event on the previous call's stream), so consecutive calls may use
 * different streams without racing on the workspace. */
KNN_B200_API int knn_b200_create(int device, knn_b200_ctx **out_ctx);
KNN_B200_API void knn_b200_destroy(knn_b200_ctx *ctx);

/* Full drop-in solve on one device.  host_vectors: n x d float32 row-major
 * (pageable or pinned).  out_index/out_dist: n x min(k, n-1), host memory.
 * Validates n >= 2, d >= 1, k >= 1 (ConfigError) and, on the device, that
 * every coordinate is finite and inside the metric's domain
 * (ValidationError, message as in distance.cpp:41-45 / dataset.cpp:25-27).
 * Pageable buffers of 16 MB or more are copied through the context's pinned
 * staging lanes (allocated on first use, freed by knn_b200_destroy). */
KNN_B200_API int knn_b200_solve(knn_b200_ctx *ctx, const float *host_vectors, uint32_t n, uint32_t d,
                   uint32_t k, int metric, int arith, uint32_t *out_index, float *out_dist,
                   knn_b200_stats *stats);

/* The reference's KNN_DOUBLE_ACCUM build (include/knn/types.hpp:9-13:
 * dist_t = double): coordinates stay float, every step is
 * acc + double(t) * double(t) with t = float(u - v) (distance.hpp:49-52,
 * :59-62), and distances are stored and ordered as doubles.  EXACT policy
 * only (SIMT FP64); results are bit-identical to the reference compiled with
 * -DKNN_DOUBLE_ACCUM.  Same arguments, validation and errors as
 * knn_b200_solve, with out_dist as n x min(k, n-1) doubles. */
KNN_B200_API int knn_b200_solve_f64(knn_b200_ctx *ctx, const float *host_vectors, uint32_t n, uint32_t d,
                                    uint32_t k, int metric, uint32_t *out_index, double *out_dist,
                                    knn_b200_stats *stats);

/* Device-resident shard solve: dev_vectors is the full n x d reference set
 * already on ctx's device (e.g. replicated by an NCCL broadcast); computes the
 * lists of query rows [row_begin, row_end) against all n vectors and writes
 * (row_end - row_begin) x min(k, n-1) results to device buffers.  Work is
 * enqueued on `stream` (a cudaStream_t; NULL is the legacy default stream,
 * as everywhere in the CUDA runtime).  The call
 * synchronises once after the validation pass (the reference validates before
 * any compute, engine.cpp:23) and, when stats is non-NULL, at the end; the
 * sweep itself is left in flight otherwise. */
KNN_B200_API int knn_b200_solve_rows_device(knn_b200_ctx *ctx, const float *dev_vectors, uint32_t n,
                               uint32_t d, uint32_t k, int metric, int arith,
                               uint32_t row_begin, uint32_t row_end, uint32_t *dev_out_index,
                               float *dev_out_dist, void *stream, knn_b200_stats *stats);

/* KNNV dataset files (the reference's load_dataset, io.cpp:64-97): magic
 * "KNNV", u32 version 1, u32 n, u32 d (little endian), then n x d float32.
 * knn_b200_knnv_header reads and checks the header (host only).
 * knn_b200_load_knnv_device reads the payload straight into dev_out
 * (capacity floats, caller-owned) through the context's pinned staging lanes
 * -- parallel preads overlapping the DMA, no whole-file host copy -- then
 * checks n >= 2, d >= 1 and every coordinate finite on the device, with the
 * reference's messages (IoError -> KNN_B200_ERR_IO, the Dataset checks ->
 * KNN_B200_ERR_VALIDATION). */
KNN_B200_API int knn_b200_knnv_header(const char *path, uint32_t *out_n, uint32_t *out_d);
KNN_B200_API int knn_b200_load_knnv_device(knn_b200_ctx *ctx, const char *path, float *dev_out, uint64_t capacity,
                                           uint32_t *out_n, uint32_t *out_d, void *stream);

/* Synthetic inputs on the device, bit-identical to the reference's
 * generate_dataset (src/io.cpp:57-62, include/knn/rng.hpp:13-23): element i of
 * the row-major n x d buffer is the (i+1)-th SplitMix64(seed) unit float.  The
 * SplitMix64 state is a Weyl sequence, so element i is computed directly as
 * mix(seed + (i+1) * 0x9e3779b97f4a7c15). */
KNN_B200_API int knn_b200_generate_device(knn_b200_ctx *ctx, float *dev_out, uint64_t count,
                                          uint64_t seed, void *stream /* NULL = legacy default */);

/* Single-process multi-GPU solve (the reference's n_lanes, engine.cpp:37-56):
 * uses min(n_gpus, device count) devices, one host thread each.  The host
 * buffer goes to device 0 once and is replicated by an NCCL broadcast
 * (ncclCommInitAll communicator); each device then runs its rank of the
 * sharded solve (knn_b200_solve_sharded_device) and writes its contiguous
 * row shard straight into the host outputs. */
KNN_B200_API int knn_b200_solve_multi(const float *host_vectors, uint32_t n, uint32_t d, uint32_t k,
                         int metric, int arith, uint32_t n_gpus, uint32_t *out_index,
                         float *out_dist, knn_b200_stats *stats);

/* knn_b200_solve_multi for the KNN_DOUBLE_ACCUM build: the same query-row
 * shards over min(n_gpus, device count) devices, each running the FP64 EXACT
 * sweep of knn_b200_solve_f64; out_dist is n x min(k, n-1) doubles. */
KNN_B200_API int knn_b200_solve_multi_f64(const float *host_vectors, uint32_t n, uint32_t d, uint32_t k,
                                          int metric, uint32_t n_gpus, uint32_t *out_index, double *out_dist,
                                          knn_b200_stats *stats);

/* ---- Multi-GPU: the sharded triangle -------
 *
 * The reference's lanes (engine.cpp:27-59; schedule.cpp:40-75 boustrophedon
 * lane_of_row; merge.cpp:10-78 merge_all) as GPUs: every unordered pair is
 * computed once across all ranks, each rank keeps row-side lists for its own
 * rows, sends column-side candidates to the rows' owners (NCCL all-to-all)
 * and merges them; results end in contiguous row shards.  One rank per GPU,
 * in one process (knn_b200_solve_multi) or one process per GPU (these calls
 * under torchrun / MPI). */

/* Test hook: dev_out (m x n fp32) = the tensor core's dot products of the
 * fp16 rows dev_a_f16 (m x d) and dev_b_f16 (n x d), row-major, computed with
 * the sweep's own instruction (tcgen05.mma kind::f16, FP32 accumulation in
 * TMEM).  Measures the accumulation error the TENSOR policy's proof bounds
 * (DESIGN.md §4). */
KNN_B200_API int knn_b200_debug_tc_dots(knn_b200_ctx *ctx, const void *dev_a_f16, uint32_t m, const void *dev_b_f16,
                                        uint32_t n, uint32_t d, float *dev_out, void *stream);

/* Host-only (no device needed): the sharded triangle's ownership of the
 * `units` 256-row units of the second column order.  Unit u goes to rank
 * lane_of_row(u) (schedule.cpp:40-44, boustrophedon over `world` ranks); a
 * rank's units, ascending, are dealt to its min(count, pairs_max) CTA pairs in
 * snake order.  out_units (units entries) lists rank 0's units in launch
 * order, then rank 1's, ...; out_counts (world entries) their counts. */
KNN_B200_API int knn_b200_tri_unit_plan(uint32_t units, uint32_t world, uint32_t pairs_max, uint32_t *out_units,
                                        uint32_t *out_counts);

/* 128 opaque bytes (an ncclUniqueId) for knn_b200_comm_init; rank 0 creates
 * it and ships it to the other ranks out of band. */
KNN_B200_API int knn_b200_comm_unique_id(void *out_id /* 128 bytes */);

/* Bind an NCCL communicator of `world` ranks to ctx (its device).  Collective:
 * every rank calls it with the same id. */
KNN_B200_API int knn_b200_comm_init(knn_b200_ctx *ctx, const void *id, int rank, int world);

/* In-place broadcast of `bytes` device bytes from rank `root` (the reference
 * set's one replication, north_star (3)). */
KNN_B200_API int knn_b200_comm_broadcast(knn_b200_ctx *ctx, void *dev_buf, uint64_t bytes, int root,
                                         void *stream);

/* Collective sharded solve.  dev_vectors: the full n x d set on every rank.
 * Rank r receives rows [R r, min(R (r + 1), n)), R = ceil(n / world), of the
 * result in dev_out_index / dev_out_dist ((rows) x min(k, n-1), device).
 * Without a communicator this is the whole problem (rows [0, n)). */
KNN_B200_API int knn_b200_solve_sharded_device(knn_b200_ctx *ctx, const float *dev_vectors, uint32_t n,
                                               uint32_t d, uint32_t k, int metric, int arith,
                                               uint32_t *dev_out_index, float *dev_out_dist, void *stream,
                                               knn_b200_stats *stats);

/* Test hook: the sharded triangle's `world` rank programs run one after
 * another on ctx's device, exchanges as device copies (no NCCL); all n rows
 * land in dev_out_index / dev_out_dist (n x min(k, n-1)).  Only for problems
 * that take the triangle (else ConfigError).  rank_ms (optional, world x 4):
 * per rank [replicated prep, sample slice, sweep + binning, merge + rescore]
 * in ms; rank_xbytes (optional, world): bytes each rank sends in the
 * column-side exchange.  stats->reserved = 1 when the logs overflowed and
 * the solve fell back to the rectangular sweep. */
KNN_B200_API int knn_b200_debug_solve_sharded_loopback(knn_b200_ctx *ctx, const float *dev_vectors, uint32_t n,
                                                       uint32_t d, uint32_t k, int metric, int world,
                                                       uint32_t *dev_out_index, float *dev_out_dist, void *stream,
                                                       knn_b200_stats *stats, float *rank_ms,
                                                       uint64_t *rank_xbytes);

#ifdef __cplusplus
}
#endif

#endif /* KNN_B200_H */
