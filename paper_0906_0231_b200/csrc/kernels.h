// kernels.h -- host-side launchers for the device kernels (internal).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace knnb {

// validate: flags[0] = first non-finite flat index, flags[1] = first domain
// violation (negative coordinate when check_nonneg); both must be preset to
// all-ones by the caller.
cudaError_t launch_validate(const float* X, uint64_t count, int check_nonneg,
                            unsigned long long* flags, int sm_count, cudaStream_t stream);

cudaError_t launch_stage_sqrt(const float* X, float* Y, uint64_t count, int sm_count,
                              cudaStream_t stream);

cudaError_t launch_generate(float* out, uint64_t count, uint64_t seed, int sm_count, cudaStream_t stream);

// EXACT fused sweep.  Output slot s (0 <= s < row_end - row_begin) holds the
// list of query row `rows ? rows[s] : row_begin + s`; klist = min(k, n-1) <= 256.
// out_sqrt: report sqrtf(distance) (the Euclidean metric) -- selection is
// unaffected because sqrtf is monotone and the lists are final.  With an
// explicit row list, slot s is written to output row rows[s] - scatter_base.
// `scratch` (exact_scratch_bytes) lets few rows spread their columns over
// every SM; null forces one chunk.
cudaError_t launch_exact_fused(int metric, const float* X, uint32_t n, uint32_t d, uint32_t klist,
                               const uint32_t* rows, uint32_t row_begin, uint32_t row_end,
                               uint32_t* out_index, float* out_dist, int out_sqrt,
                               uint32_t scatter_base, void* scratch, int sm_count, cudaStream_t stream);
size_t exact_scratch_bytes(uint32_t nslots, uint32_t n, uint32_t klist, int sm_count);

constexpr uint32_t kExactMaxK = 256;  // longest list the fused EXACT kernels keep on chip

// EXACT lists longer than kExactMaxK (exact_bigk.cu): batches of query rows,
// every distance as a key, a stable segmented radix sort per row, the first
// klist kept.  f64: the KNN_DOUBLE_ACCUM fold and double distances.
cudaError_t launch_exact_bigk(int metric, int f64, const float* X, uint32_t n, uint32_t d, uint32_t klist,
                              uint32_t row_begin, uint32_t row_end, uint32_t* out_index, void* out_dist,
                              int out_sqrt, void* ws, int sm_count, cudaStream_t stream);
size_t exact_bigk_workspace_bytes(uint32_t rows, uint32_t n, int f64);
uint32_t exact_bigk_batch_rows(uint32_t rows, uint32_t n);

// EXACT sweep with double accumulation (the reference's KNN_DOUBLE_ACCUM
// build, exact_f64.cu); output rows row_begin..row_end-1 in slot order.
cudaError_t launch_exact_f64(int metric, const float* X, uint32_t n, uint32_t d, uint32_t klist,
                             uint32_t row_begin, uint32_t row_end, uint32_t* out_index, double* out_dist,
                             int out_sqrt, cudaStream_t stream);

// TENSOR policy (tensor_path.cu)
struct TensorPathArgs {
    const float* X;  // fp32, sqrt-staged for Hellinger
    uint32_t n, d, klist, kp;
    uint32_t row_begin, row_end;
    int fold;        // kSqEuclidean or kCosine
    int out_sqrt;
    uint32_t* out_index;
    float* out_dist;
    void* workspace;      // tensor_workspace_bytes(), or null: taken from alloc_ws(alloc2_ctx, bytes) on demand
    void* (*alloc_ws)(void* ctx, size_t bytes);
    void* exact_scratch;  // exact_scratch_bytes(row_end - row_begin, ...) for fallback rows
    void* host_scratch;   // 64 B pinned
    int sm_count;
    cudaStream_t stream;
    cudaEvent_t ev_sweep0, ev_sweep1;  // optional, around the sweep kernel
    // grow-only allocator for the second (band-capture) pass, sized on the
    // host once the number of unproven rows is known
    void* (*alloc2)(void* ctx, size_t bytes);
    void* alloc2_ctx;
    // grow-only device memory by slot (the threshold triangle; null: not available)
    void* (*shard_alloc)(void* ctx, int slot, size_t bytes);
    void* shard_ctx;
};
struct TensorPathResult {
    unsigned long long rescored = 0;
    uint32_t fallback_rows = 0;  // rows without a first-pass proof (band-capture pass)
    uint32_t exact_rows = 0;     // rows recomputed by the EXACT kernel
    uint32_t launches = 0;
};
uint32_t tensor_kp_for(uint32_t klist);  // 0 = unsupported
size_t tensor_workspace_bytes(uint32_t n, uint32_t d, uint32_t row_begin, uint32_t row_end, uint32_t klist,
                              int sm_count);
cudaError_t run_tensor_path(const TensorPathArgs& a, TensorPathResult& r);
bool tri_eligible(uint32_t n, uint32_t d, uint32_t klist, int fold);

// tc_probe.cu: out (m x n, fp32) = the tensor core's dots of fp16 rows
// (row-major m x d and n x d), with the sweep's MMA instruction.
cudaError_t launch_tc_dots(const void* a_f16, uint32_t m, const void* b_f16, uint32_t n, uint32_t d, float* out,
                           cudaStream_t stream);

// The triangle sweep sharded over `world` ranks (tri_shard.cuh).
// alloc(ctx, slot, bytes): grow-only device memory per slot.  a.row_begin = 0,
// a.row_end = n; a.out_* are full n-row arrays that receive the rank's own
// rows (loopback: every rank's rows).  *overflow: column-side logs overflowed
// (the caller redoes the solve without the triangle).
typedef void* (*ShardAlloc)(void* ctx, int slot, size_t bytes);
constexpr uint32_t kTriMaxWorld = 64;
// Unit ownership (host): rank r's units are units[sum(counts[<r]) ...], in the
// order its CTA pairs take them.
void tri_unit_plan(uint32_t U, uint32_t world, uint32_t pairs_max, uint32_t* units, uint32_t* counts);
// tcap: the threshold triangle (10 < k <= 128) instead of the list triangle (k <= 10).
bool tcap_eligible(uint32_t n, uint32_t d, uint32_t klist);
cudaError_t run_tri_loopback(const TensorPathArgs& a, uint32_t world, ShardAlloc alloc, void* actx,
                             TensorPathResult& r, float* rank_ms, unsigned long long* xbytes, bool* overflow,
                             bool tcap);
}  // namespace knnb
typedef struct ncclComm* ncclComm_t;
namespace knnb {
cudaError_t run_tri_nccl(const TensorPathArgs& a, ncclComm_t comm, uint32_t rank, uint32_t world, ShardAlloc alloc,
                         void* actx, TensorPathResult& r, bool* overflow, bool tcap);

}  // namespace knnb
