// exact_bigk.cu -- EXACT policy for lists longer than the fused kernels hold.
//
// The reference keeps min(k, n-1) neighbours per row for any k (heap.cpp:66-70:
// HeapStore capacity; NeighborHeap push/drain heap.cpp:18-42).  The fused
// kernels (exact_fused.cu, exact_f64.cu) keep a row's list in shared memory,
// which caps it at kExactMaxK = 256 entries.  Longer lists take this path:
//
//   1. tile kernel   a batch of B query rows against every column, 64 x 64
//                    tiles, the reference fold (FSUB/FMUL/FADD in coordinate
//                    order, distance.hpp:98-105) -- every distance written
//                    out as an order-preserving key, self as the empty key;
//   2. segmented radix sort (CUB) of each row's n keys.  Float keys are
//                    (ordered distance << 32 | index), unique, so their order
//                    is the reference's (distance, index) order (heap.hpp:21-24);
//                    double keys carry the index as the sort's value, laid out
//                    in column order, and the radix sort is stable, so equal
//                    distances keep ascending index order;
//   3. the first min(k, n-1) keys of each row become its list.
//
// This is HBM-bound (B x n keys written, sorted, read), not fused: it serves
// k > 256, where a list per row no longer fits on chip.
#include <cub/device/device_segmented_radix_sort.cuh>
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

#include "common.cuh"
#include "kernels.h"

namespace knnb {

namespace {

constexpr int BK_BM = 64, BK_BN = 64, BK_DC = 32, BK_PAD = 4, BK_THREADS = 256;

__device__ __forceinline__ uint64_t double_to_ordered_bk(double v) {
    const uint64_t b = uint64_t(__double_as_longlong(v + 0.0));  // -0.0 -> +0.0
    return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double ordered_to_double_bk(uint64_t o) {
    const uint64_t b = (o & 0x8000000000000000ull) ? (o & 0x7fffffffffffffffull) : ~o;
    return __longlong_as_double(static_cast<long long>(b));
}

template <int METRIC, bool F64>
__device__ __forceinline__ void step_bk(float u, float v, float& a32, double& a64) {
    if constexpr (F64) {
        // distance.hpp:49-52 with dist_t = double: FSUB, exact widened product, one rounding
        if constexpr (METRIC == kCosine) a64 = __fma_rn(double(u), double(v), a64);
        else if constexpr (METRIC == kManhattan) a64 = __dadd_rn(a64, double(fabsf(__fsub_rn(u, v))));
        else {
            const double t = double(__fsub_rn(u, v));
            a64 = __fma_rn(t, t, a64);
        }
    } else {
        a32 = fold_step<METRIC>(u, v, a32);
    }
}

struct BigkParams {
    const float* X;
    uint32_t n, d;
    uint32_t row0, rows;  // batch: query rows row0 .. row0 + rows - 1
    uint64_t* keys;       // [rows][n]: F64 = ordered double, else (ordered float << 32 | col)
    uint32_t* cols;       // F64 only: [rows][n] column index (the sort's values)
};

template <int METRIC, bool F64>
__global__ void __launch_bounds__(BK_THREADS) bigk_tile_kernel(const BigkParams p) {
    __shared__ __align__(16) float sa[BK_DC][BK_BM + BK_PAD];
    __shared__ __align__(16) float sb[BK_DC][BK_BN + BK_PAD];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, tx = tid & 15, ty = tid >> 4;
    const uint32_t s0 = blockIdx.x * BK_BM, c0 = blockIdx.y * BK_BN;
    float a32[4][4];
    double a64[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            a32[i][j] = 0.0f;
            a64[i][j] = 0.0;
        }
    for (uint32_t j0 = 0; j0 < p.d; j0 += BK_DC) {
        // coordinates past d are 0 on both sides: a +0.0 step leaves the bits unchanged
        const uint32_t j = j0 + lane;
        for (int rr = warp; rr < BK_BM; rr += BK_THREADS / 32) {
            const uint32_t s = s0 + rr, col = c0 + rr;
            sa[lane][rr] = (s < p.rows && j < p.d) ? p.X[size_t(p.row0 + s) * p.d + j] : 0.0f;
            sb[lane][rr] = (col < p.n && j < p.d) ? p.X[size_t(col) * p.d + j] : 0.0f;
        }
        __syncthreads();
#pragma unroll 8
        for (int jj = 0; jj < BK_DC; ++jj) {
            const float4 q4 = *reinterpret_cast<const float4*>(&sa[jj][ty * 4]);
            const float4 r4 = *reinterpret_cast<const float4*>(&sb[jj][tx * 4]);
            const float qv[4] = {q4.x, q4.y, q4.z, q4.w};
            const float rv[4] = {r4.x, r4.y, r4.z, r4.w};
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int c = 0; c < 4; ++c) step_bk<METRIC, F64>(rv[c], qv[i], a32[i][c], a64[i][c]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const uint32_t s = s0 + ty * 4 + i;
        if (s >= p.rows) continue;
        const uint32_t q = p.row0 + s;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const uint32_t col = c0 + tx * 4 + c;
            if (col >= p.n) continue;
            const size_t at = size_t(s) * p.n + col;
            if constexpr (F64) {
                const double dist = METRIC == kCosine       ? __dsub_rn(1.0, a64[i][c])
                                    : METRIC == kRootSquares ? __dsqrt_rn(a64[i][c])
                                                             : a64[i][c];
                p.keys[at] = col == q ? kEmptyKey : double_to_ordered_bk(dist);
                p.cols[at] = col;
            } else {
                p.keys[at] = col == q ? kEmptyKey : make_key(fold_finalize<METRIC>(a32[i][c]), col);
            }
        }
    }
}

// The first klist sorted keys of every row of the batch -> the output rows.
template <bool F64>
__global__ void bigk_emit_kernel(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ cols, uint32_t n,
                                 uint32_t rows, uint32_t klist, int out_sqrt, uint32_t* __restrict__ out_index,
                                 void* __restrict__ out_dist) {
    const size_t total = size_t(rows) * klist;
    for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += size_t(gridDim.x) * blockDim.x) {
        const size_t s = i / klist, t = i % klist;
        const uint64_t key = keys[s * n + t];
        if constexpr (F64) {
            out_index[i] = cols[s * n + t];
            const double dv = ordered_to_double_bk(key);
            static_cast<double*>(out_dist)[i] = out_sqrt ? __dsqrt_rn(dv) : dv;
        } else {
            out_index[i] = uint32_t(key);
            const float dv = ordered_to_float(uint32_t(key >> 32));
            static_cast<float*>(out_dist)[i] = out_sqrt ? __fsqrt_rn(dv) : dv;
        }
    }
}

__global__ void bigk_offsets_kernel(int* __restrict__ off, uint32_t rows, uint32_t n) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i <= rows; i += gridDim.x * blockDim.x)
        off[i] = int(uint64_t(i) * n);
}

// Rows per batch: at most ~2^27 keys (1 GB of keys, double-buffered) and
// under 2^31 sort items.
uint32_t bigk_batch(uint32_t rows, uint32_t n) {
    uint64_t b = (uint64_t(1) << 27) / n;
    if (b < 1) b = 1;
    return uint32_t(b < rows ? b : rows);
}

template <bool F64>
size_t bigk_sort_temp(uint32_t batch, uint32_t n) {
    size_t t = 0;
    const int items = int(uint64_t(batch) * n);
    if constexpr (F64)
        cub::DeviceSegmentedRadixSort::SortPairs(nullptr, t, static_cast<const uint64_t*>(nullptr),
                                                 static_cast<uint64_t*>(nullptr), static_cast<const uint32_t*>(nullptr),
                                                 static_cast<uint32_t*>(nullptr), items, int(batch),
                                                 static_cast<const int*>(nullptr), static_cast<const int*>(nullptr) + 1);
    else
        cub::DeviceSegmentedRadixSort::SortKeys(nullptr, t, static_cast<const uint64_t*>(nullptr),
                                                static_cast<uint64_t*>(nullptr), items, int(batch),
                                                static_cast<const int*>(nullptr), static_cast<const int*>(nullptr) + 1);
    return t;
}

size_t al256(size_t x) { return (x + 255) / 256 * 256; }

template <bool F64>
size_t bigk_bytes(uint32_t rows, uint32_t n) {
    const uint32_t b = bigk_batch(rows, n);
    const size_t items = size_t(b) * n;
    size_t s = 2 * al256(items * 8) + al256((size_t(b) + 1) * 4) + al256(bigk_sort_temp<F64>(b, n));
    if (F64) s += 2 * al256(items * 4);
    return s;
}

template <int METRIC, bool F64>
cudaError_t run_bigk(const float* X, uint32_t n, uint32_t d, uint32_t klist, uint32_t row_begin, uint32_t row_end,
                     uint32_t* out_index, void* out_dist, int out_sqrt, void* ws, int sm_count, cudaStream_t st) {
    const uint32_t rows = row_end - row_begin;
    const uint32_t b = bigk_batch(rows, n);
    const size_t items = size_t(b) * n;
    uint8_t* w = static_cast<uint8_t*>(ws);
    auto take = [&](size_t x) {
        uint8_t* q = w;
        w += al256(x);
        return q;
    };
    uint64_t* k0 = reinterpret_cast<uint64_t*>(take(items * 8));
    uint64_t* k1 = reinterpret_cast<uint64_t*>(take(items * 8));
    int* off = reinterpret_cast<int*>(take((size_t(b) + 1) * 4));
    size_t tb = bigk_sort_temp<F64>(b, n);
    void* temp = take(tb);
    uint32_t* v0 = F64 ? reinterpret_cast<uint32_t*>(take(items * 4)) : nullptr;
    uint32_t* v1 = F64 ? reinterpret_cast<uint32_t*>(take(items * 4)) : nullptr;
    cudaError_t e;
    for (uint32_t r0 = 0; r0 < rows; r0 += b) {
        const uint32_t m = rows - r0 < b ? rows - r0 : b;
        BigkParams p{X, n, d, row_begin + r0, m, k0, v0};
        bigk_tile_kernel<METRIC, F64><<<dim3((m + BK_BM - 1) / BK_BM, (n + BK_BN - 1) / BK_BN), BK_THREADS, 0, st>>>(p);
        bigk_offsets_kernel<<<(m + 256) / 256, 256, 0, st>>>(off, m, n);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
        const int mi = int(size_t(m) * n);
        if constexpr (F64)
            e = cub::DeviceSegmentedRadixSort::SortPairs(temp, tb, k0, k1, v0, v1, mi, int(m), off, off + 1, 0, 64, st);
        else
            e = cub::DeviceSegmentedRadixSort::SortKeys(temp, tb, k0, k1, mi, int(m), off, off + 1, 0, 64, st);
        if (e != cudaSuccess) return e;
        const size_t obase = size_t(r0) * klist;
        void* od = F64 ? static_cast<void*>(static_cast<double*>(out_dist) + obase)
                       : static_cast<void*>(static_cast<float*>(out_dist) + obase);
        bigk_emit_kernel<F64><<<sm_count * 4, 256, 0, st>>>(k1, v1, n, m, klist, out_sqrt, out_index + obase, od);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    return cudaSuccess;
}

}  // namespace

uint32_t exact_bigk_batch_rows(uint32_t rows, uint32_t n) { return bigk_batch(rows, n); }

size_t exact_bigk_workspace_bytes(uint32_t rows, uint32_t n, int f64) {
    return f64 ? bigk_bytes<true>(rows, n) : bigk_bytes<false>(rows, n);
}

cudaError_t launch_exact_bigk(int metric, int f64, const float* X, uint32_t n, uint32_t d, uint32_t klist,
                              uint32_t row_begin, uint32_t row_end, uint32_t* out_index, void* out_dist,
                              int out_sqrt, void* ws, int sm_count, cudaStream_t stream) {
    if (row_end <= row_begin) return cudaSuccess;
    // Hellinger arrives sqrt-staged and folds exactly like sqeuclidean.
    auto run = [&](auto m, auto f) {
        return run_bigk<decltype(m)::value, decltype(f)::value>(X, n, d, klist, row_begin, row_end, out_index,
                                                                 out_dist, out_sqrt, ws, sm_count, stream);
    };
    using T = std::true_type;
    using F = std::false_type;
    switch (metric) {
    case kCosine: return f64 ? run(std::integral_constant<int, kCosine>{}, T{}) : run(std::integral_constant<int, kCosine>{}, F{});
    case kManhattan:
        return f64 ? run(std::integral_constant<int, kManhattan>{}, T{})
                   : run(std::integral_constant<int, kManhattan>{}, F{});
    case kRootSquares:
        return f64 ? run(std::integral_constant<int, kRootSquares>{}, T{})
                   : run(std::integral_constant<int, kRootSquares>{}, F{});
    default:
        return f64 ? run(std::integral_constant<int, kSqEuclidean>{}, T{})
                   : run(std::integral_constant<int, kSqEuclidean>{}, F{});
    }
}

}  // namespace knnb
