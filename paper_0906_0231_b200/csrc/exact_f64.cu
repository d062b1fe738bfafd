// exact_f64.cu -- EXACT policy for the reference's KNN_DOUBLE_ACCUM build.
//
// Reference (paths under /root/reference/proj):
//   dist_t = double          include/knn/types.hpp:9-13, CMakeLists.txt:11,
//                            src/CMakeLists.txt:16-18
//   step_staged              include/knn/distance.hpp:49-52 / :59-62:
//                              const float t = su - sv;          (FP32 FSUB)
//                              return acc + dist_t(t) * dist_t(t);
//   fold_distance            include/knn/distance.hpp:98-105 (coordinates 0..d-1)
//   Neighbor order           include/knn/heap.hpp:21-24 (double distance, index)
//
// Arithmetic.  t is a float, so double(t) * double(t) has at most 48
// significant bits and is exact in double; acc + t*t therefore rounds once,
// which is exactly what one DFMA does.  The fold below is FSUB (rn), one
// F2F.F64.F32 widening and one DFMA per coordinate -- bit-identical to the
// reference's separately written multiply and add.  The cosine fold
// (acc + u*v) has the same property (float*float is exact in
// double).
//
// B200 design.  Same shape as exact_fused.cu: one CTA owns BM query rows and
// sweeps every column in 64-wide tiles staged through shared memory; the
// distance tile never leaves the SM.  Keys are 128-bit:
// (order-preserving u64 of the double) << 32 | index, so the unsigned order
// is the reference's (distance, index) order.  With 16-byte keys a 256-entry
// list for 64 rows does not fit in shared memory, so k > 128 runs with
// BM = 32 rows per CTA.  The widening runs on the XU pipe (16/clk/SM), which
// bounds this kernel below the DFMA rate; this policy is a correctness build,
// not the throughput path.
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "kernels.h"

namespace knnb {

namespace {

using key128 = unsigned __int128;

constexpr int F64_BN = 64;  // reference columns per tile (reference c1)
constexpr int F64_DC = 32;  // coordinates per staged chunk (reference c2)
constexpr int F64_PAD = 4;
#ifndef F64_MR
#define F64_MR 2  // query rows per thread (A/B knob: -DF64_MR=4)
#endif

__device__ __forceinline__ uint64_t double_to_ordered(double v) {
    const uint64_t b = uint64_t(__double_as_longlong(v + 0.0));  // -0.0 -> +0.0 (compares equal)
    return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}

__device__ __forceinline__ double ordered_to_double(uint64_t o) {
    const uint64_t b = (o & 0x8000000000000000ull) ? (o & 0x7fffffffffffffffull) : ~o;
    return __longlong_as_double(static_cast<long long>(b));
}

__device__ __forceinline__ key128 make_key128(double dist, uint32_t index) {
    return (key128(double_to_ordered(dist)) << 32) | index;
}

constexpr key128 kEmpty128 = ~key128(0);

template <int METRIC>
__device__ __forceinline__ double fold_step_f64(float u, float v, double acc) {
    if constexpr (METRIC == kCosine) {
        return __fma_rn(double(u), double(v), acc);  // product exact: == acc + u*v
    } else if constexpr (METRIC == kManhattan) {
        return __dadd_rn(acc, double(fabsf(__fsub_rn(u, v))));  // acc + dist_t(fabs(u - v))
    } else {
        const double t = double(__fsub_rn(u, v));
        return __fma_rn(t, t, acc);  // product exact: == acc + t*t
    }
}

template <int METRIC>
__device__ __forceinline__ double fold_finalize_f64(double acc) {
    if constexpr (METRIC == kCosine) return __dsub_rn(1.0, acc);
    if constexpr (METRIC == kRootSquares) return __dsqrt_rn(acc);
    return acc;
}

template <int BM, int KCAP>
struct F64Smem {
    float a[F64_DC][BM + F64_PAD];
    float b[F64_DC][F64_BN + F64_PAD];
    key128 cand[BM][F64_BN];
    key128 list[BM][KCAP];
    key128 thr[BM];
    uint32_t cnt[BM];
    uint32_t fill[BM];
    uint32_t qrow[BM];
};

// Merge c unsorted candidates into the ascending list of `fill` keys, keeping
// the smallest klist (keys are unique: final slot = rank in own set + rank in
// the other set).
template <int KCAP>
__device__ __forceinline__ void warp_merge_row128(key128* list, const key128* cand, uint32_t fill, uint32_t c,
                                                  uint32_t klist, int lane) {
    constexpr int LPL = (KCAP + 31) / 32;
    constexpr int CPL = (F64_BN + 31) / 32;
    key128 lv[LPL];
    uint32_t lpos[LPL];
#pragma unroll
    for (int m = 0; m < LPL; ++m) {
        const uint32_t i = lane + 32 * m;
        lpos[m] = 0xffffffffu;
        if (i < fill) {
            lv[m] = list[i];
            uint32_t rc = 0;
            for (uint32_t t = 0; t < c; ++t) rc += cand[t] < lv[m];
            lpos[m] = i + rc;
        }
    }
    key128 cv[CPL];
    uint32_t cpos[CPL];
#pragma unroll
    for (int m = 0; m < CPL; ++m) {
        const uint32_t s = lane + 32 * m;
        cpos[m] = 0xffffffffu;
        if (s < c) {
            cv[m] = cand[s];
            uint32_t rc = 0;
            for (uint32_t t = 0; t < c; ++t) rc += cand[t] < cv[m];
            uint32_t lo = 0, hi = fill;
            while (lo < hi) {
                const uint32_t mid = (lo + hi) >> 1;
                if (list[mid] < cv[m]) lo = mid + 1; else hi = mid;
            }
            cpos[m] = rc + lo;
        }
    }
    __syncwarp();
#pragma unroll
    for (int m = 0; m < LPL; ++m)
        if (lpos[m] < klist) list[lpos[m]] = lv[m];
#pragma unroll
    for (int m = 0; m < CPL; ++m)
        if (cpos[m] < klist) list[cpos[m]] = cv[m];
    __syncwarp();
}

struct F64Params {
    const float* X;  // sqrt-staged for Hellinger
    uint32_t n, d, klist;
    uint32_t row_begin, nslots;
    uint32_t* out_index;
    double* out_dist;
    int out_sqrt;
};

// MR x 4 pairs per thread: 16 column groups x BM/MR row groups.  MR = 2
// gives 16 warps per CTA: the FSUB -> F2F.F64 (XU pipe) -> DFMA chains are
// latency-bound at one CTA per SM, so more warps beat more per-thread ILP.
template <int METRIC, int BM, int KCAP, int MR>
__global__ void __launch_bounds__(BM / MR * 16) exact_f64_kernel(const F64Params p) {
    constexpr int THREADS = BM / MR * 16;
    constexpr int WARPS = THREADS / 32;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    F64Smem<BM, KCAP>& S = *reinterpret_cast<F64Smem<BM, KCAP>*>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int tx = tid & 15, ty = tid >> 4;
    const float* __restrict__ X = p.X;
    const uint32_t n = p.n, d = p.d, klist = p.klist;
    const uint32_t slot0 = blockIdx.x * BM;

    for (int i = tid; i < BM; i += THREADS) {
        const uint32_t s = slot0 + i;
        S.qrow[i] = s < p.nslots ? p.row_begin + s : 0xffffffffu;
        S.thr[i] = kEmpty128;
        S.cnt[i] = 0;
        S.fill[i] = 0;
    }
    __syncthreads();

    // Staging is register-prefetched: the global loads of the next
    // (tile, coordinate-chunk) step are in flight while this step computes.
    // Lane = coordinate, one row per warp step; coordinates past d stage as 0
    // on both sides (a 0 step adds +0.0, leaving the accumulator's bits).
    constexpr int RPW = F64_BN / WARPS;  // staged rows per warp and side
    const uint32_t nchunk = (d + F64_DC - 1) / F64_DC;
    float ra[RPW], rb[RPW];
    auto prefetch = [&](uint32_t c0, uint32_t j0) {
        const uint32_t j = j0 + lane;
#pragma unroll
        for (int m = 0; m < RPW; ++m) {
            const int rr = warp + m * WARPS;
            ra[m] = 0.0f;
            if (rr < BM) {
                const uint32_t q = S.qrow[rr];
                if (q != 0xffffffffu && j < d) ra[m] = X[size_t(q) * d + j];
            }
            const uint32_t col = c0 + rr;
            rb[m] = (col < n && j < d) ? X[size_t(col) * d + j] : 0.0f;
        }
    };
    prefetch(0, 0);
    for (uint32_t c0 = 0; c0 < n; c0 += F64_BN) {
        double acc[MR][4];
#pragma unroll
        for (int i = 0; i < MR; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;

        for (uint32_t jc = 0; jc < nchunk; ++jc) {
#pragma unroll
            for (int m = 0; m < RPW; ++m) {
                const int rr = warp + m * WARPS;
                if (rr < BM) S.a[lane][rr] = ra[m];
                S.b[lane][rr] = rb[m];
            }
            __syncthreads();
            if (jc + 1 < nchunk) prefetch(c0, (jc + 1) * F64_DC);
            else if (c0 + F64_BN < n) prefetch(c0 + F64_BN, 0);
#pragma unroll 4
            for (int jj = 0; jj < F64_DC; ++jj) {
                float av[MR];
                if constexpr (MR == 4) {
                    const float4 a4 = *reinterpret_cast<const float4*>(&S.a[jj][ty * 4]);
                    av[0] = a4.x; av[1] = a4.y; av[2] = a4.z; av[3] = a4.w;
                } else if constexpr (MR == 2) {
                    const float2 a2 = *reinterpret_cast<const float2*>(&S.a[jj][ty * 2]);
                    av[0] = a2.x; av[1] = a2.y;
                } else {
                    av[0] = S.a[jj][ty];
                }
                const float4 b4 = *reinterpret_cast<const float4*>(&S.b[jj][tx * 4]);
                const float bv[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
                for (int i = 0; i < MR; ++i)
#pragma unroll
                    for (int c = 0; c < 4; ++c) acc[i][c] = fold_step_f64<METRIC>(bv[c], av[i], acc[i][c]);
            }
            __syncthreads();
        }

#pragma unroll
        for (int i = 0; i < MR; ++i) {
            const int rr = ty * MR + i;
            const uint32_t q = S.qrow[rr];
            if (q == 0xffffffffu) continue;
            const key128 thr = S.thr[rr];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const uint32_t col = c0 + tx * 4 + c;
                if (col >= n || col == q) continue;
                const key128 key = make_key128(fold_finalize_f64<METRIC>(acc[i][c]), col);
                if (key < thr) {
                    const uint32_t s = atomicAdd(&S.cnt[rr], 1u);
                    S.cand[rr][s] = key;
                }
            }
        }
        __syncthreads();
        for (int rr = warp; rr < BM; rr += WARPS) {
            const uint32_t c = S.cnt[rr];
            if (c == 0) continue;
            const uint32_t fill = S.fill[rr];
            warp_merge_row128<KCAP>(S.list[rr], S.cand[rr], fill, c, klist, lane);
            if (lane == 0) {
                const uint32_t nf = min(fill + c, klist);
                S.fill[rr] = nf;
                S.thr[rr] = nf == klist ? S.list[rr][klist - 1] : kEmpty128;
                S.cnt[rr] = 0;
            }
        }
        __syncthreads();
    }

    for (int rr = warp; rr < BM; rr += WARPS) {
        const uint32_t s = slot0 + rr;
        if (s >= p.nslots) continue;
        for (uint32_t t = lane; t < klist; t += 32) {
            const key128 key = S.list[rr][t];
            p.out_index[size_t(s) * klist + t] = uint32_t(key);
            const double dv = ordered_to_double(uint64_t(key >> 32));
            p.out_dist[size_t(s) * klist + t] = p.out_sqrt ? __dsqrt_rn(dv) : dv;
        }
    }
}

constexpr int kF64MR = F64_MR;

template <int METRIC, int BM, int KCAP>
cudaError_t launch_f64_t(const F64Params& p, cudaStream_t stream) {
    // 32-row CTAs (k > 128) keep 16 warps with one row per thread
    constexpr int MR = BM == 32 ? 1 : kF64MR;
    const size_t smem = sizeof(F64Smem<BM, KCAP>);
    auto kern = exact_f64_kernel<METRIC, BM, KCAP, MR>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    kern<<<(p.nslots + BM - 1) / BM, BM / MR * 16, smem, stream>>>(p);
    return cudaGetLastError();
}

template <int METRIC>
cudaError_t launch_f64_m(const F64Params& p, cudaStream_t stream) {
    if (p.klist <= 32) return launch_f64_t<METRIC, 64, 32>(p, stream);
    if (p.klist <= 64) return launch_f64_t<METRIC, 64, 64>(p, stream);
    if (p.klist <= 128) return launch_f64_t<METRIC, 64, 128>(p, stream);
    return launch_f64_t<METRIC, 32, 256>(p, stream);
}

}  // namespace

cudaError_t launch_exact_f64(int metric, const float* X, uint32_t n, uint32_t d, uint32_t klist,
                             uint32_t row_begin, uint32_t row_end, uint32_t* out_index, double* out_dist,
                             int out_sqrt, cudaStream_t stream) {
    if (row_end <= row_begin) return cudaSuccess;
    if (klist > kExactMaxK) return cudaErrorInvalidValue;
    const F64Params p{X, n, d, klist, row_begin, row_end - row_begin, out_index, out_dist, out_sqrt};
    // Hellinger arrives sqrt-staged and folds exactly like sqeuclidean.
    if (metric == kCosine) return launch_f64_m<kCosine>(p, stream);
    if (metric == kManhattan) return launch_f64_m<kManhattan>(p, stream);
    if (metric == kRootSquares) return launch_f64_m<kRootSquares>(p, stream);
    return launch_f64_m<kSqEuclidean>(p, stream);
}

}  // namespace knnb
