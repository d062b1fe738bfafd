// exact_fused.cu -- EXACT policy: fused Phase 1 + Phase 2 on SIMT FP32.
//
// Reference (paths under /root/reference/proj):
//   Phase 1  fill_tile<Metric>   src/dist_kernel.cpp:42-115  (bsize x c1 x c2 blocking,
//            per-pair fold over coordinates 0..d-1 in order)
//   Phase 2  k_smallest_push     src/select.cpp:60-130 (root-hint filter, buffer, flush)
//            NeighborHeap        src/heap.cpp:18-64
//
// B200 design.  One CTA owns EX_BM query rows and sweeps every reference
// column in EX_BN-wide tiles; coordinates are staged through shared memory in
// EX_DC-wide chunks (the paper's C2 chunking).  Each thread
// accumulates a 4x4 micro-tile with __fsub_rn/__fmul_rn/__fadd_rn -- the same
// separately rounded sub/mul/add sequence, in the same coordinate order, as
// fold_distance (include/knn/distance.hpp:98-105) -- so every distance is
// bit-identical to the reference.  The distance tile never leaves the SM:
// each value is compared against its row's admission threshold (the
// reference's root hint, heap.hpp:86-90, here exact because one CTA owns the
// row) and survivors are appended to a per-row shared-memory buffer, which a
// warp then merges into the row's sorted top-k list by rank computation.
// Keys are (ordered distance bits << 32 | index), so the u64 order is the
// reference's (distance, index) order and ties break to the smaller index.
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "kernels.h"

namespace knnb {

constexpr int EX_BM = 64;        // query rows per CTA (reference bsize)
constexpr int EX_BN = 64;        // reference columns per tile (reference c1)
constexpr int EX_DC = 32;        // coordinates per staged chunk (reference c2)
constexpr int EX_THREADS = 256;  // 16 x 16 threads, 4 x 4 pairs each
constexpr int EX_PAD = 4;

template <int KCAP>
struct ExactSmem {
    float a[EX_DC][EX_BM + EX_PAD];  // query chunk, coordinate-major
    float b[EX_DC][EX_BN + EX_PAD];  // reference chunk, coordinate-major
    uint64_t cand[EX_BM][EX_BN];     // per-row survivor buffer (one tile can't overflow it)
    uint64_t list[EX_BM][KCAP];      // per-row sorted top-k keys
    uint64_t thr[EX_BM];             // admission threshold: list[k-1] once full, else +inf
    uint32_t cnt[EX_BM];
    uint32_t fill[EX_BM];
};

// Merge `c` unsorted candidate keys into the ascending list of `fill` keys,
// keeping the smallest `klist`.  Keys are unique, so each element's final
// slot is its rank in its own set plus its rank in the other set.
template <int KCAP>
__device__ __forceinline__ void warp_merge_row(uint64_t* list, const uint64_t* cand, uint32_t fill,
                                               uint32_t c, uint32_t klist, int lane) {
    constexpr int LPL = (KCAP + 31) / 32;
    constexpr int CPL = (EX_BN + 31) / 32;
    uint64_t lv[LPL];
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
    uint64_t cv[CPL];
    uint32_t cpos[CPL];
#pragma unroll
    for (int m = 0; m < CPL; ++m) {
        const uint32_t s = lane + 32 * m;
        cpos[m] = 0xffffffffu;
        if (s < c) {
            cv[m] = cand[s];
            uint32_t rc = 0;
            for (uint32_t t = 0; t < c; ++t) rc += cand[t] < cv[m];
            uint32_t lo = 0, hi = fill;  // lower_bound in the list
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

struct ExactParams {
    const float* X;
    uint32_t n, d, klist;
    const uint32_t* rows;     // explicit query rows, or null for row_begin + slot
    uint32_t row_begin, nslots;
    uint32_t col_chunk;       // columns per blockIdx.y chunk
    uint32_t* out_index;      // final lists (unsplit launch) ...
    float* out_dist;
    int out_sqrt;
    uint32_t scatter_base;    // with `rows`: output row = rows[s] - scatter_base
    uint64_t* partial;        // ... or per-chunk partial key lists [chunk][slot][klist]
};

template <int METRIC, int KCAP>
__global__ void __launch_bounds__(EX_THREADS) exact_fused_kernel(const ExactParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    ExactSmem<KCAP>& S = *reinterpret_cast<ExactSmem<KCAP>*>(smem_raw);
    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int warp = tid >> 5;
    const int tx = tid & 15;
    const int ty = tid >> 4;
    const float* __restrict__ X = p.X;
    const uint32_t n = p.n, d = p.d, klist = p.klist;
    // Slot s of this CTA is output slot (blockIdx.x*EX_BM + s); its query row
    // is row_begin + slot, or rows[slot] when an explicit row list is given
    // (the tensor path's fallback rows).  blockIdx.y selects a column chunk:
    // few rows are spread over every SM by splitting their columns, and the
    // per-chunk lists are merged by exact_merge_kernel.
    const uint32_t slot0 = blockIdx.x * EX_BM;
    const uint32_t cbeg = blockIdx.y * p.col_chunk;
    const uint32_t cend = min(n, cbeg + p.col_chunk);

    __shared__ uint32_t qrow[EX_BM];
    for (int i = tid; i < EX_BM; i += EX_THREADS) {
        const uint32_t s = slot0 + i;
        qrow[i] = s < p.nslots ? (p.rows ? p.rows[s] : p.row_begin + s) : 0xffffffffu;
        S.thr[i] = kEmptyKey;
        S.cnt[i] = 0;
        S.fill[i] = 0;
    }
    __syncthreads();
    const uint32_t kcap = min(klist, cend - cbeg);  // a chunk may hold fewer than k columns

    for (uint32_t c0 = cbeg; c0 < cend; c0 += EX_BN) {
        float acc[4][4];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] = 0.0f;

        for (uint32_t j0 = 0; j0 < d; j0 += EX_DC) {
            // Coalesced staging: lane = coordinate, one row per warp step.
            // Coordinates past d are staged as 0 on both sides; a 0 step adds
            // +0.0 to a non-negative (or, for cosine, any non -0.0)
            // accumulator, which leaves its bits unchanged.
            const uint32_t j = j0 + lane;
            for (int rr = warp; rr < EX_BM; rr += EX_THREADS / 32) {
                const uint32_t q = qrow[rr];
                S.a[lane][rr] = (q != 0xffffffffu && j < d) ? X[size_t(q) * d + j] : 0.0f;
                const uint32_t col = c0 + rr;
                S.b[lane][rr] = (col < cend && j < d) ? X[size_t(col) * d + j] : 0.0f;
            }
            __syncthreads();
#pragma unroll 8
            for (int jj = 0; jj < EX_DC; ++jj) {
                const float4 a4 = *reinterpret_cast<const float4*>(&S.a[jj][ty * 4]);
                const float4 b4 = *reinterpret_cast<const float4*>(&S.b[jj][tx * 4]);
                const float av[4] = {a4.x, a4.y, a4.z, a4.w};
                const float bv[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int c = 0; c < 4; c += 2)  // packed terms for columns c, c + 1 (FADD2/FMUL2)
                        fold_step2<METRIC>(bv[c], bv[c + 1], av[i], av[i], acc[i][c], acc[i][c + 1]);
            }
            __syncthreads();
        }

        // Phase 2 filter: the tile stays on chip.
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int rr = ty * 4 + i;
            const uint32_t q = qrow[rr];
            if (q == 0xffffffffu) continue;
            const uint64_t thr = S.thr[rr];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const uint32_t col = c0 + tx * 4 + c;
                if (col >= cend || col == q) continue;
                const uint64_t key = make_key(fold_finalize<METRIC>(acc[i][c]), col);
                if (key < thr) {
                    const uint32_t s = atomicAdd(&S.cnt[rr], 1u);
                    S.cand[rr][s] = key;
                }
            }
        }
        __syncthreads();
        for (int rr = warp; rr < EX_BM; rr += EX_THREADS / 32) {
            const uint32_t c = S.cnt[rr];
            if (c == 0) continue;
            const uint32_t fill = S.fill[rr];
            warp_merge_row<KCAP>(S.list[rr], S.cand[rr], fill, c, klist, lane);
            if (lane == 0) {
                const uint32_t nf = min(fill + c, klist);
                S.fill[rr] = nf;
                S.thr[rr] = nf == klist ? S.list[rr][klist - 1] : kEmptyKey;
                S.cnt[rr] = 0;
            }
        }
        __syncthreads();
    }

    for (int rr = warp; rr < EX_BM; rr += EX_THREADS / 32) {
        const uint32_t s = slot0 + rr;
        if (s >= p.nslots) continue;
        if (p.partial) {
            uint64_t* out = p.partial + (size_t(blockIdx.y) * p.nslots + s) * klist;
            for (uint32_t t = lane; t < klist; t += 32) out[t] = t < S.fill[rr] ? S.list[rr][t] : kEmptyKey;
            continue;
        }
        (void)kcap;
        const size_t orow = p.rows ? size_t(qrow[rr] - p.scatter_base) : size_t(s);
        for (uint32_t t = lane; t < klist; t += 32) {
            const uint64_t key = S.list[rr][t];
            p.out_index[orow * klist + t] = uint32_t(key);
            const float dv = ordered_to_float(uint32_t(key >> 32));
            p.out_dist[orow * klist + t] = p.out_sqrt ? __fsqrt_rn(dv) : dv;
        }
    }
}

// k-way merge of the per-chunk lists of one slot (one warp per slot): the
// column chunks are disjoint, so the union's k smallest keys are the answer.
__global__ void __launch_bounds__(256) exact_merge_kernel(const ExactParams p, uint32_t nchunks) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t s = blockIdx.x * 8 + warp;
    if (s >= p.nslots) return;
    const uint32_t klist = p.klist;
    const uint32_t q = p.rows ? p.rows[s] : p.row_begin + s;
    const size_t orow = p.rows ? size_t(q - p.scatter_base) : size_t(s);
    // each lane walks the heads of chunks lane, lane+32, ...
    constexpr int MAXC = 8;  // up to 256 chunks
    uint32_t head[MAXC];
#pragma unroll
    for (int m = 0; m < MAXC; ++m) head[m] = 0;
    for (uint32_t t = 0; t < klist; ++t) {
        uint64_t best = kEmptyKey;
        int bm = -1;
#pragma unroll
        for (int m = 0; m < MAXC; ++m) {
            const uint32_t c = lane + 32 * m;
            if (c < nchunks && head[m] < klist) {
                const uint64_t v = p.partial[(size_t(c) * p.nslots + s) * klist + head[m]];
                if (v < best) {
                    best = v;
                    bm = m;
                }
            }
        }
        uint64_t wbest = best;
        for (int o = 16; o; o >>= 1) {
            const uint64_t other = __shfl_xor_sync(0xffffffffu, wbest, o);
            wbest = other < wbest ? other : wbest;
        }
        if (bm >= 0 && best == wbest && wbest != kEmptyKey) {
#pragma unroll
            for (int m = 0; m < MAXC; ++m)
                if (m == bm) ++head[m];
        }
        if (lane == 0) {
            p.out_index[orow * klist + t] = uint32_t(wbest);
            const float dv = ordered_to_float(uint32_t(wbest >> 32));
            p.out_dist[orow * klist + t] = p.out_sqrt ? __fsqrt_rn(dv) : dv;
        }
    }
}

template <int METRIC, int KCAP>
static cudaError_t launch_exact_t(ExactParams p, uint32_t nchunks, cudaStream_t stream) {
    const size_t smem = sizeof(ExactSmem<KCAP>);
    auto kern = exact_fused_kernel<METRIC, KCAP>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    const dim3 grid((p.nslots + EX_BM - 1) / EX_BM, nchunks);
    kern<<<grid, EX_THREADS, smem, stream>>>(p);
    if ((e = cudaGetLastError()) != cudaSuccess || nchunks == 1) return e;
    exact_merge_kernel<<<(p.nslots + 7) / 8, 256, 0, stream>>>(p, nchunks);
    return cudaGetLastError();
}

template <int METRIC>
static cudaError_t launch_exact_m(ExactParams p, uint32_t nchunks, cudaStream_t stream) {
    if (p.klist <= 32) return launch_exact_t<METRIC, 32>(p, nchunks, stream);
    if (p.klist <= 64) return launch_exact_t<METRIC, 64>(p, nchunks, stream);
    if (p.klist <= 128) return launch_exact_t<METRIC, 128>(p, nchunks, stream);
    return launch_exact_t<METRIC, 256>(p, nchunks, stream);
}

// Column chunks for `nslots` rows: enough CTAs to cover every SM about twice
// (at most 256 chunks, each at least 4 column tiles wide).
static uint32_t exact_chunks(uint32_t nslots, uint32_t n, int sm_count) {
    const uint32_t rb = (nslots + EX_BM - 1) / EX_BM;
    uint32_t c = (2u * uint32_t(sm_count) + rb - 1) / rb;
    const uint32_t cmax = (n + 4 * EX_BN - 1) / (4 * EX_BN);
    if (c > cmax) c = cmax;
    if (c > 256) c = 256;
    return c < 1 ? 1 : c;
}

// Scratch for any launch of up to `max_slots` rows (the fallback row count is
// only known on the device).
size_t exact_scratch_bytes(uint32_t max_slots, uint32_t n, uint32_t klist, int sm_count) {
    size_t best = 0;
    const uint32_t rbs = (max_slots + EX_BM - 1) / EX_BM;
    for (uint32_t rb = 1; rb <= rbs; ++rb) {
        const uint32_t slots = rb * EX_BM < max_slots ? rb * EX_BM : max_slots;
        const uint32_t c = exact_chunks(slots, n, sm_count);
        if (c > 1) {
            const size_t b = size_t(c) * slots * klist * 8;
            if (b > best) best = b;
        }
        if (c == 1) break;  // more rows only shrink the chunk count
    }
    return best;
}

cudaError_t launch_exact_fused(int metric, const float* X, uint32_t n, uint32_t d, uint32_t klist,
                               const uint32_t* rows, uint32_t row_begin, uint32_t row_end,
                               uint32_t* out_index, float* out_dist, int out_sqrt, uint32_t scatter_base,
                               void* scratch, int sm_count, cudaStream_t stream) {
    if (row_end <= row_begin) return cudaSuccess;
    ExactParams p{X, n, d, klist, rows, row_begin, row_end - row_begin, n, out_index, out_dist, out_sqrt,
                  scatter_base, nullptr};
    const uint32_t nchunks = scratch ? exact_chunks(p.nslots, n, sm_count) : 1;
    if (nchunks > 1) {
        p.col_chunk = (n + nchunks - 1) / nchunks;
        p.partial = static_cast<uint64_t*>(scratch);
    }
    const uint32_t nch = nchunks > 1 ? (n + p.col_chunk - 1) / p.col_chunk : 1;
    // Hellinger arrives sqrt-staged and folds exactly like sqeuclidean.
    switch (metric) {
    case kCosine: return launch_exact_m<kCosine>(p, nch, stream);
    case kManhattan: return launch_exact_m<kManhattan>(p, nch, stream);
    case kRootSquares: return launch_exact_m<kRootSquares>(p, nch, stream);
    default: return launch_exact_m<kSqEuclidean>(p, nch, stream);
    }
}

}  // namespace knnb
