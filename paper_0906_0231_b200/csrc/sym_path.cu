// sym_path.cu -- symmetric TENSOR sweep: every tile serves both its rows and
// its columns (north_star (2), "symmetric distances reuse each tile for both
// rows"; the reference's k_smallest_push offers each tile entry to both
// endpoints, src/select.cpp:60-91).
//
// Geometry.  P blocks of 128 query rows (UMMA M), Q tiles of 256 columns
// (UMMA N); tile(i) = i / 256.  An unordered pair {i, j} with tile(i) <
// tile(j) is computed once, in the tile (block(i), tile(j)): the row side
// offers j to i's list, the column side offers i to j's list.  Pairs inside
// one tile are handled by a diagonal prepass with the row side only (both
// directions are rows there).
//
// Ownership without locks.
//   * Row-side lists (two 16-entry segments per row) live in the registers of
//     the CTA holding the row's block for its whole sweep.
//   * Column-side lists (one 16-entry list per row) live in global memory and
//     are loaded into shared memory for one visit of a tile.  The visitors of
//     tile q are the blocks p = 0 .. 2q-1; visitor p waits until the tile's
//     version counter reads p and bumps it when done, so visits are exclusive
//     and ordered.  Each CTA takes its blocks in increasing order
//     (boustrophedon waves, the reference's lane_of_row, schedule.cpp:40-44,
//     to balance the triangle), so the lowest unfinished visit is always
//     runnable: no deadlock.
//   * Column-side candidates found by the row-owning threads are queued per
//     column in shared memory and merged by one thread per column.
//   * A prepass sweeps each block's own tile (row side, self excluded) and
//     seeds the column-side list of every row with a copy of its row-side
//     top 16, so column-side thresholds start finite (the rescore drops the
//     duplicate copies; list maxima still bound their exclusions).
// Completeness: every column not in one of a row's three lists was rejected
// by a list whose maximum only decreases; the rescore's proof uses the
// smallest maximum over full lists.
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "common.cuh"
#include "kernels.h"
#include "sm100_ptx.cuh"
#include "sweep_common.cuh"

namespace knnb {

constexpr int SY_BM = 128;
constexpr int SY_BN = 256;
constexpr int SY_KPL = 16;
constexpr int SY_EW = 8;
constexpr int SY_THREADS = 64 + 32 * SY_EW;
constexpr int SY_QC = 12;    // shared queue entries per column
constexpr int SY_OVF = 128;  // global overflow entries per column (a block has 128 rows)
constexpr uint32_t SY_A_CHUNK = SY_BM * 128;
constexpr uint32_t SY_B_CHUNK = SY_BN * 128;
constexpr int SY_STAGES = 3;
constexpr uint32_t SY_A_BYTES = 4 * SY_A_CHUNK;  // d <= 256: the block's rows stay resident
constexpr uint32_t SY_CL_BYTES = SY_KPL * SY_BN * 8;          // column lists (y, idx) [16][256]
constexpr uint32_t SY_Q_BYTES = SY_QC * SY_BN * 8;            // queues (y, row) [QC][256]
constexpr uint32_t SY_SMEM = 1024 + SY_A_BYTES + SY_STAGES * SY_B_CHUNK + SY_CL_BYTES + 2 * SY_BN * 4 +
                             SY_Q_BYTES + SY_BN * 4 + 256;
static_assert(SY_SMEM <= 232448, "symmetric sweep shared memory");

struct SymParams {
    const uint8_t* xh;
    const float* alpha;
    uint32_t n, npad, kc;
    uint32_t nrb, ntiles;
    int diag;              // 1: prepass over each block's own tile
    uint64_t* cand;        // [nrb*128][48]: row-side segments at [0,32); column list copied to [32,48) later
    uint64_t* cstate;      // [ntiles*256][16] column-side lists
    uint32_t* version;     // [ntiles] completed visits
    uint64_t* overflow;    // [gridDim][256][SY_OVF]
    int dbg;               // dev timing knob (KNN_B200_SYM_DEBUG): 1 = no visit ordering (racy), 2 = no column side
};

__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release_u32(uint32_t* p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void epi_barrier() { asm volatile("bar.sync 1, 256;" ::: "memory"); }

// Block taken by CTA c in wave w (boustrophedon, schedule.cpp:40-44).
__device__ __forceinline__ uint32_t sym_block(uint32_t w, uint32_t c, uint32_t G) {
    return w * G + ((w & 1) ? G - 1 - c : c);
}

__global__ void __launch_bounds__(SY_THREADS, 1) tensor_sym_kernel(const SymParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* a_smem = smem;
    uint8_t* stage_smem = smem + SY_A_BYTES;
    float* cl_a = reinterpret_cast<float*>(stage_smem + SY_STAGES * SY_B_CHUNK);  // [16][256]
    uint32_t* cl_i = reinterpret_cast<uint32_t*>(cl_a + SY_KPL * SY_BN);           // [16][256]
    float* thr_c = reinterpret_cast<float*>(cl_i + SY_KPL * SY_BN);                // [256]
    float* thr_p = thr_c + SY_BN;                                                   // [256] prefilter
    float* q_y = thr_p + SY_BN;                                                     // [QC][256]
    uint32_t* q_r = reinterpret_cast<uint32_t*>(q_y + SY_QC * SY_BN);              // [QC][256]
    uint32_t* q_n = q_r + SY_QC * SY_BN;                                            // [256]
    uint64_t* bars = reinterpret_cast<uint64_t*>(q_n + SY_BN);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * SY_STAGES + 6);
    constexpr int S = SY_STAGES;

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t G = gridDim.x, c = blockIdx.x;
    const uint32_t waves = (p.nrb + G - 1) / G;
    const uint32_t bar0 = ptx::smem_u32(bars);
    auto full_bar = [&](int s) { return bar0 + 8u * s; };
    auto empty_bar = [&](int s) { return bar0 + 8u * (S + s); };
    auto tfull_bar = [&](int b) { return bar0 + 8u * (2 * S + b); };
    auto tempty_bar = [&](int b) { return bar0 + 8u * (2 * S + 2 + b); };
    const uint32_t afull_bar = bar0 + 8u * (2 * S + 4);
    const uint32_t aempty_bar = bar0 + 8u * (2 * S + 5);
    // tiles of block pb: the diagonal tile (prepass) or every tile above it
    auto tile_range = [&](uint32_t pb, uint32_t& q0, uint32_t& q1) {
        const uint32_t qd = pb / 2;
        if (p.diag) {
            q0 = qd;
            q1 = qd + 1;
        } else {
            q0 = qd + 1;
            q1 = p.ntiles > q0 ? p.ntiles : q0;
        }
    };

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < S; ++s) {
            ptx::mbar_init(full_bar(s), 1);
            ptx::mbar_init(empty_bar(s), 1);
        }
        for (int b = 0; b < 2; ++b) {
            ptx::mbar_init(tfull_bar(b), 1);
            ptx::mbar_init(tempty_bar(b), SY_EW);
        }
        ptx::mbar_init(afull_bar, 1);
        ptx::mbar_init(aempty_bar, 1);
        ptx::fence_mbar_init();
    }
    if (warp == 1) ptx::tmem_alloc(ptx::smem_u32(tmem_slot), 2 * SY_BN);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ---------------- TMA producer ----------------
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0, a_phase = 0;
            for (uint32_t w = 0; w < waves; ++w) {
                const uint32_t pb = sym_block(w, c, G);
                if (pb >= p.nrb) continue;
                uint32_t q0, q1;
                tile_range(pb, q0, q1);
                if (q0 >= q1) continue;
                ptx::mbar_wait(aempty_bar, a_phase ^ 1);
                ptx::mbar_arrive_expect_tx(afull_bar, p.kc * SY_A_CHUNK);
                for (uint32_t kc = 0; kc < p.kc; ++kc)
                    ptx::bulk_g2s(ptx::smem_u32(a_smem + kc * SY_A_CHUNK),
                                  p.xh + (size_t(kc) * p.npad + size_t(pb) * SY_BM) * 128, SY_A_CHUNK, afull_bar);
                a_phase ^= 1;
                for (uint32_t q = q0; q < q1; ++q)
                    for (uint32_t kc = 0; kc < p.kc; ++kc) {
                        ptx::mbar_wait(empty_bar(stage), phase ^ 1);
                        ptx::mbar_arrive_expect_tx(full_bar(stage), SY_B_CHUNK);
                        ptx::bulk_g2s(ptx::smem_u32(stage_smem + stage * SY_B_CHUNK),
                                      p.xh + (size_t(kc) * p.npad + size_t(q) * SY_BN) * 128, SY_B_CHUNK,
                                      full_bar(stage));
                        if (++stage == S) {
                            stage = 0;
                            phase ^= 1;
                        }
                    }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer ----------------
        if (lane == 0) {
            constexpr uint32_t idesc = ptx::idesc_f16_f32(SY_BM, SY_BN);
            int stage = 0;
            uint32_t phase = 0, a_phase = 0, tcount = 0;
            for (uint32_t w = 0; w < waves; ++w) {
                const uint32_t pb = sym_block(w, c, G);
                if (pb >= p.nrb) continue;
                uint32_t q0, q1;
                tile_range(pb, q0, q1);
                if (q0 >= q1) continue;
                ptx::mbar_wait(afull_bar, a_phase);
                a_phase ^= 1;
                for (uint32_t q = q0; q < q1; ++q, ++tcount) {
                    const uint32_t b = tcount & 1, use = tcount >> 1;
                    ptx::mbar_wait(tempty_bar(b), (use & 1) ^ 1);
                    ptx::tc_fence_after();
                    const uint32_t d_tmem = tmem + b * SY_BN;
                    for (uint32_t kc = 0; kc < p.kc; ++kc) {
                        ptx::mbar_wait(full_bar(stage), phase);
                        ptx::tc_fence_after();
                        const uint32_t a_addr = ptx::smem_u32(a_smem + kc * SY_A_CHUNK);
                        const uint32_t b_addr = ptx::smem_u32(stage_smem + stage * SY_B_CHUNK);
#pragma unroll
                        for (uint32_t k = 0; k < 4; ++k)
                            ptx::mma_f16_ss(d_tmem, ptx::sw128_kmajor_desc(a_addr + 32 * k),
                                            ptx::sw128_kmajor_desc(b_addr + 32 * k), idesc, (kc | k) != 0);
                        ptx::mma_commit(empty_bar(stage));
                        if (++stage == S) {
                            stage = 0;
                            phase ^= 1;
                        }
                    }
                    ptx::mma_commit(tfull_bar(b));
                }
                ptx::mma_commit(aempty_bar);
            }
        }
    } else {
        // ---------------- epilogue: 8 warps, thread = (row of the block, column half) ----------------
        const int ew = warp - 2;
        const int quad = warp & 3;
        const int seg = ew / 4;
        const int rl = quad * 32 + lane;
        const uint32_t et = uint32_t(ew) * 32 + lane;  // 0..255: column owner in flushes
        const float kInf = __int_as_float(0x7f800000);
        const uint32_t lane_addr = tmem + (uint32_t(quad * 32) << 16);
        const uint32_t seg0 = seg * (SY_BN / 2);
        uint64_t* ovf = p.overflow + size_t(c) * SY_BN * SY_OVF;
        float la[SY_KPL];
        uint32_t lx[SY_KPL];
        ListMax thr{kInf, 0};
        auto reg_argmax = [&]() -> ListMax {
            float mv[8];
            uint32_t ms[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const bool r = la[2 * i + 1] > la[2 * i];
                mv[i] = r ? la[2 * i + 1] : la[2 * i];
                ms[i] = r ? 2 * i + 1 : 2 * i;
            }
#pragma unroll
            for (int w2 = 4; w2 >= 1; w2 >>= 1)
#pragma unroll
                for (int i = 0; i < w2; ++i) {
                    const bool r = mv[i + w2] > mv[i];
                    mv[i] = r ? mv[i + w2] : mv[i];
                    ms[i] = r ? ms[i + w2] : ms[i];
                }
            return ListMax{mv[0], ms[0]};
        };
        auto insert_row = [&](float y, uint32_t col) {
#pragma unroll
            for (int s = 0; s < SY_KPL; ++s) {
                const bool h = uint32_t(s) == thr.slot;
                la[s] = h ? y : la[s];
                lx[s] = h ? col : lx[s];
            }
            thr = reg_argmax();
        };
        auto load_vec32 = [&](const float* src, float (&bt)[32]) {
            const float4* s4 = reinterpret_cast<const float4*>(src);
#pragma unroll
            for (int q4 = 0; q4 < 8; ++q4) {
                const float4 f = s4[q4];
                bt[4 * q4] = f.x;
                bt[4 * q4 + 1] = f.y;
                bt[4 * q4 + 2] = f.z;
                bt[4 * q4 + 3] = f.w;
            }
        };
        uint32_t tcount = 0;
        for (uint32_t w = 0; w < waves; ++w) {
            const uint32_t pb = sym_block(w, c, G);
            if (pb >= p.nrb) continue;
            uint32_t q0, q1;
            tile_range(pb, q0, q1);
            const uint32_t row = pb * SY_BM + rl;
            const bool valid = row < p.n;
            uint64_t* rstate = p.cand + size_t(row) * 48 + seg * SY_KPL;
#pragma unroll
            for (int s = 0; s < SY_KPL; ++s) {
                const uint64_t key = (p.diag || !valid) ? kEmptyKey : rstate[s];
                la[s] = key == kEmptyKey ? kInf : ordered_to_float(uint32_t(key >> 32));
                lx[s] = uint32_t(key);
            }
            thr = reg_argmax();
            if (!valid) thr.a = -kInf;
            const float alpha_i = valid ? p.alpha[row] : kInf;
            // column-side prefilter: fl(-2 dot - thrP_j) < -alpha_i (1 - 1e-6),
            // thrP_j = thrC_j + 1e-6 (|thrC_j| + alpha_j), is a superset of
            // fl(alpha_i - 2 dot) < thrC_j: y' >= -alpha_j bounds |y'| and the
            // slack covers both roundings (2^-24 each) many times over.
            const float c_lim = valid ? __fmul_rn(-alpha_i, 1.0f - 1e-6f) : -kInf;
            for (uint32_t q = q0; q < q1; ++q, ++tcount) {
                const uint32_t b = tcount & 1, use = tcount >> 1;
                const bool sym = !p.diag && p.dbg != 2;
                if (sym) {
                    // exclusive, ordered visit of tile q (visitors 0 .. 2q-1)
                    if (et == 0 && p.dbg != 1) {
                        uint32_t spins = 0;
                        while (ld_acquire_u32(p.version + q) != pb) {
                            __nanosleep(64);
                            if (++spins == (1u << 27)) __trap();  // ordering bug: fail, do not hang
                        }
                    }
                    epi_barrier();
                    const uint32_t crow = q * SY_BN + et;
                    const uint64_t* cs = p.cstate + size_t(crow) * SY_KPL;
                    float cm = -kInf;
#pragma unroll
                    for (int s = 0; s < SY_KPL; ++s) {
                        const uint64_t key = __ldcg(reinterpret_cast<const unsigned long long*>(cs + s));
                        const float a = key == kEmptyKey ? kInf : ordered_to_float(uint32_t(key >> 32));
                        cl_a[s * SY_BN + et] = a;
                        cl_i[s * SY_BN + et] = uint32_t(key);
                        cm = fmaxf(cm, a);
                    }
                    const bool live = crow < p.n;
                    thr_c[et] = live ? cm : -kInf;
                    thr_p[et] = !live ? -kInf
                                : cm == kInf ? kInf
                                             : __fadd_rn(cm, 1e-6f * __fadd_rn(fabsf(cm), p.alpha[crow]));
                    q_n[et] = 0;
                    epi_barrier();
                }
                ptx::mbar_wait(tfull_bar(b), use & 1);
                ptx::tc_fence_after();
                const uint32_t cbase = q * SY_BN + seg0;
                const uint32_t taddr = lane_addr + b * SY_BN + seg0;
                auto process = [&](const uint32_t (&v)[32], const float (&bt)[32], uint32_t col0, uint32_t cloc) {
                    // row side: y = fl(beta_j - 2 dot)
                    float m[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        const float2 y2 = ptx::ffma2_m2(v[2 * i], v[2 * i + 1], bt[2 * i], bt[2 * i + 1]);
                        m[i] = fminf(y2.x, y2.y);
                    }
#pragma unroll
                    for (int w2 = 8; w2 >= 1; w2 >>= 1)
#pragma unroll
                        for (int i = 0; i < w2; ++i) m[i] = fminf(m[i], m[i + w2]);
                    if (__any_sync(0xffffffffu, m[0] < thr.a)) {
                        uint32_t pm = 0;
#pragma unroll
                        for (int i = 0; i < 16; ++i) {
                            const float2 y2 = ptx::ffma2_m2(v[2 * i], v[2 * i + 1], bt[2 * i], bt[2 * i + 1]);
                            if (fminf(y2.x, y2.y) < thr.a) pm |= 1u << i;
                        }
                        uint32_t any = __reduce_or_sync(0xffffffffu, pm);
                        while (any) {
                            const int i = __ffs(any) - 1;
                            any &= any - 1;
                            if ((pm >> i) & 1u) {
                                const uint32_t col = col0 + 2 * i;
                                const float2 b2 = *reinterpret_cast<const float2*>(p.alpha + col);
                                uint32_t v0 = v[0], v1 = v[1];
#pragma unroll
                                for (int t2 = 1; t2 < 16; ++t2)
                                    if (t2 == i) {
                                        v0 = v[2 * t2];
                                        v1 = v[2 * t2 + 1];
                                    }
                                const float2 y2 = ptx::ffma2_m2(v0, v1, b2.x, b2.y);
                                if (y2.x < thr.a && col < p.n && col != row) insert_row(y2.x, col);
                                if (y2.y < thr.a && col + 1 < p.n && col + 1 != row) insert_row(y2.y, col + 1);
                            }
                        }
                    }
                    if (!sym) return;
                    // column side: candidate row i for column j's list, y' = fl(alpha_i - 2 dot)
                    float tc[32];
                    load_vec32(thr_p + cloc, tc);
                    float zm[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        const float2 z2 = ptx::ffma2_m2(v[2 * i], v[2 * i + 1], -tc[2 * i], -tc[2 * i + 1]);
                        zm[i] = fminf(z2.x, z2.y);
                    }
#pragma unroll
                    for (int w2 = 8; w2 >= 1; w2 >>= 1)
#pragma unroll
                        for (int i = 0; i < w2; ++i) zm[i] = fminf(zm[i], zm[i + w2]);
                    const bool ccand = zm[0] < c_lim;
                    if (__any_sync(0xffffffffu, ccand)) {
                        uint32_t pm = 0;
                        if (ccand) {
#pragma unroll
                            for (int i = 0; i < 16; ++i) {
                                const float2 z2 =
                                    ptx::ffma2_m2(v[2 * i], v[2 * i + 1], -tc[2 * i], -tc[2 * i + 1]);
                                if (fminf(z2.x, z2.y) < c_lim) pm |= 1u << i;
                            }
                        }
                        while (pm) {  // per-lane: queue pushes need no warp convergence
                            const int i = __ffs(pm) - 1;
                            pm &= pm - 1;
                            uint32_t v0 = v[0], v1 = v[1];
#pragma unroll
                            for (int t2 = 1; t2 < 16; ++t2)
                                if (t2 == i) {
                                    v0 = v[2 * t2];
                                    v1 = v[2 * t2 + 1];
                                }
                            const float2 y2 = ptx::ffma2_m2(v0, v1, alpha_i, alpha_i);
#pragma unroll
                            for (int e = 0; e < 2; ++e) {
                                const uint32_t jl = cloc + 2 * i + e;  // tile-local column
                                const float yv = e ? y2.y : y2.x;
                                if (yv < thr_c[jl]) {
                                    uint32_t at;
                                    asm volatile("atom.shared.add.u32 %0, [%1], 1;"
                                                 : "=r"(at)
                                                 : "r"(ptx::smem_u32(q_n + jl))
                                                 : "memory");
                                    if (at < uint32_t(SY_QC)) {
                                        q_y[at * SY_BN + jl] = yv;
                                        q_r[at * SY_BN + jl] = row;
                                    } else if (at < uint32_t(SY_QC + SY_OVF)) {
                                        ovf[size_t(jl) * SY_OVF + (at - SY_QC)] =
                                            (uint64_t(__float_as_uint(yv)) << 32) | row;
                                    }
                                }
                            }
                        }
                    }
                };
                uint32_t va[32], vb[32];
                float ba[32], bb[32];
                ptx::tmem_ld_32x32b_x32(taddr, va);
                load_vec32(p.alpha + cbase, ba);
#pragma unroll 1
                for (int c0 = 0; c0 < SY_BN / 2; c0 += 64) {
                    ptx::tmem_wait_ld();
                    ptx::tmem_ld_32x32b_x32(taddr + c0 + 32, vb);
                    load_vec32(p.alpha + cbase + c0 + 32, bb);
                    process(va, ba, cbase + c0, seg0 + c0);
                    ptx::tmem_wait_ld();
                    if (c0 + 64 < SY_BN / 2) {
                        ptx::tmem_ld_32x32b_x32(taddr + c0 + 64, va);
                        load_vec32(p.alpha + cbase + c0 + 64, ba);
                    } else {
                        ptx::tc_fence_before();
                        __syncwarp();
                        if (lane == 0) ptx::mbar_arrive(tempty_bar(b));
                    }
                    process(vb, bb, cbase + c0 + 32, seg0 + c0 + 32);
                }
                if (sym) {
                    epi_barrier();
                    // flush: thread et owns column et of the tile (row crow's list)
                    const uint32_t crow = q * SY_BN + et;
                    if (crow < p.n) {
                        const uint32_t a_base = ptx::smem_u32(cl_a + et), i_base = ptx::smem_u32(cl_i + et);
                        ListMax cmx = list_rescan<SY_KPL, SY_BN * 4>(a_base);
                        const uint32_t nq = min(q_n[et], uint32_t(SY_QC + SY_OVF));
                        for (uint32_t e = 0; e < nq; ++e) {
                            float yv;
                            uint32_t r;
                            if (e < uint32_t(SY_QC)) {
                                yv = q_y[e * SY_BN + et];
                                r = q_r[e * SY_BN + et];
                            } else {
                                const uint64_t k = ovf[size_t(et) * SY_OVF + (e - SY_QC)];
                                yv = __uint_as_float(uint32_t(k >> 32));
                                r = uint32_t(k);
                            }
                            if (yv < cmx.a) cmx = list_replace_max<SY_KPL, SY_BN * 4>(a_base, i_base, cmx.slot, yv, r);
                        }
                        uint64_t* cs = p.cstate + size_t(crow) * SY_KPL;
#pragma unroll
                        for (int s = 0; s < SY_KPL; ++s) {
                            const uint32_t ci = cl_i[s * SY_BN + et];
                            cs[s] = ci == 0xffffffffu ? kEmptyKey
                                                      : (uint64_t(float_to_ordered(cl_a[s * SY_BN + et])) << 32) | ci;
                        }
                    }
                    epi_barrier();
                    if (et == 0) {
                        __threadfence();
                        st_release_u32(p.version + q, pb + 1);
                    }
                }
            }
            if (valid) {
#pragma unroll
                for (int s = 0; s < SY_KPL; ++s)
                    rstate[s] = lx[s] == 0xffffffffu ? kEmptyKey : (uint64_t(float_to_ordered(la[s])) << 32) | lx[s];
            }
            if (p.diag) {
                // seed the row's column-side list with its row-side top 16
                // (both halves of the row meet in shared memory)
                float* sa = cl_a;        // [2][16][128] scratch
                uint32_t* si = cl_i;
#pragma unroll
                for (int s = 0; s < SY_KPL; ++s) {
                    sa[(seg * SY_KPL + s) * SY_BM + rl] = la[s];
                    si[(seg * SY_KPL + s) * SY_BM + rl] = lx[s];
                }
                epi_barrier();
                if (seg == 0 && valid) {
                    float va2[2 * SY_KPL];
                    uint32_t vi2[2 * SY_KPL];
#pragma unroll
                    for (int s = 0; s < 2 * SY_KPL; ++s) {
                        va2[s] = sa[s * SY_BM + rl];
                        vi2[s] = si[s * SY_BM + rl];
                    }
                    uint64_t* cs = p.cstate + size_t(row) * SY_KPL;
                    // 16 smallest of 32 (repeated minimum extraction)
                    for (int s = 0; s < SY_KPL; ++s) {
                        float bv = va2[0];
                        uint32_t bi = vi2[0];
                        int best = 0;
#pragma unroll
                        for (int t2 = 1; t2 < 2 * SY_KPL; ++t2) {
                            const bool lt = va2[t2] < bv || (va2[t2] == bv && vi2[t2] < bi);
                            bv = lt ? va2[t2] : bv;
                            bi = lt ? vi2[t2] : bi;
                            best = lt ? t2 : best;
                        }
#pragma unroll
                        for (int t2 = 0; t2 < 2 * SY_KPL; ++t2) {
                            va2[t2] = t2 == best ? kInf : va2[t2];
                            vi2[t2] = t2 == best ? 0xfffffffeu : vi2[t2];
                        }
                        cs[s] = bi >= 0xfffffffeu ? kEmptyKey : (uint64_t(float_to_ordered(bv)) << 32) | bi;
                    }
                }
                epi_barrier();
            }
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem, 2 * SY_BN);
    }
}

// cand[row][32..48) = the row's column-side list
__global__ void sym_concat_kernel(uint64_t* cand, const uint64_t* cstate, uint32_t n) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n * SY_KPL) return;
    const uint32_t row = i / SY_KPL, s = i % SY_KPL;
    cand[size_t(row) * 48 + 32 + s] = cstate[size_t(row) * SY_KPL + s];
}

size_t sym_workspace_bytes(uint32_t n, int sm_count) {
    const uint32_t ntiles = (n + SY_BN - 1) / SY_BN;
    size_t b = 0;
    auto add = [&](size_t x) { b += (x + 255) / 256 * 256; };
    add(size_t(ntiles) * SY_BN * SY_KPL * 8);        // cstate
    add(size_t(ntiles) * 4);                          // versions
    add(size_t(sm_count) * SY_BN * SY_OVF * 8);      // overflow queues
    return b;
}

cudaError_t run_sym_sweep(const uint8_t* xh, const float* alpha, uint32_t n, uint32_t npad, uint32_t kc,
                          uint64_t* cand, void* ws, int sm_count, cudaStream_t st) {
    const uint32_t ntiles = (n + SY_BN - 1) / SY_BN;
    const uint32_t nrb = (n + SY_BM - 1) / SY_BM;
    uint8_t* w = static_cast<uint8_t*>(ws);
    auto take = [&](size_t x) {
        uint8_t* q = w;
        w += (x + 255) / 256 * 256;
        return q;
    };
    uint64_t* cstate = reinterpret_cast<uint64_t*>(take(size_t(ntiles) * SY_BN * SY_KPL * 8));
    uint32_t* version = reinterpret_cast<uint32_t*>(take(size_t(ntiles) * 4));
    uint64_t* overflow = reinterpret_cast<uint64_t*>(take(size_t(sm_count) * SY_BN * SY_OVF * 8));
    cudaError_t e;
    if ((e = cudaFuncSetAttribute(tensor_sym_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(SY_SMEM))) !=
        cudaSuccess)
        return e;
    if ((e = cudaMemsetAsync(version, 0, size_t(ntiles) * 4, st)) != cudaSuccess) return e;
    const uint32_t grid = nrb < uint32_t(sm_count) ? nrb : uint32_t(sm_count);
    const char* dbg = getenv("KNN_B200_SYM_DEBUG");
    SymParams sp{xh, alpha, n, npad, kc, nrb, ntiles, 1, cand, cstate, version, overflow, dbg ? atoi(dbg) : 0};
    tensor_sym_kernel<<<grid, SY_THREADS, SY_SMEM, st>>>(sp);  // diagonal prepass
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    sp.diag = 0;
    // every CTA spins on other CTAs' visits: all must be resident (one per SM)
    void* args[] = {&sp};
    if ((e = cudaLaunchCooperativeKernel(reinterpret_cast<void*>(tensor_sym_kernel), dim3(grid), dim3(SY_THREADS),
                                         args, SY_SMEM, st)) != cudaSuccess)
        return e;
    sym_concat_kernel<<<(n * SY_KPL + 255) / 256, 256, 0, st>>>(cand, cstate, n);
    return cudaGetLastError();
}

}  // namespace knnb
