// sym_path.cu -- symmetric TENSOR sweep: every tile serves both its rows and
// its columns (north_star (2), "symmetric distances reuse each tile for both
// rows"; the reference's k_smallest_push offers each tile entry to both
// endpoints, src/select.cpp:60-91).
//
// Geometry.  nrb blocks of 128 query rows (UMMA M), T tiles of 256 columns
// (UMMA N); tile(i) = i / 256, so tile t holds blocks 2t and 2t+1.  The G
// persistent CTAs take the blocks in waves: wave w = blocks [wG, wG+Gw), CTA
// c holds block wG+c (G is even, so a wave's rows are whole tiles
// [t_lo, t_hi]).  Every unordered pair is covered once:
//   * prepass (diag launch): each block against its own tile, row side only,
//     self excluded -- both directions are rows there;
//   * band: each block against the other tiles of its own wave, row side
//     only (both directions again, since every block of the wave does it);
//   * rectangle: each block against every later tile (t > t_hi), both sides:
//     the row side offers column j to row i's lists, the column side offers
//     row i to row j's column-side list.
//
// Ownership.
//   * Row-side lists (two 16-entry segments per row, by column half) live in
//     registers of the CTA holding the block, for the whole wave.
//   * Column-side lists (one 16-entry list per row) live in global memory in
//     shared-memory layout ([tile][slot][256] y and index planes).  A visit
//     filters the tile's columns against published thresholds (a stale
//     threshold is an upper bound: lists only improve), queues candidates in
//     shared memory, and merges them into the tile's lists: a list-agent warp
//     bulk-loads the tile's y plane (double-buffered) once a per-tile version
//     counter says the previous visitor is done, the merging threads write
//     changed entries through to global memory, and the agent bumps the
//     version -- the visits of a tile are exclusive and in a fixed order.
//   * Rectangle steps are rotated (CTA r visits tile (s + 2r) mod L at step
//     s), so consecutive visitors of a tile are two steps apart: the agent's
//     version wait, list load and store overlap the sweep instead of forming a
//     lock-step chain; the 2G-tile window still fits in L2.  Late waves whose
//     rectangle is narrower than 2G tiles visit in plain order (rank = r).
// Deadlock freedom: releases wait only on the CTA's own merge, and a load
// waits only on the tile's previous visitor, which sits at a strictly earlier
// (wave, step) -- or, in plain order, a smaller rank.  Modelled for many n by
// tools/sym_schedule_check.py (tests/test_sym_schedule.py).
// Completeness: every column not in one of a row's three lists was rejected
// by (or evicted from) the list it was offered to, whose maximum only
// decreases; the rescore's proof uses the smallest maximum over full lists.
// The prepass seeds each column-side list with a copy of the row's top 16,
// so thresholds start finite; the rescore drops the duplicate copies.
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
constexpr int SY_AGENT_WARP = 2 + SY_EW;
constexpr int SY_THREADS = 64 + 32 * SY_EW + 32;
constexpr int SY_QC = 8;     // shared queue entries per column
// consecutive visitors of a rectangle tile are SY_SPREAD steps apart (the
// 148 x SY_SPREAD-tile window of fp16 tiles must stay L2-resident)
#ifndef SY_SPREAD
#define SY_SPREAD 2
#endif
constexpr int SY_OVF = 128;  // global overflow entries per column (a block has 128 rows)
constexpr uint32_t SY_A_CHUNK = SY_BM * 128;
constexpr uint32_t SY_B_CHUNK = SY_BN * 128;
constexpr int SY_STAGES = 3;
constexpr uint32_t SY_A_BYTES = 4 * SY_A_CHUNK;            // d <= 256: the block's rows stay resident
constexpr uint32_t SY_LIST_PLANE = SY_KPL * SY_BN * 4;     // one [16][256] y plane (double-buffered)
constexpr uint32_t SY_SMEM = 1024 + SY_A_BYTES + SY_STAGES * SY_B_CHUNK + 2 * SY_LIST_PLANE +
                             2 * SY_QC * SY_BN * 4 + 2 * SY_BN * 4 + 32 + 256;
static_assert(SY_SMEM <= 232448, "symmetric sweep shared memory");

struct SymParams {
    const uint8_t* xh;
    const float* alpha;
    uint32_t n, npad, kc;
    uint32_t nrb, ntiles;
    int diag;            // 1: prepass over each block's own tile
    uint64_t* cand;      // [nrb*128][48]: row-side segments at [0,32); column list copied to [32,48) later
    float* cla;          // [ntiles][16][256] column-side list y
    uint32_t* cli;       // [ntiles][16][256] column-side list index
    float* thr_pub;      // [ntiles*256] published column-side prefilter thresholds
    uint32_t* version;   // [ntiles] completed rectangle visits
    uint64_t* overflow;  // [gridDim][256][SY_OVF]
    const float* bmin;   // [npad / 32] smallest column norm per 32-column chunk
    int dbg;             // dev timing knob (KNN_B200_SYM_DEBUG): 2 = no column side, 3 = also no rotation (wrong results)
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

// One CTA's visits in one wave.
struct SymWave {
    uint32_t b, r, Gw, t_lo, t_hi, nband, L, base;
    bool rot, live;
    __device__ SymWave(const SymParams& p, uint32_t w, uint32_t c) {
        const uint32_t G = gridDim.x;
        Gw = p.nrb - w * G < G ? p.nrb - w * G : G;
        r = c;
        b = w * G + c;
        live = c < Gw;
        t_lo = (w * G) / 2;
        t_hi = (w * G + Gw - 1) / 2;
        nband = t_hi - t_lo;  // the wave's tiles except the block's own
        L = p.ntiles > t_hi + 1 ? p.ntiles - t_hi - 1 : 0;
        rot = SY_SPREAD * Gw <= L && p.dbg != 3;
        base = G * w;
    }
    __device__ uint32_t visits(int diag) const { return diag ? 1u : nband + L; }
    __device__ uint32_t tile(int diag, uint32_t j) const {
        if (diag) return b / 2;
        if (j < nband) {
            const uint32_t t = t_lo + j;
            return t >= b / 2 ? t + 1 : t;
        }
        const uint32_t s = j - nband;
        return t_hi + 1 + (rot ? (s + SY_SPREAD * r) % L : s);
    }
    // position of this CTA's visit among the wave's visits of rectangle tile t
    __device__ uint32_t rank(uint32_t t) const {
        if (!rot) return base + r;
        const uint32_t qq = t - t_hi - 1;
        const uint32_t c1 = qq / SY_SPREAD < Gw - 1 ? qq / SY_SPREAD : Gw - 1;
        return base + (r <= c1 ? c1 - r : c1 + 1 + (Gw - 1 - r));
    }
};

__global__ void __launch_bounds__(SY_THREADS, 1) tensor_sym_kernel(const SymParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* a_smem = smem;
    uint8_t* stage_smem = smem + SY_A_BYTES;
    float* cl_a = reinterpret_cast<float*>(stage_smem + SY_STAGES * SY_B_CHUNK);  // [2][16][256] y planes
    float* q_y = cl_a + 2 * SY_KPL * SY_BN;                                         // [QC][256]
    uint32_t* q_r = reinterpret_cast<uint32_t*>(q_y + SY_QC * SY_BN);              // [QC][256]
    float* thr_p = reinterpret_cast<float*>(q_r + SY_QC * SY_BN);                  // [256]
    uint32_t* q_n = reinterpret_cast<uint32_t*>(thr_p + SY_BN);                    // [256]
    float* chunk_thr = reinterpret_cast<float*>(q_n + SY_BN);                      // [8] per 32 columns
    uint64_t* bars = reinterpret_cast<uint64_t*>(chunk_thr + 8);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * SY_STAGES + 9);
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
    auto lfull_bar = [&](int b) { return bar0 + 8u * (2 * S + 6 + b); };  // column-list y plane loaded
    const uint32_t lmerged_bar = bar0 + 8u * (2 * S + 8);  // column lists merged (8 epilogue warps)

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
        ptx::mbar_init(lfull_bar(0), 1);
        ptx::mbar_init(lfull_bar(1), 1);
        ptx::mbar_init(lmerged_bar, SY_EW);
        ptx::fence_mbar_init();
    }
    if (warp == 1) ptx::tmem_alloc(ptx::smem_u32(tmem_slot), 2 * SY_BN);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const bool colside = !p.diag && p.dbg != 2 && p.dbg != 3;

    if (warp == 0) {
        // ---------------- TMA producer ----------------
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0, a_phase = 0;
            for (uint32_t w = 0; w < waves; ++w) {
                const SymWave sw(p, w, c);
                if (!sw.live) continue;
                const uint32_t nv = sw.visits(p.diag);
                if (nv == 0) continue;
                ptx::mbar_wait(aempty_bar, a_phase ^ 1);
                ptx::mbar_arrive_expect_tx(afull_bar, p.kc * SY_A_CHUNK);
                for (uint32_t kc = 0; kc < p.kc; ++kc)
                    ptx::bulk_g2s(ptx::smem_u32(a_smem + kc * SY_A_CHUNK),
                                  p.xh + (size_t(kc) * p.npad + size_t(sw.b) * SY_BM) * 128, SY_A_CHUNK, afull_bar);
                a_phase ^= 1;
                for (uint32_t j = 0; j < nv; ++j) {
                    const uint32_t q = sw.tile(p.diag, j);
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
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer ----------------
        if (lane == 0) {
            constexpr uint32_t idesc = ptx::idesc_f16_f32(SY_BM, SY_BN);
            int stage = 0;
            uint32_t phase = 0, a_phase = 0, tcount = 0;
            for (uint32_t w = 0; w < waves; ++w) {
                const SymWave sw(p, w, c);
                if (!sw.live) continue;
                const uint32_t nv = sw.visits(p.diag);
                if (nv == 0) continue;
                ptx::mbar_wait(afull_bar, a_phase);
                a_phase ^= 1;
                for (uint32_t j = 0; j < nv; ++j, ++tcount) {
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
    } else if (warp == SY_AGENT_WARP) {
        // ---------------- list agent: ordered, exclusive rectangle visits ----------------
        // Visit v's y plane is loaded into buffer v % 2 once the tile's
        // previous visitor has released it; visit v is released as soon as
        // the epilogue has merged it (the merging threads write changed
        // entries straight to global memory and fence).  Releases never wait
        // on other CTAs, so the waits-for graph follows (wave, step, rank)
        // strictly downwards: no deadlock.
        if (lane == 0 && colside) {
            uint32_t merged_phase = 0, vbase = 0;
            for (uint32_t w = 0; w < waves; ++w) {
                const SymWave sw(p, w, c);
                if (!sw.live || sw.L == 0) continue;
                uint32_t nload = 0, nrel = 0, spins = 0, nap = 32;
                uint32_t lt = sw.tile(0, sw.nband), lver = sw.rank(lt);  // next load
                uint32_t rt = lt, rver = lver;                               // next release
                while (nrel < sw.L) {
                    bool progressed = false;
                    if (nload < sw.L && nload < nrel + 2 && ld_acquire_u32(p.version + lt) == lver) {
                        ptx::fence_proxy_async_global();
                        const uint32_t v = vbase + nload;
                        ptx::mbar_arrive_expect_tx(lfull_bar(v & 1), SY_LIST_PLANE);
                        ptx::bulk_g2s(ptx::smem_u32(cl_a + (v & 1) * SY_KPL * SY_BN),
                                      p.cla + size_t(lt) * SY_KPL * SY_BN, SY_LIST_PLANE, lfull_bar(v & 1));
                        if (++nload < sw.L) {
                            lt = sw.tile(0, sw.nband + nload);
                            lver = sw.rank(lt);
                        }
                        progressed = true;
                    }
                    if (nrel < nload && ptx::mbar_test(lmerged_bar, merged_phase)) {
                        merged_phase ^= 1;
                        __threadfence();
                        st_release_u32(p.version + rt, rver + 1);
                        if (++nrel < sw.L) {
                            rt = sw.tile(0, sw.nband + nrel);
                            rver = sw.rank(rt);
                        }
                        progressed = true;
                    }
                    if (progressed) {
                        spins = 0;
                        nap = 32;
                    } else {
                        __nanosleep(nap);  // back off: this warp shares a scheduler with epilogue warps
                        nap = nap < 512 ? 2 * nap : 512;
                        if (++spins == (1u << 25)) __trap();  // ordering bug: fail, do not hang
                    }
                }
                vbase += sw.L;
            }
        }
    } else {
        // ---------------- epilogue: 8 warps, thread = (row of the block, column half) ----------------
        const int ew = warp - 2;
        const int quad = warp & 3;
        const int seg = ew / 4;
        const int rl = quad * 32 + lane;
        const uint32_t et = uint32_t(ew) * 32 + lane;  // 0..255: column owner in merges
        const float kInf = __int_as_float(0x7f800000);
        const uint32_t lane_addr = tmem + (uint32_t(quad * 32) << 16);
        const uint32_t seg0 = seg * (SY_BN / 2);
        uint64_t* ovf = p.overflow + size_t(c) * SY_BN * SY_OVF;
        float la[SY_KPL];
        uint32_t lx[SY_KPL];
        ListMax thr{kInf, 0};
        uint32_t vcount = 0;  // rectangle visits so far (list buffer and phase)
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
        // prefetched published threshold of this thread's column in the next rectangle visit
        auto thr_fetch = [&](uint32_t t) -> float {
            const uint32_t crow = t * SY_BN + et;
            return crow < p.n ? __ldcg(p.thr_pub + crow) : -kInf;
        };
        uint32_t tcount = 0;
        for (uint32_t w = 0; w < waves; ++w) {
            const SymWave sw(p, w, c);
            if (!sw.live) continue;
            const uint32_t nv = sw.visits(p.diag);
            const uint32_t row = sw.b * SY_BM + rl;
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
            float thr_next = (colside && sw.L) ? thr_fetch(sw.tile(0, sw.nband)) : -kInf;
            for (uint32_t j = 0; j < nv; ++j, ++tcount) {
                const uint32_t q = sw.tile(p.diag, j);
                const uint32_t b = tcount & 1, use = tcount >> 1;
                const bool sym = colside && j >= sw.nband;
                if (sym) {
                    thr_p[et] = thr_next;
                    q_n[et] = 0;
                    float cm = thr_next;  // this warp's 32 columns: the column-side chunk bound
                    for (int o = 16; o; o >>= 1) cm = fmaxf(cm, __shfl_xor_sync(0xffffffffu, cm, o));
                    if (lane == 0) chunk_thr[et >> 5] = cm;
                    epi_barrier();
                    if (j + 1 < nv) thr_next = thr_fetch(sw.tile(0, j + 1));
                }
                ptx::mbar_wait(tfull_bar(b), use & 1);
                ptx::tc_fence_after();
                const uint32_t cbase = q * SY_BN + seg0;
                const uint32_t taddr = lane_addr + b * SY_BN + seg0;
                // One 32-column chunk (col0: global column, cloc: tile-local).
                // Hot path, both sides on the raw dots and one max tree:
                //   row side    y  = fl(beta_j - 2 dot) < thr_i    needs dot > (bmin_chunk - thr_i) / 2;
                //   column side y' = fl(alpha_i - 2 dot) < thrP_j  needs dot > (alpha_i - max_chunk thrP) / 2.
                // Both bounds get a 2^-20 slack (rounding of y at y ~ thr is
                // ~2^-24 |thr|), so they are supersets of the exact tests the
                // rare paths then apply.
                auto process = [&](const uint32_t (&v)[32], uint32_t col0, uint32_t cloc) {
                    float r1[11], r2[4];
#pragma unroll
                    for (int j2 = 0; j2 < 10; ++j2)
                        r1[j2] = fmaxf(fmaxf(__uint_as_float(v[3 * j2]), __uint_as_float(v[3 * j2 + 1])),
                                       __uint_as_float(v[3 * j2 + 2]));
                    r1[10] = fmaxf(__uint_as_float(v[30]), __uint_as_float(v[31]));
#pragma unroll
                    for (int j2 = 0; j2 < 3; ++j2) r2[j2] = fmaxf(fmaxf(r1[3 * j2], r1[3 * j2 + 1]), r1[3 * j2 + 2]);
                    r2[3] = fmaxf(r1[9], r1[10]);
                    const float dmax = fmaxf(fmaxf(fmaxf(r2[0], r2[1]), r2[2]), r2[3]);
                    const float bm = __ldg(p.bmin + (col0 >> 5));
                    float hr = __fmul_rn(__fsub_rn(bm, thr.a), 0.5f);
                    if (fabsf(hr) < kInf) hr = __fsub_rn(hr, 9.5367431640625e-07f * (fabsf(bm) + fabsf(thr.a)));
                    const bool fire_r = dmax > hr;
                    bool fire_c = false;
                    if (sym && valid) {
                        const float tcm = chunk_thr[cloc >> 5];
                        float hc = __fmul_rn(__fsub_rn(alpha_i, tcm), 0.5f);
                        if (fabsf(hc) < kInf) hc = __fsub_rn(hc, 9.5367431640625e-07f * (fabsf(alpha_i) + fabsf(tcm)));
                        fire_c = dmax > hc;
                    }
                    if (!__any_sync(0xffffffffu, fire_r || fire_c)) return;
                    if (__any_sync(0xffffffffu, fire_r)) {
                        // row side rare path: exact y, per-lane pair mask, warp-uniform walk
                        float bt[32];
                        load_vec32(p.alpha + col0, bt);
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
                    if (fire_c) {
                        // column side: exact prefilter per column, fl(-2 dot - thrP_j) <
                        // -alpha_i (1 - 1e-6) is a superset of fl(alpha_i - 2 dot) < thrP_j
                        // (y' >= -alpha_j bounds |y'|; the slack covers both roundings),
                        // then per-lane queue pushes (no convergence needed)
                        float tc[32];
                        load_vec32(thr_p + cloc, tc);
                        const float c_lim = __fmul_rn(-alpha_i, 1.0f - 1e-6f);
                        uint32_t pm = 0;
#pragma unroll
                        for (int i = 0; i < 16; ++i) {
                            const float2 z2 = ptx::ffma2_m2(v[2 * i], v[2 * i + 1], -tc[2 * i], -tc[2 * i + 1]);
                            if (fminf(z2.x, z2.y) < c_lim) pm |= 1u << i;
                        }
                        while (pm) {
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
                                if (yv < thr_p[jl]) {
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
                ptx::tmem_ld_32x32b_x32(taddr, va);
#pragma unroll 1
                for (int c0 = 0; c0 < SY_BN / 2; c0 += 64) {
                    ptx::tmem_wait_ld();
                    ptx::tmem_ld_32x32b_x32(taddr + c0 + 32, vb);
                    process(va, cbase + c0, seg0 + c0);
                    ptx::tmem_wait_ld();
                    if (c0 + 64 < SY_BN / 2) {
                        ptx::tmem_ld_32x32b_x32(taddr + c0 + 64, va);
                    } else {
                        ptx::tc_fence_before();
                        __syncwarp();
                        if (lane == 0) ptx::mbar_arrive(tempty_bar(b));
                    }
                    process(vb, cbase + c0 + 32, seg0 + c0 + 32);
                }
                if (sym) {
                    epi_barrier();  // every candidate queued
                    const uint32_t lb = vcount & 1;
                    ptx::mbar_wait(lfull_bar(lb), (vcount >> 1) & 1);
                    ++vcount;
                    // merge: thread et owns column et of the tile (row crow's list)
                    const uint32_t crow = q * SY_BN + et;
                    if (crow < p.n && q_n[et] != 0) {
                        const uint32_t a_base = ptx::smem_u32(cl_a + lb * SY_KPL * SY_BN + et);
                        float* ga = p.cla + size_t(q) * SY_KPL * SY_BN + et;
                        uint32_t* gi = p.cli + size_t(q) * SY_KPL * SY_BN + et;
                        ListMax cmx = list_rescan<SY_KPL, SY_BN * 4>(a_base);
                        bool wrote = false;
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
                            if (yv < cmx.a) {
                                sts_f32(a_base + cmx.slot * (SY_BN * 4), yv);
                                ga[cmx.slot * SY_BN] = yv;
                                gi[cmx.slot * SY_BN] = r;
                                wrote = true;
                                cmx = list_rescan<SY_KPL, SY_BN * 4>(a_base);
                            }
                        }
                        if (wrote) __threadfence();  // changed entries before the agent's release
                        if (nq)
                            p.thr_pub[crow] = cmx.a == kInf ? kInf
                                                            : __fadd_rn(cmx.a, 1e-6f * __fadd_rn(fabsf(cmx.a),
                                                                                                 p.alpha[crow]));
                    }
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive(lmerged_bar);
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
                float* sa = cl_a;  // [2][16][128] scratch
                uint32_t* si = reinterpret_cast<uint32_t*>(cl_a + SY_KPL * SY_BN);
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
                    const uint32_t t = row / SY_BN, pos = row % SY_BN;
                    float* ga = p.cla + size_t(t) * SY_KPL * SY_BN + pos;
                    uint32_t* gi = p.cli + size_t(t) * SY_KPL * SY_BN + pos;
                    float mx = -kInf;
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
                        const bool empty = bi >= 0xfffffffeu;
                        ga[s * SY_BN] = empty ? kInf : bv;
                        gi[s * SY_BN] = empty ? 0xffffffffu : bi;
                        mx = fmaxf(mx, empty ? kInf : bv);
                    }
                    p.thr_pub[row] = mx == kInf ? kInf : __fadd_rn(mx, 1e-6f * __fadd_rn(fabsf(mx), p.alpha[row]));
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
__global__ void sym_concat_kernel(uint64_t* cand, const float* cla, const uint32_t* cli, uint32_t n) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n * SY_KPL) return;
    const uint32_t row = i / SY_KPL, s = i % SY_KPL;
    const size_t at = size_t(row / SY_BN) * SY_KPL * SY_BN + size_t(s) * SY_BN + row % SY_BN;
    const uint32_t ci = cli[at];
    cand[size_t(row) * 48 + 32 + s] = ci == 0xffffffffu ? kEmptyKey : make_key(cla[at], ci);
}

size_t sym_workspace_bytes(uint32_t n, int sm_count) {
    const uint32_t ntiles = (n + SY_BN - 1) / SY_BN;
    size_t b = 0;
    auto add = [&](size_t x) { b += (x + 255) / 256 * 256; };
    add(size_t(ntiles) * SY_BN * SY_KPL * 4);     // cla
    add(size_t(ntiles) * SY_BN * SY_KPL * 4);     // cli
    add(size_t(ntiles) * SY_BN * 4);              // thr_pub
    add(size_t(ntiles) * 4);                      // versions
    add(size_t(sm_count) * SY_BN * SY_OVF * 8);  // overflow queues
    return b;
}

cudaError_t run_sym_sweep(const uint8_t* xh, const float* alpha, const float* bmin, uint32_t n, uint32_t npad,
                          uint32_t kc, uint64_t* cand, void* ws, int sm_count, cudaStream_t st) {
    const uint32_t ntiles = (n + SY_BN - 1) / SY_BN;
    const uint32_t nrb = (n + SY_BM - 1) / SY_BM;
    uint8_t* w = static_cast<uint8_t*>(ws);
    auto take = [&](size_t x) {
        uint8_t* q = w;
        w += (x + 255) / 256 * 256;
        return q;
    };
    float* cla = reinterpret_cast<float*>(take(size_t(ntiles) * SY_BN * SY_KPL * 4));
    uint32_t* cli = reinterpret_cast<uint32_t*>(take(size_t(ntiles) * SY_BN * SY_KPL * 4));
    float* thr_pub = reinterpret_cast<float*>(take(size_t(ntiles) * SY_BN * 4));
    uint32_t* version = reinterpret_cast<uint32_t*>(take(size_t(ntiles) * 4));
    uint64_t* overflow = reinterpret_cast<uint64_t*>(take(size_t(sm_count) * SY_BN * SY_OVF * 8));
    cudaError_t e;
    if ((e = cudaFuncSetAttribute(tensor_sym_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(SY_SMEM))) !=
        cudaSuccess)
        return e;
    if ((e = cudaMemsetAsync(version, 0, size_t(ntiles) * 4, st)) != cudaSuccess) return e;
    // persistent: one CTA per SM; an even count when there is more than one
    // wave, so every wave's rows are whole tiles
    uint32_t grid = nrb < uint32_t(sm_count) ? nrb : uint32_t(sm_count);
    if (grid < nrb) grid &= ~1u;
    const char* dbg = getenv("KNN_B200_SYM_DEBUG");
    SymParams sp{xh, alpha, n, npad, kc, nrb, ntiles, 1, cand, cla, cli, thr_pub, version, overflow, bmin,
                 dbg ? atoi(dbg) : 0};
    tensor_sym_kernel<<<grid, SY_THREADS, SY_SMEM, st>>>(sp);  // prepass: own tiles, seeds column lists
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    sp.diag = 0;
    // CTAs wait on each other's tile visits: all must be resident (one per SM)
    void* args[] = {&sp};
    if ((e = cudaLaunchCooperativeKernel(reinterpret_cast<void*>(tensor_sym_kernel), dim3(grid), dim3(SY_THREADS),
                                         args, SY_SMEM, st)) != cudaSuccess)
        return e;
    sym_concat_kernel<<<(n * SY_KPL + 255) / 256, 256, 0, st>>>(cand, cla, cli, n);
    return cudaGetLastError();
}

}  // namespace knnb
