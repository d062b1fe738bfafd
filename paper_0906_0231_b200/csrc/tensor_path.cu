// tensor_path.cu -- TENSOR policy: tcgen05 FP16 filter + exact FP32 re-score.
//
// The reference (src/dist_kernel.cpp:42-115 + src/select.cpp:60-130) computes
// every pair with the exact fold and funnels it into per-row heaps.  Here the
// n x n work runs on the 5th-generation tensor cores instead:
//
//   prep     x^_i = fp16_rn(s * (x_i - mu))   (mu = column mean, s = 2^e so
//            |x^| <= 65504), stored as 128-byte-swizzled K-major planes
//            [ceil(d/64)][npad][64] with the columns sorted by norm;
//            alpha_i = ||x^_i||^2 (fp32); and, in fp64, the exact quantisation
//            error rho_i = ||x^_i - s (x_i - mu)|| and ||x^_i|| for the error
//            bound.  (cosine: mu = 0, alpha = s^2, input order.)
//   sweep    persistent tcgen05 kernel (CTA pairs, M = 256, when d <= 256):
//            TMA bulk copies -> smem ring -> tcgen05.mma kind::f16 (FP32
//            accumulators in TMEM, double-buffered) -> epilogue warps, one
//            thread per (query row, column half), ranking y = beta_j - 2 dot
//            in per-row lists after a per-chunk bound test on the raw dots.
//            The n x n matrix never leaves the SM.  For large whole problems
//            the triangle sweep computes each unordered pair once (row side
//            into the lists, column side into fixed-threshold append logs).
//   rescore  per row: the exact reference fold (FSUB/FMUL/FADD, coordinates in
//            order) on the best candidates, the top-k by (distance, index), and
//            a proof that nothing outside the candidates can belong to the
//            top-k: A_max > s^2 T' + 2E, with T the exact k-th distance and E
//            a rigorous bound on |A - s^2 D_ref|.  Rows without
//            a proof take a band-capture second sweep, and the few whose band
//            overflows are recomputed by the EXACT kernel.
// Result: bit-identical to brute_force_knn.
#include <cub/device/device_radix_sort.cuh>
#include <algorithm>
#include <cstdio>
#include <type_traits>
#include <cuda_fp16.h>
#include <cuda_fp8.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "common.cuh"
#include "kernels.h"
#include "sm100_ptx.cuh"
#include "sweep_common.cuh"

namespace knnb {

constexpr int TS_BM = 128;
// A list slot holding only a bound: (threshold, kVirtualIdx).  The triangle
// sweep seeds its row-side lists with the sample pass's threshold this way:
// every column offered later and rejected has y >= the list maximum, so the
// maximum stays a valid bound, and far fewer columns get inserted.
constexpr uint32_t kVirtualIdx = 0xfffffffeu;
constexpr uint32_t TS_A_CHUNK = TS_BM * 128;  // 128 rows x 128 B (64 fp16 of K)
constexpr uint32_t TS_SMEM_MAX = 232448;
constexpr int TS_MAX_RES_KC = 4;              // A resident in smem when d <= 256
constexpr int kTriCap = 256;   // triangle mode: column-side buffer entries per row
constexpr int kTriRank = 4;    // its threshold: the 4th smallest y over the row's sample columns
constexpr int kTriSampleKpl = 4;  // sample lists: two of 4 per row hold the 4 smallest of the sample (6: +1 ms at C2)
constexpr int kTriStride = 16; // sample: every 16th sorted column (C2: 0.6% of rows to the capture pass;
                               // measured against 12/6 (0.05%): step -5 ms, tools/_knobs.sh)
constexpr int kTriBucket = 1024;  // second order: thresholds sorted within 1024-column norm buckets
constexpr int kLogChunk = 1024;   // column-side pool: entries per chunk

// EW epilogue warps (4 or 8).  With 8, two warps share each TMEM lane
// quadrant and split every tile's columns in halves; each half keeps its own
// list of KPL entries per row (NSEG = 2 list segments per row).
// PAIR: a cluster of two CTAs runs M = 256 tcgen05.mma (cta_group::2); each
// CTA stages its own 128 query rows and half of every reference tile, which
// halves the L2->SM operand traffic per CTA.
template <int KPL, int BN, bool ARES, int EW, bool PAIR = false>
struct TSLayout {
    static constexpr int NSEG = EW / 4;
    static constexpr int THREADS = 64 + 32 * EW;  // warp 0 TMA producer, warp 1 MMA issuer, epilogue warps
    static constexpr uint32_t B_CHUNK = (PAIR ? BN / 2 : BN) * 128;
    static constexpr uint32_t STAGE = B_CHUNK + (ARES ? 0 : TS_A_CHUNK);
    static constexpr uint32_t A_BYTES = ARES ? TS_MAX_RES_KC * TS_A_CHUNK : 0;
    static constexpr uint32_t LIST_ROWS = TS_BM * NSEG;                 // list "columns"
    static constexpr bool REGLIST = KPL <= 16;  // lists in registers, no shared-memory list arrays
    static constexpr uint32_t LISTS = REGLIST ? 0 : LIST_ROWS * KPL * 8;
    static constexpr uint32_t MISC = 512;  // barriers, TMEM address, the unit queue
    static constexpr uint32_t AVAIL = TS_SMEM_MAX - 1024 - MISC - LISTS - A_BYTES;
    static constexpr int STAGES_RAW = int(AVAIL / STAGE);
#ifndef KNN_TS_STAGE_CAP
#define KNN_TS_STAGE_CAP 6
#endif
    // (PAIR stages are half-size: allow twice as many for the same bytes in flight)
    static constexpr int STAGE_CAP = PAIR ? 2 * KNN_TS_STAGE_CAP : KNN_TS_STAGE_CAP;
    static constexpr int STAGES = STAGES_RAW > STAGE_CAP ? STAGE_CAP : STAGES_RAW;
    static_assert(STAGES >= 2, "shared memory budget too small for a 2-stage ring");
    static constexpr uint32_t SMEM = 1024 + A_BYTES + STAGES * STAGE + LISTS + MISC;
    static constexpr uint32_t TMEM_COLS = 2 * BN;  // two accumulator buffers
    static constexpr uint32_t STRIDE = LIST_ROWS * 4;  // bytes between entries of one list
};

// The sweep's bound tests compare raw dots with h = (a - b) / 2 less a slack
// that covers the rounding of y = fl(beta - 2 dot) and of h itself.  h is
// formed as bound_half(a, 1) + bound_half(b, -1): each half rounded down by
// 2^-19 of its magnitude (infinities pass through) -- one FADD per chunk in
// the sweep, the halves precomputed per column chunk (chunk_min_kernel,
// chunk_max_kernel) and per row.  A smaller h admits a superset: exact.
__device__ __forceinline__ float bound_half(float x, float sign) {
    const float h = x * (0.5f * sign);
    return fabsf(x) <= 3.402823466e+38f ? h - 1.9073486328125e-06f * fabsf(x) : h;  // finite: less the slack
}

struct SweepParams {
    const uint8_t* xh;    // swizzled fp16 planes
    const float* alpha;   // [npad], +inf on padding rows
    uint32_t n, npad, kc;
    uint32_t row_begin, row_end;
    uint32_t group_tiles;  // column tiles per L2-resident column group
    int debug_mode;        // profiling only (KNN_B200_DEBUG_SWEEP): 1 = TMEM loads only, 2 = release only,
                           // 3 = no TMA loads, 4 = filter without insertions
    uint64_t* cand;       // [(row_end - row_begin) * NSEG * KPL], segment-major per row;
                          // also the list state carried between column groups
    const uint8_t* xa;    // A-operand (query) planes: xh itself, or the gathered rows of a second pass
    uint32_t npad_a;
    // band-capture pass (CAPTURE kernels): per query slot a fixed y threshold;
    // every column with y <= threshold is appended to the slot's buffer
    const float* cap_thr;
    uint32_t* cap_cnt;
    uint64_t* cap_buf;
    uint32_t cap;
    const float* bmin;  // [2 npad / 32] smallest column norm of every 32-column chunk, then its bound_half
    // triangle mode (TRI kernels): rows and columns are the same sorted set;
    // a row unit sweeps only tiles >= its own and also offers each of its rows
    // to the columns' fixed-threshold buffers (the column side)
    const float* tc;     // [npad] column-side threshold: a row enters column j's buffer iff y' < tc[j]
    const float* tcmax;  // [2 npad / 32] its maximum per 32-column chunk, then its bound_half(., -1)
    uint64_t* lkey;      // column-side candidates: key (y', row) and column, in a pool of
    uint32_t* lcol;      //   kLogChunk-entry chunks; each epilogue warp fills its own chunk and
    uint32_t* lcnt;      //   takes the next free one (one atomic on *lnext) when it is full;
    uint32_t* lnext;     //   lcnt[c] = entries in chunk c (tri_scatter_kernel bins them by column)
    uint32_t nchunks;    // pool size; *lnext > nchunks = overflow (the host redoes the call)
    // E4M3 operands (kind::f8f6f4, PAIR kernels; the triangle's sample pass):
    // xh/xa hold E4M3 planes, kc counts 128-element chunks
    int e4m3;
    // Sharded triangle (TRI): this rank's 256-row units, in the order the
    // persistent CTA pairs take them (pair p: units[p], units[p + pairs], ...);
    // row-side lists are stored per local unit (cand row = lu * 256 + r).
    // Null: every unit 0, 1, ... of [row_begin, row_end).
    const uint32_t* units;
    uint32_t nunits;
    unsigned long long* cta_ns;  // profiling only (KNN_B200_DEBUG_CTA_TIMES): per CTA [start, end] globaltimer
    // Dynamic unit queue (TRI; null: the static walk above).  Work items
    // (local unit lu, column group g) are claimed from qctr[g]; units must be
    // ascending (a group's units with work are then a prefix).  udone[lu]
    // counts the epilogue warps that saved the unit's list state, so the pair
    // taking (lu, g + 1) waits for the one that ran (lu, g).  Zeroed per launch.
    uint32_t* qctr;
    uint32_t* udone;
};

// Candidate keys from the norm-sorted sweep carry sweep-order column indices;
// map them to input indices once (the rescores and the reference's
// (distance, index) tie-break work in input order).
// (n: the size of perm -- a sharded rank's padding slots hold stale keys
// from earlier calls, which must not be looked up)
__global__ void remap_kernel(uint64_t* __restrict__ keys, size_t count, const uint32_t* __restrict__ perm,
                             uint32_t n) {
    for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += size_t(gridDim.x) * blockDim.x) {
        const uint64_t k = keys[i];
        if (k != kEmptyKey && uint32_t(k) != kVirtualIdx && uint32_t(k) < n)
            keys[i] = (k & 0xffffffff00000000ull) | perm[uint32_t(k)];
    }
}

// The same for the capture buffers: only the first min(cnt, cap) entries of
// each slot were written.
__global__ void remap_capture_kernel(uint64_t* __restrict__ buf, const uint32_t* __restrict__ cnt, uint32_t m,
                                     uint32_t cap, const uint32_t* __restrict__ perm) {
    const uint32_t slot = blockIdx.x;
    if (slot >= m) return;
    const uint32_t c = min(cnt[slot], cap);
    uint64_t* b = buf + size_t(slot) * cap;
    for (uint32_t i = threadIdx.x; i < c; i += blockDim.x) {
        const uint64_t k = b[i];
        b[i] = (k & 0xffffffff00000000ull) | perm[uint32_t(k)];
    }
}

// The dynamic unit queue's item walk (DYN sweeps): this CTA's next item
// (column group g, local unit lu), false when the queue is drained.  role 0:
// the claiming producer (leader, warp 0); 1: a consumer in the leader; 2: a
// consumer in the peer.  warp_wide: the whole warp calls this (lane 0
// releases the queue slot).  Out of line: it runs once per item.
constexpr int kQN = 4;                 // queue slots
constexpr uint64_t kQEnd = ~0ull;      // the end-of-work item
struct ItemWalk {
    const uint32_t* units;
    uint32_t* qctr;
    uint32_t g_first, g_step, ngroups, ntiles, group_tiles, unit0, unit_step, nunits;
    uint32_t qbar0;  // qfull[kQN], qempty[kQN] mbarriers
    uint64_t* qitem;
    bool dyn, tri, pair;
    uint32_t g = 0, lu = 0, qi = 0;
    bool started = false;
};

__device__ __noinline__ bool item_next(ItemWalk& w, int role, bool warp_wide) {
    auto unit_id = [&](uint32_t lu) { return w.units ? __ldg(w.units + lu) : lu; };
    const int s = w.qi % kQN;
    const uint32_t ph = (w.qi / kQN) & 1;
    const uint32_t qfull = w.qbar0 + 8u * s, qempty = w.qbar0 + 8u * (kQN + s);
    ++w.qi;
    if (role == 0) {
        uint64_t item = kQEnd;
        while (w.g < w.ngroups) {
            const uint32_t t1 = min(w.ntiles, (w.g + 1) * w.group_tiles);
            const uint32_t lu = atomicAdd(w.qctr + w.g, 1u);
            if (lu < w.nunits && unit_id(lu) < t1) {  // (units ascending: a group's units with work are a prefix)
                w.lu = lu;
                item = (uint64_t(w.g) << 32) | lu;
                break;
            }
            ++w.g;  // the group's units are all taken
        }
        ptx::mbar_wait_cluster(qempty, ph ^ 1);
        w.qitem[s] = item;
        if (w.pair) {
            ptx::st_shared_cluster_u64(ptx::mapa_shared(ptx::smem_u32(w.qitem + s), 1), item);
            ptx::mbar_arrive_remote(ptx::mapa_shared(qfull, 1));
        }
        ptx::mbar_arrive(qfull);
        return item != kQEnd;
    }
    if (role == 2) ptx::mbar_wait_cluster(qfull, ph);
    else ptx::mbar_wait(qfull, ph);
    const uint64_t item = w.qitem[s];
    if (warp_wide) __syncwarp();
    if (!warp_wide || (threadIdx.x & 31) == 0) {
        if (role == 2) ptx::mbar_arrive_remote(ptx::mapa_shared(qempty, 0));
        else ptx::mbar_arrive(qempty);
    }
    w.g = uint32_t(item >> 32);
    w.lu = uint32_t(item);
    return item != kQEnd;
}

// Persistent sweep.  Work item = (column group g, row block rb); every CTA
// walks g = 0, 1, ... and, inside a group, its row blocks rb = blockIdx.x,
// blockIdx.x + gridDim.x, ...  All CTAs therefore stream the same column
// group at the same time and a group's reference tiles (sized to fit in L2)
// come from HBM once per group instead of once per row block.  The per-row
// candidate lists are written to `cand` at the end of each item and read
// back when the row block's next group starts.
// TCAP (with TRI): the threshold triangle -- both sides of every pair go to
// the pool against fixed per-row thresholds p.tc (no lists); the rows' pool
// entries are then rescored exactly like the band-capture pass.
// DYN (with TRI): the work items come from the dynamic unit queue (p.qctr);
// otherwise from the static walk.  Separate instantiations: the static walk's
// inlined loop is what the single-GPU list triangle runs (the queue's code in
// the same kernel cost C2 ~8% even when unused).
template <int KPL, int BN, bool ARES, int EW, bool CAPTURE, bool PAIR = false, bool TRI = false, bool TCAP = false,
          bool DYN = false>
__global__ void __launch_bounds__(TSLayout<KPL, BN, ARES, EW, PAIR>::THREADS, 1)
tensor_sweep_kernel(const SweepParams p) {
    using L = TSLayout<KPL, BN, ARES, EW, PAIR>;
    static_assert(!PAIR || !CAPTURE, "CTA pairs: no capture");
    static_assert(!TRI || (PAIR && BN == 256 && KPL <= 16), "triangle mode: CTA pairs, 256-column tiles");
    static_assert(!TCAP || TRI, "threshold mode is a triangle mode");
    constexpr int S = L::STAGES;
    constexpr int NSEG = L::NSEG;
    constexpr int SEG_COLS = BN / NSEG;  // columns of a tile one epilogue warp filters
    static_assert(SEG_COLS % 64 == 0 && (KPL % 16 == 0 || KPL < 16) && KPL % 2 == 0 && KPL <= SEG_COLS,
                  "tile / list shape");
    constexpr bool REGLIST = L::REGLIST && !CAPTURE;
    constexpr bool DIRECT = !REGLIST && KPL % 32 == 0;  // fill the first KPL columns without the filter
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* a_smem = smem;
    uint8_t* stage_smem = smem + L::A_BYTES;
    float* list_a = reinterpret_cast<float*>(stage_smem + S * L::STAGE);        // [KPL][LIST_ROWS]
    uint32_t* list_i = reinterpret_cast<uint32_t*>(list_a + KPL * L::LIST_ROWS);  // [KPL][LIST_ROWS]
    uint64_t* bars = reinterpret_cast<uint64_t*>(stage_smem + S * L::STAGE + L::LISTS);
    // bars: full[S], empty[S], tfull[2], tempty[2], afull, aempty
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * S + 6);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t ntiles = (p.n + BN - 1) / BN;
    const uint32_t nrb = (p.row_end - p.row_begin + TS_BM - 1) / TS_BM;
    const uint32_t ngroups = (ntiles + p.group_tiles - 1) / p.group_tiles;
    // Work units: row blocks, or (PAIR) pairs of row blocks 2u (leader) and
    // 2u+1 (peer); an odd last pair's peer block is all padding rows.
    uint32_t rank = 0;
    if constexpr (PAIR) rank = ptx::cluster_ctarank();
    const bool leader = rank == 0;
    const uint32_t unit0 = PAIR ? blockIdx.x / 2 : blockIdx.x;
    const uint32_t unit_step = PAIR ? gridDim.x / 2 : gridDim.x;
    const uint32_t nunits = p.units ? p.nunits : (PAIR ? (nrb + 1) / 2 : nrb);
    auto unit_id = [&](uint32_t lu) { return p.units ? __ldg(p.units + lu) : lu; };
    auto unit_block = [&](uint32_t u) { return PAIR ? 2 * u + rank : u; };
    // TRI: a pair unit's 256 rows are exactly tile u; it sweeps tiles >= u
    auto tri_start = [&](uint32_t u) -> uint32_t { return TRI ? u : 0u; };
    // Column groups: all of them in order (lists carry over from group to
    // group) -- except in CAPTURE mode, whose fixed thresholds let blockIdx.y
    // take a share of the groups so that few rows still fill the GPU.
    const uint32_t g_first = CAPTURE ? blockIdx.y : 0;
    const uint32_t g_step = CAPTURE ? gridDim.y : 1;
    const uint32_t bar0 = ptx::smem_u32(bars);
    auto full_bar = [&](int s) { return bar0 + 8u * s; };
    auto empty_bar = [&](int s) { return bar0 + 8u * (S + s); };
    auto tfull_bar = [&](int b) { return bar0 + 8u * (2 * S + b); };
    auto tempty_bar = [&](int b) { return bar0 + 8u * (2 * S + 2 + b); };
    const uint32_t afull_bar = bar0 + 8u * (2 * S + 4);
    const uint32_t aempty_bar = bar0 + 8u * (2 * S + 5);
    auto wait = [&](uint32_t bar, uint32_t parity) { ptx::mbar_wait(bar, parity); };
    // The dynamic unit queue (p.qctr): the leader's producer claims items and
    // publishes them through a QN-slot ring held in both CTAs' shared memory;
    // every other role (MMA issuer, epilogue warps, the peer's producer and
    // forwarder) takes the same items in the same order.
    constexpr int QN = kQN;
    static_assert(!DYN || TRI, "the unit queue serves the triangle sweeps");
    constexpr bool dyn = DYN;
    const uint32_t qbar0 = bar0 + 8u * (2 * S + 7);
    auto qfull_bar = [&](int s) { return qbar0 + 8u * s; };
    auto qempty_bar = [&](int s) { return qbar0 + 8u * (QN + s); };
    uint64_t* qitem = bars + 2 * S + 7 + 2 * QN;
    // This CTA's next work item: the queue (DYN: item_next, out of line) or
    // the static walk, inlined -- column groups in order; inside a group,
    // units unit0, unit0 + unit_step, ... that have tiles in the group.
    auto next = [&](ItemWalk& w, int role, bool warp_wide) -> bool {
        if constexpr (DYN) {
            if (role == 0) return item_next(w, 0, false);  // the claimer: out of line
            // consumers, inline: a call here costs the epilogue's hot loop
            // registers (C2: +8% instructions from rematerialised addresses)
            const int s = w.qi % kQN;
            const uint32_t ph = (w.qi / kQN) & 1;
            ++w.qi;
            if (role == 2) ptx::mbar_wait_cluster(qfull_bar(s), ph);
            else ptx::mbar_wait(qfull_bar(s), ph);
            const uint64_t item = qitem[s];
            if (warp_wide) __syncwarp();
            if (!warp_wide || lane == 0) {
                if (role == 2) ptx::mbar_arrive_remote(ptx::mapa_shared(qempty_bar(s), 0));
                else ptx::mbar_arrive(qempty_bar(s));
            }
            w.g = uint32_t(item >> 32);
            w.lu = uint32_t(item);
            return item != kQEnd;
        } else {
            for (;;) {
                if (!w.started) {
                    w.started = true;
                    w.g = g_first;
                    w.lu = unit0;
                } else {
                    w.lu += unit_step;
                }
                if (w.lu >= nunits) {
                    w.g += g_step;
                    w.lu = unit0;
                }
                if (w.g >= ngroups) return false;
                const uint32_t t0 = w.g * p.group_tiles, t1 = min(ntiles, t0 + p.group_tiles);
                if (w.lu < nunits && max(t0, tri_start(unit_id(w.lu))) < t1) return true;
            }
        }
    };
    auto make_walk = [&]() {
        ItemWalk w;
        w.units = p.units;
        w.qctr = p.qctr;
        w.g_first = g_first, w.g_step = g_step, w.ngroups = ngroups, w.ntiles = ntiles;
        w.group_tiles = p.group_tiles, w.unit0 = unit0, w.unit_step = unit_step, w.nunits = nunits;
        w.qbar0 = qbar0;
        w.qitem = qitem;
        w.dyn = dyn, w.tri = TRI, w.pair = PAIR;
        return w;
    };

    if (warp == 0 && lane == 0) {
        // PAIR: the leader's operand barriers also count the peer's
        // forwarded arrival, and its accumulator-empty barriers the peer's
        // epilogue warps; MMA completions are multicast to both CTAs.
        const uint32_t fwd = PAIR && leader ? 2 : 1;
        for (int s = 0; s < S; ++s) {
            ptx::mbar_init(full_bar(s), fwd);
            ptx::mbar_init(empty_bar(s), 1);
        }
        for (int b = 0; b < 2; ++b) {
            ptx::mbar_init(tfull_bar(b), 1);
            ptx::mbar_init(tempty_bar(b), (PAIR ? 2 : 1) * EW);  // one arrive per epilogue warp
        }
        ptx::mbar_init(afull_bar, fwd);
        ptx::mbar_init(aempty_bar, 1);
        if (dyn)
            for (int s = 0; s < QN; ++s) {
                ptx::mbar_init(qfull_bar(s), 1);
                // the leader's MMA issuer and epilogue warps, the peer's producer, forwarder and epilogue warps
                ptx::mbar_init(qempty_bar(s), 1 + EW + (PAIR ? 2 + EW : 0));
            }
        ptx::fence_mbar_init();
    }
    if constexpr (PAIR) {
        if (p.cta_ns && threadIdx.x == 0) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            p.cta_ns[2 * blockIdx.x] = t;
        }
        if (warp == 1) ptx::tmem_alloc_pair(ptx::smem_u32(tmem_slot), L::TMEM_COLS);
        ptx::tc_fence_before();
        ptx::cluster_sync();
    } else {
        if (warp == 1) ptx::tmem_alloc(ptx::smem_u32(tmem_slot), L::TMEM_COLS);
        ptx::tc_fence_before();
        __syncthreads();
    }
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ---------------- TMA producer (one lane) ----------------
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0, a_phase = 0;
            ItemWalk cur = make_walk();
            while (next(cur, leader ? 0 : 2, false)) {
                const uint32_t g = cur.g, lu = cur.lu;
                const uint32_t t0 = g * p.group_tiles, t1 = min(ntiles, t0 + p.group_tiles);
                {
                    const uint32_t u = unit_id(lu);
                    const uint32_t r0 = p.row_begin + unit_block(u) * TS_BM;
                    const uint32_t ts = max(t0, tri_start(u));
                    if constexpr (ARES) {  // A stays resident for the item; reload once the MMA released it
                        wait(aempty_bar, a_phase ^ 1);
                        ptx::mbar_arrive_expect_tx(afull_bar, p.kc * TS_A_CHUNK);
                        for (uint32_t kc = 0; kc < p.kc; ++kc)
                            ptx::bulk_g2s(ptx::smem_u32(a_smem + kc * TS_A_CHUNK),
                                          p.xa + (size_t(kc) * p.npad_a + r0) * 128, TS_A_CHUNK, afull_bar);
                        a_phase ^= 1;
                    }
                    for (uint32_t t = ts; t < t1; ++t) {
                        for (uint32_t kc = 0; kc < p.kc; ++kc) {
                            wait(empty_bar(stage), phase ^ 1);
                            if (p.debug_mode == 3) {  // profiling: MMA on stale tiles, no loads
                                ptx::mbar_arrive(full_bar(stage));
                                if (++stage == S) {
                                    stage = 0;
                                    phase ^= 1;
                                }
                                continue;
                            }
                            ptx::mbar_arrive_expect_tx(full_bar(stage), L::STAGE);
                            uint8_t* dst = stage_smem + stage * L::STAGE;
                            // PAIR: this CTA's half of the tile's columns
                            ptx::bulk_g2s(ptx::smem_u32(dst),
                                          p.xh + (size_t(kc) * p.npad + size_t(t) * BN + rank * (BN / 2)) * 128,
                                          L::B_CHUNK, full_bar(stage));
                            if constexpr (!ARES)
                                ptx::bulk_g2s(ptx::smem_u32(dst + L::B_CHUNK),
                                              p.xa + (size_t(kc) * p.npad_a + r0) * 128, TS_A_CHUNK, full_bar(stage));
                            if (++stage == S) {
                                stage = 0;
                                phase ^= 1;
                            }
                        }
                    }
                }
            }
        }
    } else if (warp == 1 && PAIR && !leader) {
        // ---------------- peer: forward operand arrivals to the leader ----------------
        if (lane == 0) {
            const uint32_t lead_full0 = ptx::mapa_shared(full_bar(0), 0);
            const uint32_t lead_afull = ptx::mapa_shared(afull_bar, 0);
            int stage = 0;
            uint32_t phase = 0, a_phase = 0;
            ItemWalk cur = make_walk();
            while (next(cur, 2, false)) {
                const uint32_t g = cur.g, lu = cur.lu;
                const uint32_t t0 = g * p.group_tiles, t1 = min(ntiles, t0 + p.group_tiles);
                const uint32_t ts = max(t0, tri_start(unit_id(lu)));
                if constexpr (ARES) {
                    wait(afull_bar, a_phase);
                    a_phase ^= 1;
                    ptx::mbar_arrive_remote_relaxed(lead_afull);
                }
                for (uint32_t t = ts; t < t1; ++t)
                    for (uint32_t kc = 0; kc < p.kc; ++kc) {
                        wait(full_bar(stage), phase);
                        ptx::mbar_arrive_remote_relaxed(lead_full0 + 8u * stage);
                        if (++stage == S) {
                            stage = 0;
                            phase ^= 1;
                        }
                    }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer (one lane; PAIR: the leader's) ----------------
        if (lane == 0) {
            constexpr uint32_t idesc = ptx::idesc_f16_f32(PAIR ? 2 * TS_BM : TS_BM, BN);
            // The operand kind is a template argument of the issue loop, not a
            // runtime select per MMA: a select compiles to a predicated
            // UTCQMMA + UTCHMMA pair per MMA, and the predicated-off one still
            // occupies the tcgen05 pipe (C2 sweep: tensor pipe 64% busy with
            // the tcgen05 pipe at 88%; cuBLAS: 96% / 96%, profiles/r02ba_*).
            auto issue = [&](auto f8) {
                [[maybe_unused]] constexpr bool F8 = decltype(f8)::value;
                auto mma = [&](uint32_t d, uint64_t a, uint64_t b, uint32_t acc) {
                    if constexpr (PAIR) {
                        if constexpr (F8) ptx::mma_e4m3_ss_pair(d, a, b, idesc, acc);
                        else ptx::mma_f16_ss_pair(d, a, b, idesc, acc);
                    } else {
                        ptx::mma_f16_ss(d, a, b, idesc, acc);
                    }
                };
                auto commit = [&](uint32_t bar) {
                    if constexpr (PAIR) ptx::mma_commit_pair(bar);
                    else ptx::mma_commit(bar);
                };
                int stage = 0;
                uint32_t phase = 0, a_phase = 0, tcount = 0;
                ItemWalk cur = make_walk();
                while (next(cur, 1, false)) {
                    const uint32_t g = cur.g, lu = cur.lu;
                    const uint32_t t0 = g * p.group_tiles, t1 = min(ntiles, t0 + p.group_tiles);
                    {
                        const uint32_t ts = max(t0, tri_start(unit_id(lu)));
                        if constexpr (ARES) {
                            wait(afull_bar, a_phase);
                            a_phase ^= 1;
                        }
                        for (uint32_t t = ts; t < t1; ++t, ++tcount) {
                            const uint32_t b = tcount & 1, use = tcount >> 1;
                            wait(tempty_bar(b), (use & 1) ^ 1);
                            ptx::tc_fence_after();
                            const uint32_t d_tmem = tmem + b * BN;
                            for (uint32_t kc = 0; kc < p.kc; ++kc) {
                                wait(full_bar(stage), phase);
                                ptx::tc_fence_after();
                                const uint8_t* bsm = stage_smem + stage * L::STAGE;
                                const uint8_t* asm_ = ARES ? a_smem + kc * TS_A_CHUNK : bsm + L::B_CHUNK;
                                const uint32_t a_addr = ptx::smem_u32(asm_);
                                const uint32_t b_addr = ptx::smem_u32(bsm);
    #pragma unroll
                                for (uint32_t k = 0; k < 4; ++k) {  // UMMA_K = 16 fp16 = 32 B inside the swizzle atom
                                    mma(d_tmem, ptx::sw128_kmajor_desc(a_addr + 32 * k),
                                        ptx::sw128_kmajor_desc(b_addr + 32 * k), (kc | k) != 0);
                                }
                                commit(empty_bar(stage));
                                if (++stage == S) {
                                    stage = 0;
                                    phase ^= 1;
                                }
                            }
                            commit(tfull_bar(b));
                        }
                        if constexpr (ARES) commit(aempty_bar);  // A may be replaced once these MMAs retire
                    }
                }
            };
            if (PAIR && p.e4m3) issue(std::true_type{});
            else issue(std::false_type{});
        }
    } else {
        // ---------------- epilogue: one thread per (query row, column segment) ----------------
        const int ew = warp - 2;
        const int quad = warp & 3;       // TMEM lanes 32*quad .. +31 are this warp's
        const int seg = ew / 4;          // which column segment of every tile
        const int rl = quad * 32 + lane;
        const int lidx = seg * TS_BM + rl;  // this thread's list
        float* my_a = list_a + lidx;
        uint32_t* my_i = list_i + lidx;
        const uint32_t a_base = ptx::smem_u32(my_a), i_base = ptx::smem_u32(my_i);
        const float kInf = __int_as_float(0x7f800000);
        const uint32_t lane_addr = tmem + (uint32_t(quad * 32) << 16);
        const uint32_t seg0 = seg * SEG_COLS;
        // columns per TMEM load / filter step (16-column chunks with the
        // norms pipelined too measured 6% slower at C2)
        constexpr int W = 32;
        auto load_beta = [&](uint32_t col0, float (&bt)[W]) {
            const float4* beta4 = reinterpret_cast<const float4*>(p.alpha + col0);
#pragma unroll
            for (int q = 0; q < W / 4; ++q) {
                const float4 f = __ldg(beta4 + q);
                bt[4 * q] = f.x;
                bt[4 * q + 1] = f.y;
                bt[4 * q + 2] = f.z;
                bt[4 * q + 3] = f.w;
            }
        };
        // Register-resident list (KPL <= 16): replacing the maximum is 2 KPL
        // selects plus a 4-level (value, slot) max tree -- no memory on the
        // critical path.  Larger lists live in shared memory.
        float la[REGLIST ? KPL : 1];
        uint32_t lx[REGLIST ? KPL : 1];
        ListMax thr{kInf, 0};
        auto reg_argmax = [&]() -> ListMax {
            constexpr int H = REGLIST ? KPL / 2 : 1;
            float mv[H];
            uint32_t ms[H];
#pragma unroll
            for (int i = 0; i < H; ++i) {
                const bool r = la[REGLIST ? 2 * i + 1 : 0] > la[REGLIST ? 2 * i : 0];
                mv[i] = r ? la[REGLIST ? 2 * i + 1 : 0] : la[REGLIST ? 2 * i : 0];
                ms[i] = r ? 2 * i + 1 : 2 * i;
            }
            // tournament over H entries (any H; odd levels carry their last entry)
#pragma unroll
            for (int h = H; h > 1; h = (h + 1) / 2) {
                const int h2 = (h + 1) / 2;
#pragma unroll
                for (int i = 0; i + h2 < h; ++i) {
                    const bool r = mv[i + h2] > mv[i];
                    mv[i] = r ? mv[i + h2] : mv[i];
                    ms[i] = r ? ms[i + h2] : ms[i];
                }
            }
            return ListMax{mv[0], ms[0]};
        };
        uint32_t cap_slot = 0;
        auto insert = [&](float y, uint32_t col) {
            if constexpr (CAPTURE) {
                const uint32_t at = atomicAdd(p.cap_cnt + cap_slot, 1u);
                if (at < p.cap) p.cap_buf[size_t(cap_slot) * p.cap + at] = (uint64_t(float_to_ordered(y)) << 32) | col;
            } else if constexpr (REGLIST) {
#pragma unroll
                for (int s = 0; s < KPL; ++s) {
                    const bool h = uint32_t(s) == thr.slot;
                    la[s] = h ? y : la[s];
                    lx[s] = h ? col : lx[s];
                }
                thr = reg_argmax();
            } else {
                thr = list_replace_max<KPL, L::STRIDE>(a_base, i_base, thr.slot, y, col);
            }
        };
        uint32_t tcount = 0;
        // TRI: this warp's current chunk of the column-side pool (warp-uniform)
        uint32_t wchunk = 0xffffffffu, wfill = kLogChunk;
        // accumulator release: PAIR peers arrive on the leader's barrier
        const uint32_t tempty_rel0 = PAIR && !leader ? ptx::mapa_shared(tempty_bar(0), 0) : tempty_bar(0);
        auto release_acc = [&](uint32_t b) {
            if constexpr (PAIR) {
                if (!leader) {
                    ptx::mbar_arrive_remote_relaxed(tempty_rel0 + 8u * b);
                    return;
                }
            }
            ptx::mbar_arrive(tempty_bar(b));
        };
        ItemWalk cur = make_walk();
        while (next(cur, leader ? 1 : 2, true)) {
            const uint32_t g = cur.g, lu = cur.lu;
            const uint32_t t0 = g * p.group_tiles, t1 = min(ntiles, t0 + p.group_tiles);
            {
                const uint32_t u = unit_id(lu);
                const uint32_t tsu = tri_start(u), ts = max(t0, tsu);
                const bool fresh = TRI ? t0 <= tsu : g == 0;  // the unit's first group with work
                const uint32_t row = p.row_begin + unit_block(u) * TS_BM + rl;
                const bool valid = row < p.row_end;
                const float alpha_i = TRI && valid ? p.alpha[row] : kInf;  // column side: this row's norm
                const float alpha_h = bound_half(alpha_i, 1.0f);              // its half for the column bound
                // list slot: the row's offset in the call (or, with a unit list, in this rank's units)
                const uint32_t lrow = p.units ? lu * (PAIR ? 2 * TS_BM : TS_BM) + (PAIR ? rank * TS_BM : 0) + rl
                                              : row - p.row_begin;
                uint64_t* state = p.cand + (size_t(lrow) * NSEG + seg) * KPL;
                // Columns are ranked by y = fl(beta_j - 2 dot): alpha_i is
                // constant along a row; the rescore forms A = alpha_i + y in fp64.
                if constexpr (CAPTURE) {
                    cap_slot = row - p.row_begin;
                    // fixed threshold: admit y <= cap_thr (strict < against its successor)
                    thr = ListMax{valid ? nextafterf(p.cap_thr[cap_slot], kInf) : -kInf, 0};
                } else if constexpr (TCAP) {
                    thr = ListMax{valid ? __ldg(p.tc + row) : -kInf, 0};  // fixed: the row's threshold
                } else if constexpr (REGLIST) {
                    if (dyn && !fresh) {  // the unit's previous group may have run on another pair: wait for its lists
                        if (lane == 0) {
                            const uint32_t need = (PAIR ? 2 : 1) * EW * (g - u / p.group_tiles);
                            while (ptx::ld_acquire_gpu_u32(p.udone + lu) < need) __nanosleep(64);
                        }
                        __syncwarp();
                    }
#pragma unroll
                    for (int s = 0; s < KPL; ++s) {
                        uint64_t key = (fresh || !valid) ? kEmptyKey : __ldcg(state + s);
                        if constexpr (TRI) {
                            if (fresh && valid) key = make_key(__ldg(p.tc + row), kVirtualIdx);
                        }
                        la[s] = key == kEmptyKey ? kInf : ordered_to_float(uint32_t(key >> 32));
                        lx[s] = uint32_t(key);
                    }
                    thr = reg_argmax();
                } else if (fresh || !valid) {
#pragma unroll 4
                    for (int s = 0; s < KPL; ++s) {
                        my_a[s * L::LIST_ROWS] = kInf;
                        my_i[s * L::LIST_ROWS] = 0xffffffffu;
                    }
                    thr = ListMax{kInf, 0};
                } else {
                    for (int s = 0; s < KPL; ++s) {
                        const uint64_t key = state[s];
                        my_a[s * L::LIST_ROWS] = key == kEmptyKey ? kInf : ordered_to_float(uint32_t(key >> 32));
                        my_i[s * L::LIST_ROWS] = uint32_t(key);
                    }
                    thr = list_rescan<KPL, L::STRIDE>(a_base);
                }
                if (!valid) thr.a = -kInf;  // padding rows admit nothing
                // After a chunk's vote: the column side's appends (TRI), then the
                // row side's rare path.
                // Warp-aggregated appends to the pool: every lane walks its mask
                // m of the chunk's columns; entry (key, dest) -- the column side:
                // (y', row) for column col; the threshold triangle's row side:
                // (col) for this row.  Slots come from a ballot prefix (no
                // atomics but one per pool chunk); a select tree picks each dot.
                auto append = [&](uint32_t m, const uint32_t (&v)[W], uint32_t col0, bool rowside, float bm) {
                    while (__any_sync(0xffffffffu, m != 0)) {
                        const int bpos = m ? __ffs(m) - 1 : 0;
                        const bool ok = m != 0 && col0 + bpos < p.n;
                        m &= m - 1;
                        const uint32_t bal = __ballot_sync(0xffffffffu, ok);
                        if (wfill + __popc(bal) > uint32_t(kLogChunk)) {  // next chunk of the pool
                            uint32_t nc = 0;
                            if (lane == 0) {
                                if (wchunk < p.nchunks) p.lcnt[wchunk] = wfill;
                                nc = atomicAdd(p.lnext, 1u);
                            }
                            wchunk = __shfl_sync(0xffffffffu, nc, 0);
                            wfill = 0;
                        }
                        if (ok) {
                            const size_t slot = size_t(wchunk) * kLogChunk + wfill + __popc(bal & ((1u << lane) - 1u));
                            uint32_t t16[16];
#pragma unroll
                            for (int q = 0; q < 16; ++q) t16[q] = (bpos & 16) ? v[q + 16] : v[q];
#pragma unroll
                            for (int q = 0; q < 8; ++q) t16[q] = (bpos & 8) ? t16[q + 8] : t16[q];
#pragma unroll
                            for (int q = 0; q < 4; ++q) t16[q] = (bpos & 4) ? t16[q + 4] : t16[q];
#pragma unroll
                            for (int q = 0; q < 2; ++q) t16[q] = (bpos & 2) ? t16[q + 2] : t16[q];
                            const float dot = __uint_as_float((bpos & 1) ? t16[1] : t16[0]);
                            // key: (y relative to the destination row, the other endpoint);
                            // the row side uses the chunk's smallest norm bm for beta_j: a
                            // lower bound on y, which is all the capture rescore's ordering
                            // and skip test need (a smaller A is never skipped wrongly)
                            const uint64_t key = rowside ? make_key(__fmaf_rn(-2.0f, dot, bm), col0 + bpos)
                                                         : make_key(__fmaf_rn(-2.0f, dot, alpha_i), row);
                            if (wchunk < p.nchunks) {
                                p.lkey[slot] = key;
                                p.lcol[slot] = rowside ? row : col0 + bpos;
                            }
                        }
                        wfill += __popc(bal);
                    }
                };
                // After a chunk's vote: the column side's appends (TRI), then the
                // row side's rare path (TCAP: appends as well).
                // bm_lo (TCAP): a lower bound on the chunk's smallest column norm
                auto handle = [&](const uint32_t (&v)[W], uint32_t col0, bool fire_r, bool fire_c, float hc,
                                  float hr, float bm_lo) {
                    constexpr int P = W / 2;  // column pairs
                    float bt[W];              // the chunk's column norms
                    if constexpr (TRI) {
                        if (__any_sync(0xffffffffu, fire_c)) {
                            // admitted columns: dot > hc, a superset of y' < the chunk's
                            // largest threshold (the rescore filters the few extra)
                            uint32_t cm = 0;
                            if (fire_c) {
#pragma unroll
                                for (int j = 0; j < W; ++j)
                                    if (__uint_as_float(v[j]) > hc) cm |= 1u << j;
                            }
                            append(cm, v, col0, false, 0.0f);
                        }
                        if constexpr (TCAP) {
                            // row side against the fixed threshold: dot > hr, a
                            // superset of y < thr (the capture rescore filters)
                            if (__any_sync(0xffffffffu, fire_r)) {
                                uint32_t rm = 0;
                                if (fire_r) {
#pragma unroll
                                    for (int j = 0; j < W; ++j)
                                        if (__uint_as_float(v[j]) > hr) rm |= 1u << j;
                                }
                                append(rm, v, col0, true, bm_lo);
                            }
                            return;
                        }
                        if (!__any_sync(0xffffffffu, fire_r)) return;
                    }
                    load_beta(col0, bt);
                    // rare path: per-lane pair mask, then each lane walks its own
                    // admitted pairs; a pair's two values are picked with a
                    // 4-level select tree (no dynamic register indexing, one copy
                    // of the insertion code per call site)
                    float ye[P], yo[P];
                    uint32_t pm = 0;
#pragma unroll
                    for (int i = 0; i < P; ++i) {
                        const float2 y2 = ptx::ffma2_m2(v[2 * i], v[2 * i + 1], bt[2 * i], bt[2 * i + 1]);
                        ye[i] = y2.x;
                        yo[i] = y2.y;
                        if (fminf(ye[i], yo[i]) < thr.a) pm |= 1u << i;
                    }
                    while (pm) {  // each lane walks its own pairs (the warp: max over lanes)
                        const int i = __ffs(pm) - 1;
                        pm &= pm - 1;
                        {
                            float e8[8], o8[8];
#pragma unroll
                            for (int q = 0; q < 8; ++q) {
                                if constexpr (P == 16) {
                                    e8[q] = (i & 8) ? ye[q + 8] : ye[q];
                                    o8[q] = (i & 8) ? yo[q + 8] : yo[q];
                                } else {
                                    e8[q] = ye[q];
                                    o8[q] = yo[q];
                                }
                            }
#pragma unroll
                            for (int q = 0; q < 4; ++q) {
                                e8[q] = (i & 4) ? e8[q + 4] : e8[q];
                                o8[q] = (i & 4) ? o8[q + 4] : o8[q];
                            }
#pragma unroll
                            for (int q = 0; q < 2; ++q) {
                                e8[q] = (i & 2) ? e8[q + 2] : e8[q];
                                o8[q] = (i & 2) ? o8[q + 2] : o8[q];
                            }
                            const float y0 = (i & 1) ? e8[1] : e8[0];
                            const float y1 = (i & 1) ? o8[1] : o8[0];
                            const uint32_t col = col0 + 2 * i;
                            if (y0 < thr.a && col < p.n) insert(y0, col);
                            if (y1 < thr.a && col + 1 < p.n) insert(y1, col + 1);
                        }
                    }
                };
                // hot path: y_j = fl(beta_j - 2 dot_j) < thr needs
                // dot_j > (beta_j - thr) / 2 >= h = (min beta of the chunk - thr) / 2,
                // so the raw dots are tested against h: a 3-input FMNMX3 max
                // tree (15 instructions for 32 values), one compare, one vote
                // per two chunks, and no column-norm loads.  At the boundary
                // y ~ thr, so y's rounding is ~2^-24 |thr|; the slack covers it
                // and h's own rounding many times over -- a superset of the
                // exact test, which the rare path then applies unchanged.
                static_assert(W == 32, "max tree is laid out for 32 columns");
                auto vmax = [&](const uint32_t (&v)[W]) -> float {
                    float r1[11], r2[4];
#pragma unroll
                    for (int j = 0; j < 10; ++j)
                        r1[j] = fmaxf(fmaxf(__uint_as_float(v[3 * j]), __uint_as_float(v[3 * j + 1])),
                                      __uint_as_float(v[3 * j + 2]));
                    r1[10] = fmaxf(__uint_as_float(v[30]), __uint_as_float(v[31]));
#pragma unroll
                    for (int j = 0; j < 3; ++j) r2[j] = fmaxf(fmaxf(r1[3 * j], r1[3 * j + 1]), r1[3 * j + 2]);
                    r2[3] = fmaxf(r1[9], r1[10]);
                    return fmaxf(fmaxf(fmaxf(r2[0], r2[1]), r2[2]), r2[3]);
                };
                // h for a chunk whose smallest column norm is bm (slack 2^-20)
                auto row_bound = [&](float bm) -> float {
                    float h = __fmul_rn(__fsub_rn(bm, thr.a), 0.5f);
                    if (fabsf(h) < kInf) h = __fsub_rn(h, 9.5367431640625e-07f * (fabsf(bm) + fabsf(thr.a)));
                    return h;
                };
                // column side: y' = fl(alpha_i - 2 dot) < tc_j needs
                // dot > (alpha_i - max_chunk tc) / 2 (same slack argument)
                auto col_bound = [&](float tcm) -> float {
                    float hc = __fmul_rn(__fsub_rn(alpha_i, tcm), 0.5f);
                    if (fabsf(hc) < kInf) hc = __fsub_rn(hc, 9.5367431640625e-07f * (fabsf(alpha_i) + fabsf(tcm)));
                    return hc;
                };
                // One W-column chunk with its own bounds (the first tile of a
                // fresh shared-memory list only): direct = position among the
                // first KPL columns this thread sees, or -1.
                auto process = [&](const uint32_t (&v)[W], uint32_t col0, int direct, bool cside) {
                    float bt[W];
                    if constexpr (!REGLIST) {
                        if (direct >= 0) {  // first KPL columns: fill the list directly
                            load_beta(col0, bt);
#pragma unroll
                            for (int j = 0; j < W; ++j) {
                                const uint32_t col = col0 + j;
                                my_a[(direct + j) * L::LIST_ROWS] =
                                    col < p.n ? __fmaf_rn(-2.0f, __uint_as_float(v[j]), bt[j]) : kInf;
                                my_i[(direct + j) * L::LIST_ROWS] = col < p.n ? col : 0xffffffffu;
                            }
                            if (direct + W == KPL && valid) thr = list_rescan<KPL, L::STRIDE>(a_base);
                            return;
                        }
                    }
                    const float dmax = vmax(v);
                    const float hr1 = row_bound(__ldg(p.bmin + (col0 >> 5)));
                    const bool fire_r = dmax > hr1;
                    bool fire_c = false;
                    float hc = kInf;
                    if constexpr (TRI) {
                        if (cside && valid) {
                            hc = col_bound(__ldg(p.tcmax + (col0 >> 5)));
                            fire_c = dmax > hc;
                        }
                    }
                    if (!__any_sync(0xffffffffu, fire_r || fire_c) || p.debug_mode == 4) return;
                    handle(v, col0, fire_r, fire_c, hc, hr1, 0.0f);
                };
                constexpr int NCH = SEG_COLS / 32;
                for (uint32_t t = ts; t < t1; ++t, ++tcount) {
                    const uint32_t b = tcount & 1, use = tcount >> 1;
                    const uint32_t cbase = t * BN + seg0;
                    // the tile's chunk norms (and column thresholds) are loaded
                    // before the accumulator wait, so their L2 latency overlaps it
                    float bmv[NCH], tcm[NCH];
                    {
                        // (the chunks' bound halves: chunk_min_kernel / chunk_max_kernel)
                        const float* bp = p.bmin + p.npad / 32 + (cbase >> 5);
                        if constexpr (NCH % 4 == 0) {
#pragma unroll
                            for (int q = 0; q < NCH / 4; ++q) {
                                const float4 f = __ldg(reinterpret_cast<const float4*>(bp) + q);
                                bmv[4 * q] = f.x, bmv[4 * q + 1] = f.y, bmv[4 * q + 2] = f.z, bmv[4 * q + 3] = f.w;
                            }
                        } else {
#pragma unroll
                            for (int q = 0; q < NCH; ++q) bmv[q] = __ldg(bp + q);
                        }
#pragma unroll
                        for (int q = 0; q < NCH; ++q) tcm[q] = kInf;
                        if constexpr (TRI) {
                            if (TRI && t > tsu && valid) {
                                const float* tp = p.tcmax + p.npad / 32 + (cbase >> 5);
#pragma unroll
                                for (int q = 0; q < NCH; ++q) tcm[q] = __ldg(tp + q);
                            }
                        }
                    }
                    wait(tfull_bar(b), use & 1);
                    ptx::tc_fence_after();
                    const uint32_t taddr = lane_addr + b * BN + seg0;
                    const bool first = DIRECT && g == 0 && t == 0;
                    const bool cside = TRI && t > tsu;  // tiles above the unit's own: both sides
                    // Next tile's column norms into L1 now, so the in-loop
                    // loads of that tile hit L1 instead of paying L2 latency.
                    if (!TCAP && lane < SEG_COLS / 32 && t + 1 < t1)
                        asm volatile("prefetch.global.L1 [%0];" ::"l"(p.alpha + cbase + BN + lane * 32));
                    if (p.debug_mode && p.debug_mode != 4) {  // pipeline-ceiling experiments
                        uint32_t vd[32];
                        if (p.debug_mode == 1)
                            for (int c0 = 0; c0 < SEG_COLS; c0 += 32) {
                                ptx::tmem_ld_32x32b_x32(taddr + c0, vd);
                                ptx::tmem_wait_ld();
                                if (vd[0] == 0x7fc00001u && vd[31] == 0x7fc00001u) thr.a = 0.0f;  // keep the loads
                            }
                        ptx::tc_fence_before();
                        __syncwarp();
                        if (lane == 0) release_acc(b);
                        continue;
                    }
                    // This tile's chunk bounds, once per tile.  A row bound computed
                    // before an insertion earlier in the tile is below the fresh
                    // one (thr only falls), so it admits a superset: still exact.
                    // h = bound_half(beta_min) + bound_half(thr, -1) (row side),
                    // bound_half(alpha_i) + bound_half(tc_max, -1) (column side)
                    float hr[NCH], hcv[NCH];
                    const float thr_h = bound_half(thr.a, -1.0f);
#ifdef KNN_OLD_BOUNDS
#pragma unroll
                    for (int q = 0; q < NCH; ++q) {
                        hr[q] = row_bound(2.0f * bmv[q]);
                        hcv[q] = TRI && cside && valid ? col_bound(-2.0f * tcm[q]) : kInf;
                    }
#else
#pragma unroll
                    for (int q = 0; q < NCH; ++q) {
                        hr[q] = __fadd_rn(bmv[q], thr_h);
                        hcv[q] = TRI && cside && valid ? __fadd_rn(alpha_h, tcm[q]) : kInf;
                    }
#endif
                    uint32_t va[32], vb[32];
                    // two chunks per step: both TMEM reads, two independent max
                    // trees, one vote; column norms only for chunks that reach
                    // the rare path (from L1, prefetched one tile ahead)
#pragma unroll 1
                    for (int it = 0; it < NCH / 2; ++it) {
                        const uint32_t c0 = uint32_t(it) * 64;
                        ptx::tmem_ld_32x32b_x32(taddr + c0, va);
                        ptx::tmem_ld_32x32b_x32(taddr + c0 + 32, vb);
                        ptx::tmem_wait_ld();
                        if (it + 1 == NCH / 2) {  // this warp's part of the accumulator is in registers: release it
                            ptx::tc_fence_before();
                            __syncwarp();
                            if (lane == 0) release_acc(b);
                        }
                        if constexpr (DIRECT) {
                            if (first && c0 < uint32_t(KPL)) {
                                process(va, cbase + c0, int(c0), cside);
                                process(vb, cbase + c0 + 32, c0 + 32 < uint32_t(KPL) ? int(c0) + 32 : -1, cside);
                                continue;
                            }
                        }
                        float ha = hr[0], hb = hr[1], ca = hcv[0], cb = hcv[1], ba = bmv[0], bb = bmv[1];
#pragma unroll
                        for (int q = 1; q < NCH / 2; ++q) {
                            const bool at = it == q;
                            ha = at ? hr[2 * q] : ha;
                            hb = at ? hr[2 * q + 1] : hb;
                            if constexpr (TRI) {
                                ca = at ? hcv[2 * q] : ca;
                                cb = at ? hcv[2 * q + 1] : cb;
                            }
                            if constexpr (TCAP) {
                                ba = at ? bmv[2 * q] : ba;
                                bb = at ? bmv[2 * q + 1] : bb;
                            }
                        }
                        const float da = vmax(va), db = vmax(vb);
                        const bool ra = da > ha, rb = db > hb;
                        const bool fa = TRI && da > ca, fb = TRI && db > cb;
                        if (!__any_sync(0xffffffffu, ra || rb || fa || fb) || p.debug_mode == 4) continue;
                        // (2 bound_half(beta_min) <= beta_min: the TCAP row side's norm, no load)
                        if (__any_sync(0xffffffffu, ra || fa)) handle(va, cbase + c0, ra, fa, ca, ha, 2.0f * ba);
                        if (__any_sync(0xffffffffu, rb || fb)) handle(vb, cbase + c0 + 32, rb, fb, cb, hb, 2.0f * bb);
                    }
                }
                if (valid && !CAPTURE && !TCAP) {
                    for (int s = 0; s < KPL; ++s) {
                        float a;
                        uint32_t col;
                        if constexpr (REGLIST) {
                            a = la[s];
                            col = lx[s];
                        } else {
                            a = my_a[s * L::LIST_ROWS];
                            col = my_i[s * L::LIST_ROWS];
                        }
                        state[s] = col == 0xffffffffu ? kEmptyKey : (uint64_t(float_to_ordered(a)) << 32) | col;
                    }
                }
                if (dyn && !TCAP) {  // this warp's part of the unit's lists is saved: count it
                    __syncwarp();
                    if (lane == 0) {
                        __threadfence();
                        atomicAdd(p.udone + lu, 1u);
                    }
                }
            }
        }
        if constexpr (TRI) {
            if (lane == 0 && wchunk < p.nchunks) p.lcnt[wchunk] = wfill;
        }
    }
    ptx::tc_fence_before();
    if constexpr (PAIR) {
        ptx::cluster_sync();  // neither CTA frees TMEM while the pair's MMAs may write it
        if (p.cta_ns && threadIdx.x == 0) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            p.cta_ns[2 * blockIdx.x + 1] = t;
        }
        if (warp == 1) {
            ptx::tc_fence_after();
            ptx::tmem_dealloc_pair(tmem, L::TMEM_COLS);
        }
    } else {
        __syncthreads();
        if (warp == 1) {
            ptx::tc_fence_after();
            ptx::tmem_dealloc(tmem, L::TMEM_COLS);
        }
    }
}

// ---------------------------------------------------------------------------
// prep kernels


// ---- triangle mode helpers --------------------------------------------------

__global__ void iota_stride_kernel(uint32_t* __restrict__ out, uint32_t m, uint32_t stride) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) out[i] = i * stride;
}

__global__ void gather_alpha_kernel(const float* __restrict__ alpha, const uint32_t* __restrict__ rows, uint32_t m,
                                    uint32_t mpad, float scale, float* __restrict__ out) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < mpad; i += gridDim.x * blockDim.x)
        out[i] = i < m ? __fmul_rn(alpha[rows[i]], scale) : __int_as_float(0x7f800000);
}

// E4M3 copy of the swizzled fp16 planes for the triangle's sample pass: the
// fp16 values (|h| <= 65504, prep_kernel) times 2^-8 fit E4M3 (max 448); a
// 128-byte chunk row holds 128 elements, i.e. two fp16 chunks.  Dots come out
// scaled by 2^-16; the sample pass's norms are scaled to match
// (gather_alpha_kernel) and its thresholds scaled back (tri_threshold_kernel).
constexpr float kE4m3Scale = 0.00390625f;  // 2^-8
__global__ void e4m3_planes_kernel(const uint8_t* __restrict__ xh, uint32_t npad, uint32_t kc, uint32_t kc8,
                                   uint8_t* __restrict__ x8) {
    const uint32_t total = kc8 * npad * 8;  // 16-byte units of the E4M3 planes
    for (uint32_t u = blockIdx.x * blockDim.x + threadIdx.x; u < total; u += gridDim.x * blockDim.x) {
        const uint32_t unit = u & 7, r = (u >> 3) % npad, c8 = (u >> 3) / npad;
        const uint32_t c = 2 * c8 + (unit >> 2);  // source fp16 chunk
        uint32_t w[4] = {0u, 0u, 0u, 0u};
        if (c < kc) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {  // two 16-byte fp16 units = 16 elements
                const uint32_t lu = 2 * (unit & 3) + h;
                const uint4 v = *reinterpret_cast<const uint4*>(xh + (size_t(c) * npad + r) * 128 + ((lu ^ (r & 7)) << 4));
                const uint32_t hv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    __half2_raw h2;
                    h2.x = uint16_t(hv[q]);
                    h2.y = uint16_t(hv[q] >> 16);
                    float2 f = __half22float2(__half2(h2));
                    f.x = __fmul_rn(f.x, kE4m3Scale);
                    f.y = __fmul_rn(f.y, kE4m3Scale);
                    const uint32_t b2 = __nv_cvt_float2_to_fp8x2(f, __NV_SATFINITE, __NV_E4M3);
                    w[(4 * h + q) >> 1] |= b2 << (16 * (q & 1));
                }
            }
        }
        *reinterpret_cast<uint4*>(x8 + (size_t(c8) * npad + r) * 128 + ((unit ^ (r & 7)) << 4)) =
            make_uint4(w[0], w[1], w[2], w[3]);
    }
}

// Column-side threshold of row j: the r-th smallest y among its KP sample
// candidates (any value is correct -- it only sets how many rows the column
// side appends); padding rows get -inf (never admit).
// tl[j]: the largest of them -- a looser capture threshold for a row whose
// triangle pass ends with fewer than k candidates (the capture re-checks it).
// Rows [j0, j1) (sorted order); cand holds their lists from row j0 on.
__global__ void tri_threshold_kernel(const uint64_t* __restrict__ cand, uint32_t n, uint32_t j0, uint32_t j1,
                                     uint32_t kp, uint32_t r, float unscale, float* __restrict__ tc,
                                     float* __restrict__ tl) {
    for (uint32_t j = j0 + blockIdx.x * blockDim.x + threadIdx.x; j < j1; j += gridDim.x * blockDim.x) {
        float t = -__int_as_float(0x7f800000), l = t;
        if (j < n) {
            const uint64_t* c = cand + size_t(j - j0) * kp;
            uint64_t best = kEmptyKey, last = 0;
            for (uint32_t a = 0; a < kp; ++a) {
                uint32_t below = 0;
                for (uint32_t b = 0; b < kp; ++b) below += c[b] < c[a];
                if (below == r - 1) best = c[a];
                if (c[a] != kEmptyKey && c[a] > last) last = c[a];
            }
            t = best == kEmptyKey ? __int_as_float(0x7f800000) : __fmul_rn(ordered_to_float(uint32_t(best >> 32)), unscale);
            l = last == 0 ? l : __fmul_rn(ordered_to_float(uint32_t(last >> 32)), unscale);
        }
        tc[j] = t;
        tl[j] = l;
    }
}

// Per row: the kTriSel smallest column-side candidates (by rank, unordered)
// and the bound for everything else -- min(threshold, the next key) -- so the
// rescore handles a short fixed-size list.  An overflowed buffer is passed on
// as a count above kTriSel (no proof).
constexpr int kTriSel = 32;
// units (sharded triangle, or null): slot `row` is sorted position
// units[row / 256] * 256 + row % 256, whose threshold is thr[that position].
__global__ void __launch_bounds__(256) tri_select_kernel(const uint64_t* __restrict__ buf, const uint32_t* __restrict__ cnt,
                                                          uint32_t cap, uint32_t n, const float* __restrict__ thr,
                                                          uint64_t* __restrict__ out, uint32_t* __restrict__ out_cnt,
                                                          float* __restrict__ out_bound,
                                                          const uint32_t* __restrict__ units = nullptr) {
    __shared__ __align__(16) uint64_t ks[8][kTriCap + 2];
    const uint32_t row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (row >= n) return;
    const uint32_t c = cnt[row];
    const uint32_t m = c < cap ? c : cap;
    uint64_t* o = out + size_t(row) * kTriSel;
    uint64_t next = kEmptyKey;  // the (kTriSel+1)-th smallest
    if (m <= uint32_t(kTriSel)) {
        for (uint32_t i = lane; i < m; i += 32) o[i] = buf[size_t(row) * cap + i];
    } else {
        // a key's rank among the m (ties by position; keys are unique in
        // practice -- one entry per row of the column) is its output slot
        for (uint32_t i = lane; i < m; i += 32) ks[w][i] = buf[size_t(row) * cap + i];
        if (lane == 0) ks[w][m] = kEmptyKey;  // pad to an even count
        __syncwarp();
        const uint32_t m2 = (m + 1) & ~1u;
        for (uint32_t i = lane; i < m; i += 32) {
            const uint64_t key = ks[w][i];
            uint32_t r = 0;
            for (uint32_t j = 0; j < m2; j += 2) {
                const ulonglong2 two = *reinterpret_cast<const ulonglong2*>(&ks[w][j]);
                r += (two.x < key || (two.x == key && j < i)) + (two.y < key || (two.y == key && j + 1 < i));
            }
            if (r < uint32_t(kTriSel)) o[r] = key;
            else if (r == uint32_t(kTriSel)) next = key;
        }
        for (int s = 16; s; s >>= 1) {
            const uint64_t other = __shfl_xor_sync(0xffffffffu, next, s);
            next = other < next ? other : next;
        }
    }
    if (lane == 0) {
        float b = thr[units ? units[row >> 8] * 256 + (row & 255) : row];
        if (next != kEmptyKey) {
            const float nb = ordered_to_float(uint32_t(next >> 32));
            b = nb < b ? nb : b;
        }
        out_bound[row] = b;
        out_cnt[row] = c > cap ? uint32_t(kTriSel) + 1 : (m < uint32_t(kTriSel) ? m : uint32_t(kTriSel));
    }
}

// Second order for the triangle sweep: within consecutive buckets of the
// norm order, sort by column-side threshold, so each 32-column chunk has
// nearly equal norms (row-side bound) and nearly equal thresholds
// (column-side bound).
__global__ void tri_order_key_kernel(const float* __restrict__ tc, uint32_t n, uint32_t bucket,
                                     unsigned long long* __restrict__ key, uint32_t* __restrict__ idx) {
    for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
        key[p] = (uint64_t(p / bucket) << 32) | float_to_ordered(tc[p]);
        idx[p] = p;
    }
}

// Per-row arrays into the new order (position k holds old position order[k]).
__global__ void tri_permute_kernel(const uint32_t* __restrict__ order, uint32_t n, uint32_t npad,
                                   const float* __restrict__ alpha, const double* __restrict__ rho,
                                   const double* __restrict__ xnorm, const float* __restrict__ tc,
                                   const float* __restrict__ tl, const uint32_t* __restrict__ perm,
                                   float* __restrict__ alpha2, double* __restrict__ rho2, double* __restrict__ xnorm2,
                                   float* __restrict__ tc2, float* __restrict__ tl2, uint32_t* __restrict__ perm2) {
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < npad; k += gridDim.x * blockDim.x) {
        const uint32_t q = k < n ? order[k] : k;
        alpha2[k] = alpha[q];
        rho2[k] = rho[q];
        xnorm2[k] = xnorm[q];
        tc2[k] = tc[q];
        tl2[k] = tl[q];
        if (k < n) perm2[k] = perm[q];
    }
}

// Bin the sweep's column-side pool by column (one block per chunk); a pool
// that overflowed raises *overflow (the host then redoes the call without
// the triangle).
__global__ void tri_scatter_kernel(const uint64_t* __restrict__ lkey, const uint32_t* __restrict__ lcol,
                                   const uint32_t* __restrict__ lcnt, const uint32_t* __restrict__ lnext,
                                   uint32_t nchunks, uint32_t* __restrict__ ccnt, uint64_t* __restrict__ cbuf,
                                   uint32_t ccap, unsigned int* __restrict__ overflow) {
    const uint32_t w = blockIdx.x;
    const uint32_t used = *lnext;
    if (w == 0 && threadIdx.x == 0 && used > nchunks) atomicOr(overflow, 1u);
    if (w >= min(used, nchunks)) return;
    const uint32_t c = lcnt[w];
    const size_t base = size_t(w) * kLogChunk;
    for (uint32_t i = threadIdx.x; i < c; i += blockDim.x) {
        const uint32_t col = lcol[base + i];
        const uint32_t at = atomicAdd(ccnt + col, 1u);
        if (at < ccap) cbuf[size_t(col) * ccap + at] = lkey[base + i];
    }
}

__global__ void chunk_max_kernel(const float* __restrict__ v, uint32_t nchunks, float* __restrict__ out) {
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (warp >= nchunks) return;
    float m = v[size_t(warp) * 32 + lane];
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) {
        out[warp] = m;
        out[nchunks + warp] = bound_half(m, -1.0f);  // the column bound's per-chunk half
    }
}

// bmin[c] = smallest alpha of columns [32c, 32c + 32) (the sweep's hot-path
// bound), bmin[nchunks + c] = its bound_half (the row bound's per-chunk half)
__global__ void chunk_min_kernel(const float* __restrict__ alpha, uint32_t nchunks, float* __restrict__ bmin) {
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (warp >= nchunks) return;
    float m = alpha[size_t(warp) * 32 + lane];
    for (int o = 16; o; o >>= 1) m = fminf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) {
        bmin[warp] = m;
        bmin[nchunks + warp] = bound_half(m, 1.0f);
    }
}

__device__ __forceinline__ void atomic_max_pos_double(unsigned long long* addr, double v) {
    // non-negative doubles order like their bit patterns
    atomicMax(addr, (unsigned long long)__double_as_longlong(v));
}

// Column sums in double -> mu (any mu is correct: distances are translation
// invariant; mu only shrinks the magnitudes the fp16 filter sees).
__global__ void colsum_kernel(const float* __restrict__ X, uint32_t n, uint32_t d, double* __restrict__ acc) {
    // a block's row range, one thread per column; 8 independent partial sums
    // keep 8 loads in flight per thread (the loop was latency-bound at 1/4
    // of HBM bandwidth)
    const uint32_t rows_per = (n + gridDim.x - 1) / gridDim.x;
    const uint32_t ra = blockIdx.x * rows_per;
    const uint32_t rb = min(n, ra + rows_per);
    for (uint32_t j = threadIdx.x; j < d; j += blockDim.x) {
        double s[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        uint32_t r = ra;
        for (; r + 8 <= rb; r += 8) {
            float v[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) v[q] = __ldg(X + size_t(r + q) * d + j);
#pragma unroll
            for (int q = 0; q < 8; ++q) s[q] += v[q];
        }
        for (; r < rb; ++r) s[0] += __ldg(X + size_t(r) * d + j);
        const double t = ((s[0] + s[1]) + (s[2] + s[3])) + ((s[4] + s[5]) + (s[6] + s[7]));
        if (ra < rb) atomicAdd(acc + j, t);
    }
}

// The same sums over every rstep-th row, float4 loads (d % 4 == 0, d <= 1024,
// X 16-byte aligned): thread t owns column quad t % (d/4) of row lane
// t / (d/4); 4 rows in flight per thread; the row lanes are reduced in shared
// memory, then one double atomic per column and block.  A strided sample of
// >= 65,536 rows puts mu within a fraction of a percent of a coordinate's
// spread from the full mean -- the same conditioning for 1/rstep of the reads.
__global__ void __launch_bounds__(256) colsum4_kernel(const float* __restrict__ X, uint32_t n, uint32_t d,
                                                      uint32_t rstep, double* __restrict__ acc) {
    __shared__ double part[256][4];
    const uint32_t c4 = d >> 2, lanes = 256 / c4;
    const uint32_t t = threadIdx.x, col = t % c4, rl = t / c4;
    const uint32_t m = (n + rstep - 1) / rstep;  // sampled rows 0, rstep, 2 rstep, ...
    double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
    if (rl < lanes) {
        const float4* X4 = reinterpret_cast<const float4*>(X) + col;
        const size_t rs = size_t(rstep) * c4;  // float4s between sampled rows
        const uint32_t step = gridDim.x * lanes;
        uint32_t i = blockIdx.x * lanes + rl;
        for (; i + 3 * step < m; i += 4 * step) {
            float4 v[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) v[q] = __ldg(X4 + size_t(i + q * step) * rs);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                s0 += v[q].x;
                s1 += v[q].y;
                s2 += v[q].z;
                s3 += v[q].w;
            }
        }
        for (; i < m; i += step) {
            const float4 v = __ldg(X4 + size_t(i) * rs);
            s0 += v.x;
            s1 += v.y;
            s2 += v.z;
            s3 += v.w;
        }
    }
    part[t][0] = s0;
    part[t][1] = s1;
    part[t][2] = s2;
    part[t][3] = s3;
    __syncthreads();
    if (t < c4) {
        double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
        for (uint32_t l = 0; l < lanes; ++l) {
            a0 += part[l * c4 + t][0];
            a1 += part[l * c4 + t][1];
            a2 += part[l * c4 + t][2];
            a3 += part[l * c4 + t][3];
        }
        atomicAdd(acc + 4 * t, a0);
        atomicAdd(acc + 4 * t + 1, a1);
        atomicAdd(acc + 4 * t + 2, a2);
        atomicAdd(acc + 4 * t + 3, a3);
    }
}

__global__ void mu_finalize_kernel(const double* __restrict__ acc, uint32_t count, uint32_t d, float* __restrict__ mu) {
    for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < d; j += gridDim.x * blockDim.x)
        mu[j] = float(acc[j] / double(count));
}

// Whether X's rows can be read as float4 quads.
static inline int vec4_rows(const float* X, uint32_t d) {
    return d % 4 == 0 && (reinterpret_cast<uintptr_t>(X) & 15u) == 0;
}

// mu for the centring: column means over a strided row sample (every
// rstep-th row, rstep = n / 65,536 capped at 16) through the float4 kernel,
// or every row through the scalar one.  acc must be zeroed.
static void launch_colmean(const float* X, uint32_t n, uint32_t d, double* acc, float* mu, int sm_count,
                           cudaStream_t st) {
    const bool vec = d % 4 == 0 && d <= 1024 && (reinterpret_cast<uintptr_t>(X) & 15u) == 0;
    if (vec) {
        const uint32_t rstep = std::max<uint32_t>(1, std::min<uint32_t>(16, n / 65536));
        colsum4_kernel<<<sm_count * 4, 256, 0, st>>>(X, n, d, rstep, acc);
        mu_finalize_kernel<<<(d + 255) / 256, 256, 0, st>>>(acc, (n + rstep - 1) / rstep, d, mu);
    } else {
        colsum_kernel<<<sm_count * 4, 256, 0, st>>>(X, n, d, acc);
        mu_finalize_kernel<<<(d + 255) / 256, 256, 0, st>>>(acc, n, d, mu);
    }
}


// One pass over X (one warp per row): the largest |x - mu| (one atomic per
// block; it sets the fp16 scale) and, with key != null, each row's
// ||x - mu||^2 -- the norm order's sort key (any order is correct; this one
// makes every 32-column chunk's norms nearly equal, so the sweep's hot-path
// bound, which uses the chunk's smallest norm, is nearly exact).
__global__ void __launch_bounds__(256) center_stats_kernel(const float* __restrict__ X, uint32_t n, uint32_t d,
                                                           const float* __restrict__ mu, unsigned int* __restrict__ out,
                                                           float* __restrict__ key, uint32_t* __restrict__ idx,
                                                           int vec) {
    __shared__ float wmax[8];
    const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    float m = 0.0f;
    for (uint32_t row = blockIdx.x * 8 + w; row < n; row += gridDim.x * 8) {
        const float* xr = X + size_t(row) * d;
        float sq = 0.0f;
        if (vec) {  // float4 quads, two loads in flight per lane (d % 4 == 0, 16-byte rows)
            const float4* x4 = reinterpret_cast<const float4*>(xr);
            const float4* m4 = reinterpret_cast<const float4*>(mu);
            const uint32_t q4 = d >> 2;
            for (uint32_t u = lane; u < q4; u += 64) {
                const bool two = u + 32 < q4;
                const float4 a = __ldg(x4 + u), ma = __ldg(m4 + u);
                const float4 b = two ? __ldg(x4 + u + 32) : make_float4(0.f, 0.f, 0.f, 0.f);
                const float4 mb = two ? __ldg(m4 + u + 32) : make_float4(0.f, 0.f, 0.f, 0.f);
                const float v[8] = {__fsub_rn(a.x, ma.x), __fsub_rn(a.y, ma.y), __fsub_rn(a.z, ma.z),
                                    __fsub_rn(a.w, ma.w), __fsub_rn(b.x, mb.x), __fsub_rn(b.y, mb.y),
                                    __fsub_rn(b.z, mb.z), __fsub_rn(b.w, mb.w)};
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    m = fmaxf(m, fabsf(v[q]));
                    sq = __fadd_rn(sq, __fmul_rn(v[q], v[q]));
                }
            }
        } else {
            for (uint32_t k = lane; k < d; k += 32) {
                const float v = __fsub_rn(__ldg(xr + k), __ldg(mu + k));
                m = fmaxf(m, fabsf(v));
                sq = __fadd_rn(sq, __fmul_rn(v, v));
            }
        }
        if (key) {
            for (int o = 16; o; o >>= 1) sq = __fadd_rn(sq, __shfl_xor_sync(0xffffffffu, sq, o));
            if (lane == 0) {
                key[row] = sq;
                idx[row] = row;
            }
        }
    }
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) wmax[w] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        float b = 0.0f;
        for (int i = 0; i < 8; ++i) b = fmaxf(b, wmax[i]);
        atomicMax(out, __float_as_uint(b));
    }
}

// Power-of-two scale with |s x| <= 65504 (fp16 max), capped at 2^40.
__device__ __forceinline__ int scale_exponent(unsigned int maxabs_bits) {
    const float m = __uint_as_float(maxabs_bits);
    if (!(m > 0.0f)) return 0;
    int p;
    frexp(65504.0 / double(m), &p);  // 65504/m = f * 2^p, f in [0.5, 1)
    int e = p - 1;
    return e > 40 ? 40 : e;
}

struct PrepOut {
    uint8_t* xh;
    float* alpha;
    double* rho;
    double* xnorm;
    unsigned long long* gmax;  // [0] max xnorm, [1] max rho, [2] max alpha
};

// One warp per (padded) row, grid-stride: each lane converts 8 consecutive
// coordinates into one 16-byte unit of the swizzled planes (a full-unit
// store); the three global maxima are reduced per block, then one atomic each.
__global__ void __launch_bounds__(256) prep_kernel(const float* __restrict__ X, uint32_t n, uint32_t d, uint32_t npad,
                                                   uint32_t kc, const float* __restrict__ mu,
                                                   const unsigned int* __restrict__ maxabs, int cosine,
                                                   const uint32_t* __restrict__ perm, PrepOut o) {
    __shared__ double bmax[8][3];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int e = scale_exponent(*maxabs);
    const float s = ldexpf(1.0f, e);
    const double sd = ldexp(1.0, e);
    double mx_xn = 0.0, mx_rho = 0.0, mx_a = 0.0;
    for (uint32_t row = blockIdx.x * 8 + w; row < npad; row += gridDim.x * 8) {
        double rho2 = 0, nrm2 = 0;
        float alpha = 0.0f;
        const float* xr = X + size_t(row < n ? (perm ? perm[row] : row) : 0) * d;
        for (uint32_t u = lane; u < kc * 8; u += 32) {
            const uint32_t k0 = u * 8;
            uint32_t wd[4];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const uint32_t k = k0 + q;
                __half h = __float2half_rn(0.0f);
                if (row < n && k < d) {
                    const float x = xr[k];
                    const float m = cosine ? 0.0f : mu[k];
                    const float v = __fsub_rn(x, m);
                    h = __float2half_rn(__fmul_rn(v, s));
                    const double hv = double(__half2float(h));
                    const double exact = (double(x) - double(m)) * sd;
                    rho2 += (hv - exact) * (hv - exact);
                    nrm2 += hv * hv;
                    const float hf = __half2float(h);
                    alpha = __fadd_rn(alpha, __fmul_rn(hf, hf));
                }
                const uint32_t hb = __half_as_ushort(h);
                if (q & 1) wd[q >> 1] |= hb << 16;
                else wd[q >> 1] = hb;
            }
            const uint32_t chunk = k0 >> 6, unit = (k0 & 63) >> 3;
            *reinterpret_cast<uint4*>(o.xh + (size_t(chunk) * npad + row) * 128 + ((unit ^ (row & 7)) << 4)) =
                make_uint4(wd[0], wd[1], wd[2], wd[3]);
        }
        for (int of = 16; of; of >>= 1) {
            rho2 += __shfl_xor_sync(0xffffffffu, rho2, of);
            nrm2 += __shfl_xor_sync(0xffffffffu, nrm2, of);
            alpha = __fadd_rn(alpha, __shfl_xor_sync(0xffffffffu, alpha, of));
        }
        if (lane == 0) {
            if (row < n) {
                const float a = cosine ? __fmul_rn(s, s) : alpha;
                o.alpha[row] = a;
                const double rho = sqrt(rho2) * (1.0 + 1e-12);
                const double xn = sqrt(nrm2) * (1.0 + 1e-12);
                o.rho[row] = rho;
                o.xnorm[row] = xn;
                mx_xn = fmax(mx_xn, xn);
                mx_rho = fmax(mx_rho, rho);
                mx_a = fmax(mx_a, double(a));
            } else {
                o.alpha[row] = __int_as_float(0x7f800000);
            }
        }
    }
    if (lane == 0) {
        bmax[w][0] = mx_xn;
        bmax[w][1] = mx_rho;
        bmax[w][2] = mx_a;
    }
    __syncthreads();
    if (threadIdx.x < 3) {
        double m = 0.0;
        for (int i = 0; i < 8; ++i) m = fmax(m, bmax[i][threadIdx.x]);
        atomic_max_pos_double(o.gmax + threadIdx.x, m);
    }
}

// ---------------------------------------------------------------------------
// exact re-score + proof of completeness

struct RescoreParams {
    const float* X;       // fp32 (sqrt-staged for Hellinger)
    uint32_t n, d, klist, kp;
    uint32_t row_begin, row_end;
    const uint64_t* cand;
    const float* alpha;
    const double* rho;
    const double* xnorm;
    const unsigned long long* gmax;
    const unsigned int* maxabs;
    int fold;             // kSqEuclidean or kCosine
    int out_sqrt;
    uint32_t* out_index;
    float* out_dist;
    uint32_t* fb_count;
    uint32_t* fb_rows;
    float* fb_thr;        // capture threshold (y space) for each unproven row
    unsigned long long* rescored;
    int force_capture;    // testing: treat every row as unproven (KNN_B200_FORCE_CAPTURE=1)
    const uint32_t* rowpos;  // norm-sorted columns: input row q sits at position rowpos[q] of alpha/rho/xnorm (or null)
    const uint32_t* rowperm;  // triangle sweep: slot s is sorted position s, input row rowperm[s] (or null)
    const uint64_t* xbuf;     // [slots][XC] extra candidates (column side of the triangle sweep)
    const uint32_t* xcnt;     // [slots] their counts (> XC: overflowed)
    const float* xbound;      // [slots] y bound of the column side's exclusions
    const float* xcap;        // [sorted positions] capture threshold (y) for rows left with fewer than k candidates, or null
    const uint32_t* units;    // sharded triangle: slot s is sorted position units[s / 256] * 256 + s % 256 (or null)
};

constexpr double kTcSafety = 4.0;  // tensor-core accumulation error allowance

template <int FOLD>
__device__ __forceinline__ float exact_fold_rows(const float* __restrict__ a, const float* __restrict__ b, uint32_t d,
                                                 bool vec) {
    // The fold is strictly sequential over coordinates (bit parity); the
    // loads are batched 8 float4 deep so the random row reads overlap.
    float acc = 0.0f;
    if (vec) {
        const float4* a4 = reinterpret_cast<const float4*>(a);
        const float4* b4 = reinterpret_cast<const float4*>(b);
        const uint32_t d4 = d / 4;
        uint32_t j = 0;
        for (; j + 8 <= d4; j += 8) {
            float4 x[8], y[8];
#pragma unroll
            for (int t = 0; t < 8; ++t) {
                x[t] = __ldg(a4 + j + t);
                y[t] = __ldg(b4 + j + t);
            }
#pragma unroll
            for (int t = 0; t < 8; ++t) {
                acc = fold_step_x2<FOLD>(x[t].x, x[t].y, y[t].x, y[t].y, acc);
                acc = fold_step_x2<FOLD>(x[t].z, x[t].w, y[t].z, y[t].w, acc);
            }
        }
        for (; j < d4; ++j) {
            const float4 x = __ldg(a4 + j), y = __ldg(b4 + j);
            acc = fold_step_x2<FOLD>(x.x, x.y, y.x, y.y, acc);
            acc = fold_step_x2<FOLD>(x.z, x.w, y.z, y.w, acc);
        }
    } else {
        for (uint32_t j = 0; j < d; ++j) acc = fold_step<FOLD>(__ldg(a + j), __ldg(b + j), acc);
    }
    return fold_finalize<FOLD>(acc);
}

// The same fold with the query row staged in shared memory (d % 4 == 0): the
// candidate row streams through a two-deep pipeline of 8-float4 batches, so
// a batch's loads are in flight while the previous batch folds.  The fold is
// symmetric in its operands bit for bit ((u-v)^2, u*v).
constexpr uint32_t kStagedMaxD = 256;
template <int FOLD>
__device__ __forceinline__ float exact_fold_staged(const float* __restrict__ c, const float* q, uint32_t d) {
    const float4* c4 = reinterpret_cast<const float4*>(c);
    const float4* q4 = reinterpret_cast<const float4*>(q);
    const uint32_t d4 = d / 4;
    float acc = 0.0f;
    float4 cur[8], nxt[8];
#pragma unroll
    for (int t = 0; t < 8; ++t)
        if (uint32_t(t) < d4) cur[t] = __ldg(c4 + t);
    for (uint32_t j = 0; j < d4; j += 8) {
#pragma unroll
        for (int t = 0; t < 8; ++t)
            if (j + 8 + t < d4) nxt[t] = __ldg(c4 + j + 8 + t);
#pragma unroll
        for (int t = 0; t < 8; ++t) {
            if (j + t < d4) {
                const float4 y = q4[j + t];
                acc = fold_step_x2<FOLD>(cur[t].x, cur[t].y, y.x, y.y, acc);
                acc = fold_step_x2<FOLD>(cur[t].z, cur[t].w, y.z, y.w, acc);
            }
        }
#pragma unroll
        for (int t = 0; t < 8; ++t) cur[t] = nxt[t];
    }
    return fold_finalize<FOLD>(acc);
}

// Upper bound (scaled A space) on the approximate distance of any column whose
// exact reference distance is <= T: s^2 T' + 2E, DESIGN.md §4.
template <int FOLD>
__device__ __forceinline__ double proof_bound(uint32_t d, const unsigned int* maxabs, const unsigned long long* gmax,
                                              double nx, double rh, double al, double T) {
    const double u = 5.9604644775390625e-08;  // 2^-24
    const double dd = double(d);
    const int e = scale_exponent(*maxabs);
    const double s2 = ldexp(1.0, 2 * e);
    const double xnmax = __longlong_as_double((long long)gmax[0]);
    const double rhomax = __longlong_as_double((long long)gmax[1]);
    const double alphamax = __longlong_as_double((long long)gmax[2]);
    const double Tp = T + fabs(T) * 2.0 * (dd + 3.0) * u + 1e-300;
    const double ctc = 2.0 * kTcSafety * dd * 2.0 * u;  // 2 * c * d * 2^-23
    if (FOLD == kCosine) {
        const double eref = (dd + 2.0) * u * ((nx + rh) * (xnmax + rhomax) / s2 + 1.0);
        const double eacc = ctc * nx * xnmax + 2.0 * (rh * xnmax + rhomax * (nx + rh)) + u * 2.0 * s2 * (fabs(Tp) + 2.0);
        return 2.0 * s2 * (Tp + 2.0 * eref) + 2.0 * eacc;
    }
    // The bound only has to hold for columns j with D_ref(i, j) <= T, and
    // those lie near row i: ||s(x_j - mu)|| <= ||x^_i|| + rho_i + s sqrt(T')
    // =: X0 (triangle inequality), so their quantisation error is
    // rho_j <= 2^-11 (1 + eps) X0 + sqrt(d) 2^-25 (fp16 rounding, relative in
    // the normal range, absolute for subnormals), ||x^_j|| <= X0 + rho_j and
    // alpha_j <= ||x^_j||^2 (1 + (d + 2) u).  Each replaces the dataset-wide
    // maximum when smaller -- so one outlier row no longer widens every other
    // row's band.
    const double sqT = sqrt(s2 * fmax(Tp, 0.0));
    const double X0 = nx + rh + sqT;
    const double rho_b = 4.8828125e-04 * (1.0 + 1e-3) * X0 + sqrt(dd) * 2.98023223876953125e-08;
    const double xn_j = fmin(xnmax, X0 + rho_b);
    const double rho_j = fmin(rhomax, rho_b);
    const double al_j = fmin(alphamax, xn_j * xn_j * (1.0 + (dd + 2.0) * u));
    const double rr = rh + rho_j;
    const double e_all = (ctc + 6.0 * u) * nx * xn_j + (dd + 3.0) * u * (al + al_j) + rr * (2.0 * sqT + rr);
    return s2 * Tp + 2.0 * e_all;
}

// Warp-wide minimum of unique 64-bit keys: two redux.sync on the halves
// instead of five 64-bit shuffle rounds.
__device__ __forceinline__ uint64_t warp_min_key(uint64_t k) {
    const uint32_t hi = __reduce_min_sync(0xffffffffu, uint32_t(k >> 32));
    const uint32_t lo = __reduce_min_sync(0xffffffffu, uint32_t(k >> 32) == hi ? uint32_t(k) : 0xffffffffu);
    return (uint64_t(hi) << 32) | lo;
}
__device__ __forceinline__ uint64_t warp_max_key(uint64_t k) {
    const uint32_t hi = __reduce_max_sync(0xffffffffu, uint32_t(k >> 32));
    const uint32_t lo = __reduce_max_sync(0xffffffffu, uint32_t(k >> 32) == hi ? uint32_t(k) : 0u);
    return (uint64_t(hi) << 32) | lo;
}

// XC > 0: up to XC extra candidates per row (the triangle sweep's column side,
// p.xbuf/p.xcnt) whose exclusions are bounded by p.xbound[slot].
template <int FOLD, int KP, int NSEG, int XC = 0>
__global__ void __launch_bounds__(256) rescore_kernel(const RescoreParams p) {
    constexpr int KPL = KP / NSEG;
    constexpr int KT = KP + XC;  // candidates per row
    __shared__ uint64_t keys_s[8][KT];
    __shared__ uint64_t ak_s[8][KT];   // approximate keys
    __shared__ uint64_t ex_s[8][KT];   // exact keys of a batch
    __shared__ uint16_t todo_s[8][KT];  // a batch's candidate slots
    __shared__ __align__(16) float xq_s[8][kStagedMaxD];  // the query row (d <= kStagedMaxD, d % 4 == 0)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t slot = blockIdx.x * 8 + warp;
    if (slot >= p.row_end - p.row_begin) return;
    // slot: input order, or (p.rowperm) a position in the sorted order, or
    // (p.units) a row of this rank's units
    const uint32_t sp = p.units ? p.units[slot >> 8] * 256 + (slot & 255) : slot;
    if (p.units && sp >= p.n) return;  // padding rows of the last unit
    const uint32_t qo = p.rowperm ? p.rowperm[sp] : p.row_begin + slot;  // input row
    const uint32_t q = p.rowperm ? sp : (p.rowpos ? p.rowpos[qo] : qo);  // its sorted position
    const uint64_t* cand = p.cand + size_t(slot) * KP;
    const float* xq = p.X + size_t(qo) * p.d;
    const bool vec = (p.d % 4 == 0);
    const bool staged = vec && p.d <= kStagedMaxD;
    if (staged)
        for (uint32_t i = lane; i < p.d; i += 32) xq_s[warp][i] = __ldg(xq + i);
    constexpr int PER = (KT + 31) / 32;
    const uint32_t xn = XC ? p.xcnt[slot] : 0;
    const uint64_t* xb = XC ? p.xbuf + size_t(slot) * XC : nullptr;
    const double alpha_q = double(p.alpha[q]);
    // approximate keys (unique: distinct columns)
    uint64_t ak[PER];
#pragma unroll
    for (int m = 0; m < PER; ++m) {
        const int i = lane + 32 * m;
        if constexpr (XC > 0) ak[m] = i < KP ? cand[i] : (i < KT && uint32_t(i - KP) < xn ? xb[i - KP] : kEmptyKey);
        else ak[m] = i < KP ? cand[i] : kEmptyKey;
        if (uint32_t(ak[m]) == kVirtualIdx) ak[m] = kEmptyKey;  // a bound, not a candidate (segmax reads cand[])
        if (i < KT) keys_s[warp][i] = ak[m];
    }
    __syncwarp();
    __syncwarp();
#pragma unroll
    for (int m = 0; m < PER; ++m)
        if (lane + 32 * m < KT) ak_s[warp][lane + 32 * m] = ak[m];
    // exact fold of a batch of candidates: the wanted (lane, m) slots are
    // compacted onto consecutive lanes, so a batch is one fold stream
    uint64_t ek[PER];
    bool done[PER];
    uint32_t valid = 0;
    auto rescore_batch = [&](const bool (&want)[PER]) {
        uint32_t cnt = 0;
#pragma unroll
        for (int m = 0; m < PER; ++m) {
            const uint32_t b = __ballot_sync(0xffffffffu, want[m]);
            if (want[m]) todo_s[warp][cnt + __popc(b & ((1u << lane) - 1u))] = uint16_t(lane + 32 * m);
            cnt += __popc(b);
        }
        __syncwarp();
        for (uint32_t t = lane; t < cnt; t += 32) {
            const int i = todo_s[warp][t];
            const uint64_t a = ak_s[warp][i];
            const uint32_t col = uint32_t(a);  // input order (remap_kernel)
            uint64_t key = kEmptyKey;
            if (a != kEmptyKey && col != qo) {
                const float* xc = p.X + size_t(col) * p.d;
                // Reference argument order (larger index first) -- the fold is
                // symmetric bit for bit, kept for clarity.
                const float dist = staged ? exact_fold_staged<FOLD>(xc, xq_s[warp], p.d)
                                   : col > qo ? exact_fold_rows<FOLD>(xc, xq, p.d, vec)
                                              : exact_fold_rows<FOLD>(xq, xc, p.d, vec);
                key = make_key(dist, col);
                ++valid;
            }
            ex_s[warp][i] = key;
        }
        __syncwarp();
#pragma unroll
        for (int m = 0; m < PER; ++m)
            if (want[m]) {
                ek[m] = ex_s[warp][lane + 32 * m];
                done[m] = true;
            }
        __syncwarp();
    };
    // the computed exact keys compacted to keys_s[warp][0, c) (the rank
    // loops below run over those only, not over all KA candidates)
    int cpos[PER];  // each computed key's position in the compact array
    auto compact_exact = [&]() -> int {
        __syncwarp();
        int c = 0;
#pragma unroll
        for (int m = 0; m < PER; ++m) {
            const bool h = lane + 32 * m < KT && done[m] && ek[m] != kEmptyKey;
            const uint32_t b = __ballot_sync(0xffffffffu, h);
            cpos[m] = c + __popc(b & ((1u << lane) - 1u));
            if (h) keys_s[warp][cpos[m]] = ek[m];
            c += __popc(b);
        }
        __syncwarp();
        return c;
    };
    auto kth_exact = [&]() -> uint64_t {  // klist-th smallest exact key among the computed ones
        const int c = compact_exact();
        uint64_t kth = kEmptyKey;
#pragma unroll
        for (int m = 0; m < PER; ++m) {
            if (lane + 32 * m >= KT || !done[m] || ek[m] == kEmptyKey) continue;
            uint32_t r = 0;
            for (int j = 0; j < c; ++j) r += keys_s[warp][j] < ek[m];
            if (r == p.klist - 1) kth = ek[m];
        }
        return warp_min_key(kth);
    };
    // Phase 1: the k + 4 best candidates by approximate distance -- those
    // with fewer than k + 4 smaller keys (keys are unique: distinct columns).
    // Every lane ranks its own keys against the row's keys in shared memory:
    // independent compares, where k + 4 rounds of a warp-wide minimum were a
    // chain of k + 4 dependent shuffle reductions.
    const uint32_t r1 = p.klist + 4 < uint32_t(KT) ? p.klist + 4 : uint32_t(KT);
    bool sel[PER];
    {
        uint32_t rk[PER];
#pragma unroll
        for (int m = 0; m < PER; ++m) rk[m] = 0;
        for (int j = 0; j < KT; ++j) {
            const uint64_t o = keys_s[warp][j];
#pragma unroll
            for (int m = 0; m < PER; ++m) rk[m] += o < ak[m];
        }
#pragma unroll
        for (int m = 0; m < PER; ++m) sel[m] = lane + 32 * m < KT && ak[m] != kEmptyKey && rk[m] < r1;
    }
#pragma unroll
    for (int m = 0; m < PER; ++m) {
        done[m] = false;
        ek[m] = kEmptyKey;
    }
    rescore_batch(sel);
    // Phase 2: any other candidate whose approximate distance is inside the
    // bound implied by phase 1's k-th exact distance (those beyond cannot be
    // among the k nearest); everything when no bound exists.
    {
        const uint64_t kth1 = kth_exact();
        double lim = __longlong_as_double(0x7ff0000000000000ll);
        if (kth1 != kEmptyKey)
            lim = proof_bound<FOLD>(p.d, p.maxabs, p.gmax, p.xnorm[q], p.rho[q], alpha_q,
                                    double(ordered_to_float(uint32_t(kth1 >> 32))));
        bool want[PER], wany = false;
#pragma unroll
        for (int m = 0; m < PER; ++m) {
            want[m] = false;
            if (lane + 32 * m >= KT || done[m]) continue;
            const double a = alpha_q + double(ordered_to_float(uint32_t(ak[m] >> 32)));
            if (ak[m] != kEmptyKey && a <= lim) want[m] = true;
            else done[m] = true;  // excluded: stays empty
            wany |= want[m];
        }
        if (__any_sync(0xffffffffu, wany)) rescore_batch(want);
    }
    for (int o = 16; o; o >>= 1) valid += __shfl_xor_sync(0xffffffffu, valid, o);
    if (lane == 0) atomicAdd(p.rescored, (unsigned long long)valid);
    // final order of the exact keys
    uint64_t mine[PER];
    uint32_t rank[PER];
#pragma unroll
    for (int m = 0; m < PER; ++m) {
        mine[m] = lane + 32 * m < KT ? ek[m] : kEmptyKey;
        rank[m] = 0;
    }
    // ranks of the computed keys only (empty entries are never output)
    const int ncomp = compact_exact();
#pragma unroll
    for (int m = 0; m < PER; ++m) {
        if (mine[m] == kEmptyKey) continue;
        for (int j = 0; j < ncomp; ++j) {
            const uint64_t o = keys_s[warp][j];
            rank[m] += (o < mine[m]) || (o == mine[m] && j < cpos[m]);
        }
    }
    __syncwarp();
#pragma unroll
    for (int m = 0; m < PER; ++m)
        if (lane + 32 * m < KT && mine[m] != kEmptyKey) keys_s[warp][rank[m]] = mine[m];
    __syncwarp();
    // Each of the NSEG lists is unsorted; per list its largest key.  A list
    // holding an empty slot saw (and kept) every column of its segment, so
    // it excludes nothing; a full list excludes only columns with y >= its
    // maximum.  The bound for everything excluded is the smallest such
    // maximum over the full lists.
    uint64_t segmax[NSEG];
#pragma unroll
    for (int s = 0; s < NSEG; ++s) segmax[s] = 0;
#pragma unroll
    for (int m = 0; m < PER; ++m) {
        const int i = lane + 32 * m;
        if (i < KP) {
            const uint64_t c = cand[i];
#pragma unroll
            for (int s = 0; s < NSEG; ++s)
                if (i / KPL == s) segmax[s] = c > segmax[s] ? c : segmax[s];
        }
    }
    bool any_full = false;
    uint64_t last_approx = kEmptyKey;  // smallest maximum over full lists
#pragma unroll
    for (int s = 0; s < NSEG; ++s) {
        segmax[s] = warp_max_key(segmax[s]);
        if (segmax[s] != kEmptyKey) {
            any_full = true;
            last_approx = segmax[s] < last_approx ? segmax[s] : last_approx;
        }
    }
    bool x_overflow = false;
    if constexpr (XC > 0) {
        // the column side excluded only candidates with y >= xbound; a buffer
        // that overflowed lost candidates -- no proof for this row
        const float xbnd = p.xbound[slot];
        if (xbnd < __int_as_float(0x7f800000)) {
            const uint64_t xk = make_key(xbnd, 0u);
            any_full = true;
            last_approx = xk < last_approx ? xk : last_approx;
        }
        x_overflow = xn > uint32_t(XC);
    }
    bool complete;
    // no band (fewer than k candidates computed): p.xcap's looser threshold
    // when there is one (rescore_capture_kernel proves or rejects it), else
    // -inf, which captures nothing: the row goes to the EXACT kernel
    double cap_y = -__longlong_as_double(0x7ff0000000000000ll);
    if (!any_full && !x_overflow) {
        complete = true;  // every column was offered into a non-full list: the list holds all of them
    } else if (valid < p.klist) {
        complete = false;
        if (XC > 0 && p.xcap) cap_y = double(p.xcap[q]);
    } else {
        const uint64_t kth = keys_s[warp][p.klist - 1];
        const double T = double(ordered_to_float(uint32_t(kth >> 32)));
        // the list ranks y = fl(beta - 2 dot); A = alpha_q + y exactly in fp64
        const double a_max = double(p.alpha[q]) + double(ordered_to_float(uint32_t(last_approx >> 32)));
        const double bound = proof_bound<FOLD>(p.d, p.maxabs, p.gmax, p.xnorm[q], p.rho[q], double(p.alpha[q]), T);
        // (an overflowed column-side buffer lost candidates: no proof, but T
        // is still an upper bound on the k-th distance, so the band holds)
        complete = a_max > bound && !p.force_capture && !x_overflow;
        // every true neighbor has A <= bound, i.e. y <= bound - alpha_q: the
        // second (band-capture) pass collects exactly that band
        cap_y = bound - double(p.alpha[q]);
    }
    if (!complete) {
        if (lane == 0) {
            const uint32_t at = atomicAdd(p.fb_count, 1u);
            p.fb_rows[at] = qo;  // input order
            p.fb_thr[at] = __double2float_ru(cap_y);
        }
        return;
    }
    const size_t orow = p.rowperm ? size_t(qo) : size_t(slot);
    for (uint32_t t = lane; t < p.klist; t += 32) {
        const uint64_t key = keys_s[warp][t];
        const float dv = ordered_to_float(uint32_t(key >> 32));
        p.out_index[orow * p.klist + t] = uint32_t(key);
        p.out_dist[orow * p.klist + t] = p.out_sqrt ? __fsqrt_rn(dv) : dv;
    }
}

// ---------------------------------------------------------------------------
// second pass for unproven rows: band capture

// Copy the swizzled fp16 rows rows[0..m) into a compact plane set (re-swizzled
// for their new row positions); padding rows are zero.
// xa row r = xh row map[rows[r]] (map: input index -> sorted position, or
// null), re-swizzled for its new position.  rows null: rows[r] = row0 + r.
__global__ void gather_rows_kernel(const uint8_t* __restrict__ xh, uint32_t npad, uint32_t kc,
                                   const uint32_t* __restrict__ rows, uint32_t row0, uint32_t m, uint32_t mpad,
                                   const uint32_t* __restrict__ map, uint8_t* __restrict__ xa) {
    const uint32_t total = kc * mpad * 8;  // 16-byte units
    for (uint32_t u = blockIdx.x * blockDim.x + threadIdx.x; u < total; u += gridDim.x * blockDim.x) {
        const uint32_t unit = u & 7, r = (u >> 3) % mpad, c = (u >> 3) / mpad;
        uint4 v = make_uint4(0, 0, 0, 0);
        if (r < m) {
            const uint32_t in = rows ? rows[r] : row0 + r;
            const uint32_t src = map ? map[in] : in;
            v = *reinterpret_cast<const uint4*>(xh + (size_t(c) * npad + src) * 128 + ((unit ^ (src & 7)) << 4));
        }
        *reinterpret_cast<uint4*>(xa + (size_t(c) * mpad + r) * 128 + ((unit ^ (r & 7)) << 4)) = v;
    }
}

struct Rescore2Params {
    const float* X;
    uint32_t n, d, klist;
    uint32_t row_begin;
    const uint32_t* rows;   // unproven rows (pass-1 order)
    uint32_t m;
    const uint32_t* cnt;
    const uint64_t* buf;
    uint32_t cap;
    int out_sqrt;
    uint32_t* out_index;
    float* out_dist;
    uint32_t* fb2_count;
    uint32_t* fb2_rows;
    unsigned long long* rescored;
    // the completeness check: every true neighbor's y is <= the row's
    // threshold (proof_bound of the band's k-th exact distance)
    const float* thr;            // [m] the capture thresholds (y)
    const uint32_t* rowpos;      // input row -> position of alpha/rho/xnorm (or null)
    const float* alpha;
    const double* rho;
    const double* xnorm;
    const unsigned long long* gmax;
    const unsigned int* maxabs;
    // retry mode (the threshold triangle): a row without a proof goes to
    // fb2_rows with retry_thr = the threshold that would prove it --
    // proof_bound of the k-th exact distance among its candidates, or loose[q]
    // when it has fewer than k -- for a second capture pass (null: no retry,
    // fb2_rows go to the EXACT kernel)
    float* retry_thr;
    const float* loose;
    // two-pass split (null: one pass): rows whose band outgrows the first
    // pass's shared-memory capacity are listed here for a second pass
    uint32_t* big;
    uint32_t* nbig;
};

// Exact rescore of a captured band (one warp per row): the band holds every
// column whose approximate y is within the row's threshold, each with that y
// in its key.  The k + 4 best by approximate y are folded first; their k-th
// exact distance bounds the true k-th, so only candidates whose approximate
// A is inside proof_bound of it are folded next (the others cannot be in the
// top-k).  The band is complete -- the row proven -- when
// proof_bound(k-th exact) - alpha is inside the capture threshold.
//
// Folds run 32 candidates at a time, one per lane, in coordinate order (bit
// parity): each 32-coordinate chunk of the 32 candidate rows is staged
// through shared memory with 32 coalesced 128-byte loads (all independent, so
// the warp keeps 4 KB in flight), then every lane folds its own row from the
// tile (the query's chunk comes by shuffle).  One lane per candidate with its
// own strided loads was latency-bound (ncu: 89% long-scoreboard stalls,
// 9% of DRAM bandwidth at C3).
//
// When rows are 16-byte aligned (d % 4 == 0, the common case) the chunks move
// with cp.async (16 bytes a lane, 8 per lane per chunk) into a kBandStages
// ring in XOR-swizzled layout: row r's 16-byte group g sits at g ^ (r & 7), so
// each lane reads its row with conflict-free LDS.128 and the query chunk is a
// broadcast LDS.128 -- no register staging, no per-element shuffles, and
// kBandStages - 1 chunks in flight per warp.  The register-staged version
// issued ~4x the instructions per coordinate and was issue- and
// latency-bound (ncu at C3: issue slots 57% busy at 14 warps per SM, DRAM
// 32% of peak, 167 ms; profiles/r02bm_c3_rescore.csv).  Two stages beat three
// and four (C3 step 1.03 against 1.06 s; profiles/r02bs_configs.txt): the
// smaller ring leaves room for more warps, which also hide the sorts.
constexpr int kBandWarps = 4;
#ifndef KNN_BAND_STAGES
#define KNN_BAND_STAGES 2
#endif
constexpr int kBandStages = KNN_BAND_STAGES;
constexpr uint32_t kBandStageFloats = 32 * 32 + 32;  // 32 candidate rows + the query, 32 coordinates each
__host__ __device__ __forceinline__ size_t band_stage_bytes() {
    const size_t ring = size_t(kBandStages) * kBandStageFloats * 4, tile = 32 * 33 * 4;
    return ring > tile ? ring : tile;
}
__device__ __forceinline__ size_t band_smem_per_warp(uint32_t cap) {
    return size_t(cap) * 16 + band_stage_bytes() + 64;
}

// Ascending bitonic sort of s[0, n) (n a power of two) by one warp.
__device__ __forceinline__ void warp_bitonic_sort(uint64_t* s, uint32_t n, int lane) {
    for (uint32_t k = 2; k <= n; k <<= 1)
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            for (uint32_t t = lane; t < n / 2; t += 32) {  // every lane one compare-exchange
                const uint32_t i = (t / j) * 2 * j + (t % j), l = i + j;
                const uint64_t a = s[i], b = s[l];
                if ((a > b) == ((i & k) == 0)) {
                    s[i] = b;
                    s[l] = a;
                }
            }
            __syncwarp();
        }
}

__device__ __forceinline__ uint32_t pow2_at_least(uint32_t x) { return x <= 1 ? 1 : 1u << (32 - __clz(x - 1)); }

// One band (slot) with shared-memory room for scap (a power of two)
// candidates; defer: a band larger than that goes to the second pass's list.
//
// The band's approximate keys are sorted once (a warp bitonic sort in shared
// memory); phase 1 folds the first klist + 4, phase 2 the prefix that follows
// while alpha + y stays inside the proof bound of phase 1's k-th exact
// distance -- the same sets as selecting by rank and by bound over the
// unsorted band.  The folded exact keys are sorted for the k-th distance and
// the output order.
template <int FOLD, bool VEC>
__device__ __forceinline__ void band_row(const Rescore2Params& p, uint32_t slot, uint8_t* wbase, uint32_t scap,
                                         bool defer) {
    const int lane = threadIdx.x & 31;
    uint64_t* ak = reinterpret_cast<uint64_t*>(wbase);  // approximate keys (y, col), sorted
    uint64_t* ek = ak + scap;                             // exact keys (distance, col) of folded positions
    float* tile = reinterpret_cast<float*>(ek + scap);    // [32][33]
    const uint32_t qo = p.rows[slot];  // input order
    if (qo == 0xffffffffu) return;     // a padding slot of a rank's last unit
    const uint32_t q = p.rowpos ? p.rowpos[qo] : qo;
    const uint32_t cnt_all = p.cnt[slot];
    const bool over = cnt_all > p.cap;  // lost candidates: no proof from this buffer
    if (defer && min(cnt_all, p.cap) > scap && !(over && !p.retry_thr)) {
        if (lane == 0) p.big[atomicAdd(p.nbig, 1u)] = slot;
        return;
    }
    auto retry = [&](double thr2) {
        if (lane == 0) {
            const uint32_t at = atomicAdd(p.fb2_count, 1u);
            p.fb2_rows[at] = qo;
            if (p.retry_thr) p.retry_thr[at] = __double2float_ru(thr2);
        }
    };
    if (over && !p.retry_thr) {
        retry(0);
        return;
    }
    const uint32_t c = over ? p.cap : cnt_all;
    const uint32_t na = max(pow2_at_least(c), 2u);
    const uint64_t* in = p.buf + size_t(slot) * p.cap;
    uint32_t nv = 0;  // non-empty candidates
    for (uint32_t i = lane; i < na; i += 32) {
        uint64_t key = i < c ? in[i] : kEmptyKey;
        if (uint32_t(key) == qo) key = kEmptyKey;  // the row itself is not a candidate
        ak[i] = key;
        nv += key != kEmptyKey;
    }
    for (int o = 16; o; o >>= 1) nv += __shfl_xor_sync(0xffffffffu, nv, o);
    __syncwarp();
    warp_bitonic_sort(ak, na, lane);
    const float* xq = p.X + size_t(qo) * p.d;
    // fold the candidates at sorted positions [lo, hi) (ak -> ek, same positions)
    auto fold_range = [&](uint32_t lo, uint32_t hi) {
        if constexpr (VEC) {
            float* ring = reinterpret_cast<float*>(ek + scap);
            const uint32_t nch = (p.d + 31) / 32, grp = lane & 7;
            for (uint32_t g0 = lo; g0 < hi; g0 += 32) {
                const uint32_t nrow = min(hi - g0, 32u);
                // lane copies 16-byte group grp of rows lane/8 + 4i, i < 8
                const float* src[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const uint32_t r = uint32_t(i) * 4 + (lane >> 3);
                    src[i] = p.X + size_t(r < nrow ? uint32_t(ak[g0 + r]) : qo) * p.d + grp * 4;
                }
                auto issue = [&](uint32_t c) {
                    if (c < nch) {
                        float* st = ring + (c % kBandStages) * kBandStageFloats;
                        const uint32_t j0 = c * 32;
                        const bool gin = j0 + grp * 4 < p.d;  // d % 4 == 0: a group is wholly in or out
#pragma unroll
                        for (int i = 0; i < 8; ++i) {
                            const uint32_t r = uint32_t(i) * 4 + (lane >> 3);
                            const bool on = gin && r < nrow;
                            ptx::cp_async16(st + r * 32 + ((grp ^ (r & 7)) << 2), on ? src[i] + j0 : p.X, on ? 16u : 0u);
                        }
                        if (lane < 8) ptx::cp_async16(st + 1024 + grp * 4, gin ? xq + j0 + grp * 4 : p.X, gin ? 16u : 0u);
                    }
                    ptx::cp_async_commit();  // (empty groups keep the count uniform)
                };
#pragma unroll
                for (int c = 0; c < kBandStages - 1; ++c) issue(uint32_t(c));
                float acc = 0.0f;
                for (uint32_t c = 0; c < nch; ++c) {
                    issue(c + kBandStages - 1);
                    ptx::cp_async_wait<kBandStages - 1>();  // chunk c has landed (this lane's copies)
                    __syncwarp();                      // ... and every lane's
                    const float* st = ring + (c % kBandStages) * kBandStageFloats;
                    const float* row = st + lane * 32;
                    const float* qc = st + 1024;
                    const uint32_t ng = min(p.d - c * 32, 32u) >> 2;
                    if (ng == 8) {
#pragma unroll
                        for (uint32_t g = 0; g < 8; ++g) {
                            const float4 v = *reinterpret_cast<const float4*>(row + ((g ^ (lane & 7)) << 2));
                            const float4 q4 = *reinterpret_cast<const float4*>(qc + g * 4);
                            acc = fold_step_x2<FOLD>(v.x, v.y, q4.x, q4.y, acc);
                            acc = fold_step_x2<FOLD>(v.z, v.w, q4.z, q4.w, acc);
                        }
                    } else {
                        for (uint32_t g = 0; g < ng; ++g) {
                            const float4 v = *reinterpret_cast<const float4*>(row + ((g ^ (lane & 7)) << 2));
                            const float4 q4 = *reinterpret_cast<const float4*>(qc + g * 4);
                            acc = fold_step_x2<FOLD>(v.x, v.y, q4.x, q4.y, acc);
                            acc = fold_step_x2<FOLD>(v.z, v.w, q4.z, q4.w, acc);
                        }
                    }
                    __syncwarp();  // the stage is rewritten by the next iteration's issue
                }
                if (uint32_t(lane) < nrow)
                    ek[g0 + lane] = make_key(fold_finalize<FOLD>(acc), uint32_t(ak[g0 + lane]));
            }
            __syncwarp();
        } else {
        for (uint32_t g = lo; g < hi; g += 32) {
            const bool mine = g + lane < hi;
            const uint32_t col = mine ? uint32_t(ak[g + lane]) : qo;
            // lane r's candidate row: lanes load row r's chunk (coalesced);
            // the next chunk's 32 loads are in flight while this one folds
            float nxt[32];
            float qn = 0.0f;
            auto load_chunk = [&](uint32_t j0) {
                const uint32_t w = p.d - j0 < 32 ? p.d - j0 : 32;
#pragma unroll
                for (int r = 0; r < 32; ++r) {
                    const uint32_t cr = __shfl_sync(0xffffffffu, col, r);
                    nxt[r] = uint32_t(lane) < w ? __ldg(p.X + size_t(cr) * p.d + j0 + lane) : 0.0f;
                }
                qn = uint32_t(lane) < w ? __ldg(xq + j0 + lane) : 0.0f;
            };
            float acc = 0.0f;
            load_chunk(0);
            for (uint32_t j0 = 0; j0 < p.d; j0 += 32) {
                const uint32_t w = p.d - j0 < 32 ? p.d - j0 : 32;
#pragma unroll
                for (int r = 0; r < 32; ++r) tile[r * 33 + lane] = nxt[r];
                const float qv = qn;
                __syncwarp();
                if (j0 + 32 < p.d) load_chunk(j0 + 32);
                for (uint32_t jj = 0; jj < w; ++jj)
                    acc = fold_step<FOLD>(tile[lane * 33 + jj], __shfl_sync(0xffffffffu, qv, jj), acc);
                __syncwarp();
            }
            if (mine) ek[g + lane] = make_key(fold_finalize<FOLD>(acc), col);
        }
        __syncwarp();
        }
    };
    // sort ek[0, m) (padding with empty keys up to a power of two)
    auto sort_exact = [&](uint32_t m) {
        const uint32_t ne = max(pow2_at_least(m), 2u);
        for (uint32_t i = m + lane; i < ne; i += 32) ek[i] = kEmptyKey;
        __syncwarp();
        warp_bitonic_sort(ek, ne, lane);
    };
    // phase 1: the klist + 4 best by approximate y
    const uint32_t p1 = min(p.klist + 4, nv);
    fold_range(0, p1);
    sort_exact(p1);
    const double alpha_q = double(p.alpha[q]);
    // phase 2: the following candidates whose approximate A is inside the
    // bound of phase 1's k-th exact distance (all of them without a k-th)
    uint32_t p2 = nv;
    if (p1 >= p.klist) {
        const uint64_t kth1 = ek[p.klist - 1];
        const double lim = proof_bound<FOLD>(p.d, p.maxabs, p.gmax, p.xnorm[q], p.rho[q], alpha_q,
                                             double(ordered_to_float(uint32_t(kth1 >> 32))));
        // first position (>= p1) whose alpha + y exceeds lim: y ascends along ak
        uint32_t cut = nv;
        for (uint32_t i0 = p1; i0 < nv; i0 += 32) {
            const uint32_t i = i0 + lane;
            const bool outside = i < nv && !(alpha_q + double(ordered_to_float(uint32_t(ak[i] >> 32))) <= lim);
            const uint32_t b = __ballot_sync(0xffffffffu, outside);
            if (b) {
                cut = i0 + __ffs(b) - 1;
                break;
            }
        }
        p2 = cut;
    }
    if (p2 > p1) {
        fold_range(p1, p2);
        sort_exact(p2);
    }
    const uint32_t valid = p2;  // every folded candidate has an exact key
    if (lane == 0) atomicAdd(p.rescored, (unsigned long long)valid);
    if (valid < p.klist) {  // a proven band has >= k; a threshold guessed too low may not
        retry(p.loose ? double(p.loose[q]) : 0.0);
        return;
    }
    const uint64_t kth = ek[p.klist - 1];
    // the band's k-th exact distance bounds the true k-th from above, so
    // every true neighbor has y <= proof_bound(kth) - alpha_q: the band is
    // complete when that is inside its threshold
    const double need = proof_bound<FOLD>(p.d, p.maxabs, p.gmax, p.xnorm[q], p.rho[q], alpha_q,
                                          double(ordered_to_float(uint32_t(kth >> 32)))) - alpha_q;
    if (over || !(need <= double(p.thr[slot]))) {
        retry(need);
        return;
    }
    const size_t orow = size_t(qo - p.row_begin);
    for (uint32_t r = lane; r < p.klist; r += 32) {
        const uint64_t mk = ek[r];
        const float dv = ordered_to_float(uint32_t(mk >> 32));
        p.out_index[orow * p.klist + r] = uint32_t(mk);
        p.out_dist[orow * p.klist + r] = p.out_sqrt ? __fsqrt_rn(dv) : dv;
    }
}

// pass 0: one warp per slot, room for scap candidates, larger bands listed in
// p.big; pass 1: the listed slots (grid-stride), room for p.cap; pass 2: one
// warp per slot, room for p.cap (no split).
template <int FOLD, int NW, bool VEC>
__global__ void __launch_bounds__(32 * NW, 16 / NW) rescore_capture_kernel(const Rescore2Params p, uint32_t scap, int pass) {
    extern __shared__ __align__(16) uint8_t band_smem[];
    const int warp = threadIdx.x >> 5;
    uint8_t* wbase = band_smem + size_t(warp) * band_smem_per_warp(scap);
    if (pass == 1) {
        const uint32_t nb = *p.nbig;
        for (uint32_t i = blockIdx.x * NW + warp; i < nb; i += gridDim.x * NW) band_row<FOLD, VEC>(p, p.big[i], wbase, scap, false);
        return;
    }
    const uint32_t slot = blockIdx.x * NW + warp;
    if (slot < p.m) band_row<FOLD, VEC>(p, slot, wbase, scap, pass == 0);
}

static size_t band_smem_bytes(uint32_t cap, int warps = kBandWarps) {
    return warps * (size_t(cap) * 16 + band_stage_bytes() + 64);
}

// expect: the typical band size (0: unknown).  With r2.big set, bands up to
// ~1.25 expect (rounded up to a power of two) run in small shared-memory
// slices (2x the occupancy of slices sized for the capacity); the rest get a
// second pass.  r2.cap must be a power of two.
template <int FOLD, bool VEC>
static cudaError_t launch_rescore_capture_v(const Rescore2Params& r2, uint32_t rows, cudaStream_t st,
                                            uint32_t expect) {
    cudaError_t e;
    // (band slices hold a power of two: the bitonic sorts' size)
    uint32_t scap = 128;
    while (scap < expect + expect / 4) scap *= 2;
    if (r2.big && expect && scap < r2.cap) {
        // 8 or 4 warps per block, whichever keeps more warps per SM resident
        // (227 KB of shared memory; ~128 registers a thread: 2 blocks of 8, 4 of 4)
        const size_t per_warp = band_smem_bytes(scap, 1);
        const uint32_t w8 = 8 * std::min<uint32_t>(2, uint32_t((227u << 10) / (8 * per_warp)));
        const uint32_t w4 = 4 * std::min<uint32_t>(4, uint32_t((227u << 10) / (4 * per_warp)));
        const bool eight = w8 > w4;  // a tie goes to 4-warp blocks: a finished block frees its slices sooner
        auto k0 = eight ? rescore_capture_kernel<FOLD, 8, VEC> : rescore_capture_kernel<FOLD, 4, VEC>;
        auto k1 = rescore_capture_kernel<FOLD, kBandWarps, VEC>;
        const int nw0 = eight ? 8 : 4;
        const size_t s0 = band_smem_bytes(scap, nw0), s1 = band_smem_bytes(r2.cap);
        if ((e = cudaFuncSetAttribute(k0, cudaFuncAttributeMaxDynamicSharedMemorySize, int(s0))) != cudaSuccess) return e;
        if ((e = cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, int(s1))) != cudaSuccess) return e;
        if ((e = cudaMemsetAsync(r2.nbig, 0, 4, st)) != cudaSuccess) return e;
        k0<<<(rows + nw0 - 1) / nw0, 32 * nw0, s0, st>>>(r2, scap, 0);
        int sms = 148, dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        k1<<<std::min<uint32_t>((rows + kBandWarps - 1) / kBandWarps, uint32_t(sms) * 2), 32 * kBandWarps, s1, st>>>(
            r2, r2.cap, 1);
        return cudaGetLastError();
    }
    auto k = rescore_capture_kernel<FOLD, kBandWarps, VEC>;
    const size_t smem = band_smem_bytes(r2.cap);
    if ((e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem))) != cudaSuccess) return e;
    k<<<(rows + kBandWarps - 1) / kBandWarps, 32 * kBandWarps, smem, st>>>(r2, r2.cap, 2);
    return cudaGetLastError();
}

template <int FOLD>
static cudaError_t launch_rescore_capture(const Rescore2Params& r2, uint32_t rows, cudaStream_t st,
                                          uint32_t expect = 0) {
    // 16-byte aligned rows: the cp.async ring (KNN_B200_BAND_VEC=0: the register-staged fold)
    const char* ev = getenv("KNN_B200_BAND_VEC");
    const bool vec = r2.d % 4 == 0 && reinterpret_cast<uintptr_t>(r2.X) % 16 == 0 && !(ev && atoi(ev) == 0);
    return vec ? launch_rescore_capture_v<FOLD, true>(r2, rows, st, expect)
               : launch_rescore_capture_v<FOLD, false>(r2, rows, st, expect);
}

// ---------------------------------------------------------------------------
// host orchestration

// Candidate-list shape per k: KPL entries per list, NSEG lists per row (one
// per epilogue column segment).  A segment may hold every one of the k
// nearest, so each list needs k + 1 (the query itself) + a margin for the
// error band; the margin is where rows fail their proof and fall back.
struct TensorCfg {
    uint32_t kpl, nseg;
};

static TensorCfg tensor_cfg(uint32_t klist) {
    const uint32_t margin = klist / 4 > 8 ? klist / 4 : 8;
    if (klist + 1 + 5 <= 16) {
        const char* e = getenv("KNN_B200_LIST16_SEGMENTS");  // tuning knob: 2 (default) or 1
        if (e && atoi(e) == 1) return {16, 1};
        // Two column-half segments per row.  Shorter lists mean fewer and
        // cheaper insertions (each list sees ~KPL ln(n / KPL) records) but a
        // lower proof bound: at C2 (k = 10) KPL 12 is fastest end to end --
        // 0.3% of rows go to the capture pass -- against 16 (no fallback) and
        // 10 (5% fallback).  Tuning knob KNN_B200_KPL: 8, 10, 12, 14 or 16.
        const char* kp = getenv("KNN_B200_KPL");
        const uint32_t want = kp ? uint32_t(atoi(kp)) : 12u;
        if (want == 8 && klist <= 4) return {8, 2};
        if (want == 10 && klist <= 10) return {10, 2};
        if (want == 12 && klist + 1 <= 12) return {12, 2};
        if (want == 14 && klist + 1 <= 14) return {14, 2};
        return {16, 2};
    }
    // Two 32-entry shared-memory segments hold k up to 47: each half of the
    // columns holds about half of a row's neighbours (measured at n = 1M,
    // d = 128: k = 24/32/40 in 0.44 s with 0 / 8 / 3879 rows to the capture
    // pass, against 0.86 s for one 64-entry list at k = 24; 24-entry register
    // lists spill and lose).
    if (klist + 1 <= 48) return {32, 2};
    if (klist + 1 + margin <= 64) return {64, 1};
    if (klist + 1 + margin <= 128) return {128, 1};
    return {0, 0};  // not supported by the tensor sweep
}

uint32_t tensor_kp_for(uint32_t klist) {
    const TensorCfg c = tensor_cfg(klist);
    return c.kpl * c.nseg;
}

size_t capture_workspace_bytes(uint32_t m, uint32_t d, uint32_t cap) {
    const uint32_t mpad = (m + TS_BM - 1) / TS_BM * TS_BM;
    const uint32_t kc = (d + 63) / 64;
    size_t b = 0;
    auto add = [&](size_t x) { b += (x + 255) / 256 * 256; };
    add(size_t(kc) * mpad * 128);
    add(size_t(m) * 4 + 8);
    add(size_t(m) * cap * 8);
    add(size_t(m) * 4);
    return b;
}

// Norm-sorted order (whole problems): keys, the permutation, and CUB's
// radix-sort scratch.
static size_t sort_temp_bytes(uint32_t n) {
    size_t t = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, t, static_cast<const float*>(nullptr), static_cast<float*>(nullptr),
                                    static_cast<const uint32_t*>(nullptr), static_cast<uint32_t*>(nullptr), int(n));
    return t;
}

static size_t sort_workspace_bytes(uint32_t n) {
    return 5 * ((size_t(n) * 4 + 255) / 256 * 256) + (sort_temp_bytes(n) + 255) / 256 * 256;
}

__global__ void invert_perm_kernel(const uint32_t* __restrict__ perm, uint32_t n, uint32_t* __restrict__ pos) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) pos[perm[i]] = i;
}

// Sort the sweep's columns by norm (KNN_B200_SORT=0 disables; cosine norms
// are all equal already).  Query rows stay in input order: the sweep reads
// them from compact gathered planes.
static bool sort_selected(int cosine) {
    const char* e = getenv("KNN_B200_SORT");
    return !(e && atoi(e) == 0) && !cosine;
}

size_t tensor_workspace_bytes(uint32_t n, uint32_t d, uint32_t row_begin, uint32_t row_end, uint32_t klist,
                              int sm_count) {
    const uint32_t rows = row_end - row_begin;
    const uint32_t kp = tensor_kp_for(klist);
    const uint32_t npad = (n + 255) / 256 * 256;
    const uint32_t kc = (d + 63) / 64;
    size_t b = 0;
    auto add = [&](size_t x) { b += (x + 255) / 256 * 256; };
    add(size_t(kc) * npad * 128);  // xh
    add(size_t(npad) * 4);         // alpha
    add(size_t(npad / 32) * 8);    // bmin + bound halves
    add(size_t(npad) * 8);         // rho
    add(size_t(npad) * 8);         // xnorm
    add(size_t(d) * 8);            // mu acc
    add(size_t(d) * 4);            // mu
    add(64);                       // scalars
    add(size_t(rows) * kp * 8);    // cand
    add(size_t(rows) * 4);         // fallback rows
    add(size_t(rows) * 4);         // capture thresholds
    add(sort_workspace_bytes(n));                                 // norm-sorted columns
    add(size_t(kc) * ((rows + 255) / 256 * 256) * 128);          // query rows in input order
    return b;
}

// CTA-pair sweep (cluster of 2): one pair per two SMs, persistent.  ARES =
// false streams the query rows with every reference chunk (d > 256).
template <int KPL, int BN, int EW, bool TRI = false, bool TCAP = false, bool ARES = true, bool DYN = false>
static cudaError_t launch_sweep_pair(const SweepParams& sp, uint32_t nrows, cudaStream_t stream) {
    using L = TSLayout<KPL, BN, ARES, EW, true>;
    auto kern = tensor_sweep_kernel<KPL, BN, ARES, EW, false, true, TRI, TCAP, DYN>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(L::SMEM));
    if (e != cudaSuccess) return e;
    const uint32_t npairs = (nrows + 2 * TS_BM - 1) / (2 * TS_BM);
    int sms = 148, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const uint32_t grid_pairs = npairs < uint32_t(sms / 2) ? npairs : uint32_t(sms / 2);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * grid_pairs);
    cfg.blockDim = dim3(L::THREADS);
    cfg.dynamicSmemBytes = L::SMEM;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, sp);
}

template <int KPL, int BN, bool ARES, int EW, bool CAPTURE = false>
static cudaError_t launch_sweep_t(const SweepParams& sp, uint32_t nrows, cudaStream_t stream) {
    using L = TSLayout<KPL, BN, ARES, EW>;
    auto kern = tensor_sweep_kernel<KPL, BN, ARES, EW, CAPTURE>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(L::SMEM));
    if (e != cudaSuccess) return e;
    const uint32_t nrb = (nrows + TS_BM - 1) / TS_BM;
    int sms = 148;
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    dim3 grid(nrb < uint32_t(sms) ? nrb : uint32_t(sms));  // persistent: one CTA per SM
    if constexpr (CAPTURE) {  // few rows: split the column groups over blockIdx.y as well
        const uint32_t ntiles = (sp.n + BN - 1) / BN;
        const uint32_t ngroups = (ntiles + sp.group_tiles - 1) / sp.group_tiles;
        uint32_t gy = uint32_t(sms) / grid.x;
        gy = gy < 1 ? 1 : (gy > ngroups ? ngroups : gy);
        grid.y = gy;
    }
    kern<<<grid, L::THREADS, L::SMEM, stream>>>(sp);
    return cudaGetLastError();
}

static cudaError_t launch_sweep(TensorCfg c, bool ares, const SweepParams& sp, uint32_t nrows, cudaStream_t stream) {
    switch (c.kpl) {
    case 8:
        return ares ? launch_sweep_t<8, 256, true, 8>(sp, nrows, stream)
                    : launch_sweep_t<8, 256, false, 8>(sp, nrows, stream);
    case 10:
        return ares ? launch_sweep_t<10, 256, true, 8>(sp, nrows, stream)
                    : launch_sweep_t<10, 256, false, 8>(sp, nrows, stream);
    case 12:
        return ares ? launch_sweep_t<12, 256, true, 8>(sp, nrows, stream)
                    : launch_sweep_t<12, 256, false, 8>(sp, nrows, stream);
    case 14:
        return ares ? launch_sweep_t<14, 256, true, 8>(sp, nrows, stream)
                    : launch_sweep_t<14, 256, false, 8>(sp, nrows, stream);
    case 16:
        if (c.nseg == 1)
            return ares ? launch_sweep_t<16, 256, true, 4>(sp, nrows, stream)
                        : launch_sweep_t<16, 256, false, 4>(sp, nrows, stream);
        return ares ? launch_sweep_t<16, 256, true, 8>(sp, nrows, stream)
                    : launch_sweep_t<16, 256, false, 8>(sp, nrows, stream);
    case 32:
        return ares ? launch_sweep_t<32, 256, true, 8>(sp, nrows, stream)
                    : launch_sweep_t<32, 256, false, 8>(sp, nrows, stream);
    case 64:
        return ares ? launch_sweep_t<64, 256, true, 4>(sp, nrows, stream)
                    : launch_sweep_t<64, 256, false, 4>(sp, nrows, stream);
    default:
        return ares ? launch_sweep_t<128, 128, true, 4>(sp, nrows, stream)
                    : launch_sweep_t<128, 128, false, 4>(sp, nrows, stream);
    }
}

static cudaError_t launch_capture_sweep(bool ares, const SweepParams& sp, uint32_t nrows, cudaStream_t stream) {
    return ares ? launch_sweep_t<16, 256, true, 8, true>(sp, nrows, stream)
                : launch_sweep_t<16, 256, false, 8, true>(sp, nrows, stream);
}

template <int FOLD>
static cudaError_t launch_rescore(TensorCfg c, const RescoreParams& rp, uint32_t nrows, cudaStream_t stream) {
    const dim3 grid((nrows + 7) / 8);
    switch (c.kpl) {
    case 8: rescore_kernel<FOLD, 16, 2><<<grid, 256, 0, stream>>>(rp); break;
    case 10: rescore_kernel<FOLD, 20, 2><<<grid, 256, 0, stream>>>(rp); break;
    case 12: rescore_kernel<FOLD, 24, 2><<<grid, 256, 0, stream>>>(rp); break;
    case 14: rescore_kernel<FOLD, 28, 2><<<grid, 256, 0, stream>>>(rp); break;
    case 16:
        if (c.nseg == 1) rescore_kernel<FOLD, 16, 1><<<grid, 256, 0, stream>>>(rp);
        else rescore_kernel<FOLD, 32, 2><<<grid, 256, 0, stream>>>(rp);
        break;
    case 32: rescore_kernel<FOLD, 64, 2><<<grid, 256, 0, stream>>>(rp); break;
    case 64: rescore_kernel<FOLD, 64, 1><<<grid, 256, 0, stream>>>(rp); break;
    default: rescore_kernel<FOLD, 128, 1><<<grid, 256, 0, stream>>>(rp); break;
    }
    return cudaGetLastError();
}

// Rows without a completeness proof: a second tensor pass captures the whole
// proven band of each such row (fixed per-row thresholds fb_thr), then an
// exact rescore; only rows whose band overflows the capture buffer are
// recomputed by the EXACT kernel.  fb_rows are input rows; results go to
// a.out_* at row fb_rows[i] - a.row_begin.
struct CaptureArgs {
    const uint8_t* xh;  // the first-order (norm-sorted) planes and per-row arrays
    const float* alpha;
    const double* rho;
    const double* xnorm;
    const unsigned long long* gmax;
    const unsigned int* maxabs;
    const float* bmin;
    const uint32_t* perm;    // sorted position -> input row (null: unsorted)
    const uint32_t* rowpos;  // input row -> sorted position (null: unsorted)
    uint32_t n, npad, kc, group_tiles, cap;
    const uint32_t* fb_rows;
    const float* fb_thr;
    unsigned long long* rescored;
};

static cudaError_t run_capture(const TensorPathArgs& a, const CaptureArgs& c, uint32_t nfb, TensorPathResult& r,
                               uint32_t& launches) {
    cudaStream_t st = a.stream;
    cudaError_t e;
    const uint32_t mpad = (nfb + TS_BM - 1) / TS_BM * TS_BM;
    uint8_t* w2 = static_cast<uint8_t*>(a.alloc2(a.alloc2_ctx, capture_workspace_bytes(nfb, a.d, c.cap)));
    if (!w2) return cudaErrorMemoryAllocation;
    auto take2 = [&](size_t x) {
        uint8_t* q = w2;
        w2 += (x + 255) / 256 * 256;
        return q;
    };
    uint8_t* xa = take2(size_t(c.kc) * mpad * 128);
    uint32_t* cap_cnt = reinterpret_cast<uint32_t*>(take2(size_t(nfb) * 4 + 8));
    uint64_t* cap_buf = reinterpret_cast<uint64_t*>(take2(size_t(nfb) * c.cap * 8));
    uint32_t* fb2_rows = reinterpret_cast<uint32_t*>(take2(size_t(nfb) * 4));
    uint32_t* fb2_count = cap_cnt + nfb;
    if ((e = cudaMemsetAsync(cap_cnt, 0, size_t(nfb) * 4 + 8, st)) != cudaSuccess) return e;
    gather_rows_kernel<<<a.sm_count * 4, 256, 0, st>>>(c.xh, c.npad, c.kc, c.fb_rows, 0, nfb, mpad, c.rowpos, xa);
    SweepParams cp{c.xh,    c.alpha, c.n,  c.npad,   c.kc,    0,       nfb,   c.group_tiles, 0,
                   nullptr, xa,      mpad, c.fb_thr, cap_cnt, cap_buf, c.cap, c.bmin};
    if ((e = launch_capture_sweep(c.kc <= uint32_t(TS_MAX_RES_KC), cp, nfb, st)) != cudaSuccess) return e;
    if (c.perm) {
        remap_capture_kernel<<<nfb, 128, 0, st>>>(cap_buf, cap_cnt, nfb, c.cap, c.perm);
        ++launches;
    }
    Rescore2Params r2{a.X,     a.n,   a.d,        a.klist,     a.row_begin, c.fb_rows, nfb,      cap_cnt,
                      cap_buf, c.cap, a.out_sqrt, a.out_index, a.out_dist,  fb2_count, fb2_rows, c.rescored,
                      c.fb_thr, c.rowpos, c.alpha, c.rho, c.xnorm, c.gmax, c.maxabs};
    e = a.fold == kCosine ? launch_rescore_capture<kCosine>(r2, nfb, st) : launch_rescore_capture<kSqEuclidean>(r2, nfb, st);
    if (e != cudaSuccess) return e;
    launches += 3;
    if ((e = cudaMemcpyAsync(a.host_scratch, fb2_count, 4, cudaMemcpyDeviceToHost, st)) != cudaSuccess) return e;
    if ((e = cudaMemcpyAsync(static_cast<uint8_t*>(a.host_scratch) + 32, c.rescored, 8, cudaMemcpyDeviceToHost, st)) !=
        cudaSuccess)
        return e;
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
    const uint32_t nfb2 = *static_cast<const uint32_t*>(a.host_scratch);
    r.rescored = *reinterpret_cast<const unsigned long long*>(static_cast<const uint8_t*>(a.host_scratch) + 32);
    r.exact_rows = nfb2;
    if (getenv("KNN_B200_DEBUG_FB"))  // profiling only
        fprintf(stderr, "[run_capture] %u rows captured, %u to the EXACT kernel\n", nfb, nfb2);
    if (nfb2) {
        if ((e = launch_exact_fused(a.fold, a.X, a.n, a.d, a.klist, fb2_rows, 0, nfb2, a.out_index, a.out_dist,
                                    a.out_sqrt, a.row_begin, a.exact_scratch, a.sm_count, st)) != cudaSuccess)
            return e;
        ++launches;
    }
    return cudaSuccess;
}

static cudaError_t run_tensor_path_impl(const TensorPathArgs& a, TensorPathResult& r);

// Whole problems that take the triangle sweep (each unordered pair once):
// sorted columns (not cosine), two 12-entry lists (k <= 11), resident A
// (d <= 256), and n past the measured crossover (262K: rectangular faster,
// 524K: triangle faster).  KNN_B200_TRI=0 disables it; KNN_B200_TRI=force
// drops the size gate (testing: the sharded program at small n, sanitizers).
bool tri_eligible(uint32_t n, uint32_t d, uint32_t klist, int fold) {
    const char* te = getenv("KNN_B200_TRI");
    if (te && strcmp(te, "0") == 0) return false;
    const bool force = te && strcmp(te, "force") == 0;
    const TensorCfg cfg = tensor_cfg(klist);
    return fold != kCosine && sort_selected(0) && cfg.kpl == 12 && cfg.nseg == 2 &&
           (d + 63) / 64 <= uint32_t(TS_MAX_RES_KC) && (force ? n >= 512 : n >= 393216);
}


cudaError_t run_tensor_path(const TensorPathArgs& a, TensorPathResult& r) {
    const bool whole = a.row_begin == 0 && a.row_end == a.n && a.shard_alloc;
    // whole problems with k <= 10: the list triangle, run as the one-rank case
    // of the sharded program (tri_shard.cuh: snake-dealt units, chunk pool)
    if (whole && tri_eligible(a.n, a.d, a.klist, a.fold)) {
        bool overflow = false;
        const cudaError_t e =
            run_tri_loopback(a, 1, a.shard_alloc, a.shard_ctx, r, nullptr, nullptr, &overflow, false);
        if (e != cudaSuccess || !overflow) return e;
        r = TensorPathResult{};  // the pool overflowed (pathological data): the rectangular sweep
        return run_tensor_path_impl(a, r);
    }
    // whole problems with 10 < k <= 128: the threshold triangle (tri_shard.cuh)
    if (whole && tcap_eligible(a.n, a.d, a.klist)) {
        bool overflow = false;
        const cudaError_t e =
            run_tri_loopback(a, 1, a.shard_alloc, a.shard_ctx, r, nullptr, nullptr, &overflow, true);
        if (e != cudaSuccess || !overflow) return e;
        r = TensorPathResult{};  // the pool overflowed (pathological data): the rectangular sweep
    }
    return run_tensor_path_impl(a, r);
}

static cudaError_t run_tensor_path_impl(const TensorPathArgs& a, TensorPathResult& r) {
    const uint32_t n = a.n, d = a.d, nrows = a.row_end - a.row_begin;
    const uint32_t npad = (n + 255) / 256 * 256;
    const uint32_t kc = (d + 63) / 64;
    const TensorCfg cfg = tensor_cfg(a.klist);
    const uint32_t kp = cfg.kpl * cfg.nseg;
    const int cosine = a.fold == kCosine;
    uint8_t* w = static_cast<uint8_t*>(a.workspace);
    if (!w && a.alloc_ws)
        w = static_cast<uint8_t*>(
            a.alloc_ws(a.alloc2_ctx, tensor_workspace_bytes(n, d, a.row_begin, a.row_end, a.klist, a.sm_count)));
    if (!w) return cudaErrorMemoryAllocation;
    auto take = [&](size_t x) {
        uint8_t* p = w;
        w += (x + 255) / 256 * 256;
        return p;
    };
    uint8_t* xh = take(size_t(kc) * npad * 128);
    float* alpha = reinterpret_cast<float*>(take(size_t(npad) * 4));
    float* bmin = reinterpret_cast<float*>(take(size_t(npad / 32) * 8));  // + bound halves
    double* rho = reinterpret_cast<double*>(take(size_t(npad) * 8));
    double* xnorm = reinterpret_cast<double*>(take(size_t(npad) * 8));
    double* muacc = reinterpret_cast<double*>(take(size_t(d) * 8));
    float* mu = reinterpret_cast<float*>(take(size_t(d) * 4));
    uint8_t* scal = take(64);
    uint64_t* cand = reinterpret_cast<uint64_t*>(take(size_t(nrows) * kp * 8));
    uint32_t* fb_rows = reinterpret_cast<uint32_t*>(take(size_t(nrows) * 4));
    float* fb_thr = reinterpret_cast<float*>(take(size_t(nrows) * 4));
    const bool sorted = sort_selected(cosine);
    float* skey = reinterpret_cast<float*>(take(size_t(n) * 4));
    float* skey2 = reinterpret_cast<float*>(take(size_t(n) * 4));
    uint32_t* sidx = reinterpret_cast<uint32_t*>(take(size_t(n) * 4));
    uint32_t* perm = reinterpret_cast<uint32_t*>(take(size_t(n) * 4));    // sorted position -> input row
    uint32_t* rowpos = reinterpret_cast<uint32_t*>(take(size_t(n) * 4));  // input row -> sorted position
    size_t stemp_bytes = sort_temp_bytes(n);
    void* stemp = take(stemp_bytes);
    const uint32_t qpad = (nrows + 255) / 256 * 256;
    uint8_t* xq_planes = take(size_t(kc) * qpad * 128);  // the call's query rows, input order
    unsigned int* maxabs = reinterpret_cast<unsigned int*>(scal);
    uint32_t* fb_count = reinterpret_cast<uint32_t*>(scal + 4);
    unsigned long long* gmax = reinterpret_cast<unsigned long long*>(scal + 8);
    unsigned long long* rescored = reinterpret_cast<unsigned long long*>(scal + 32);
    cudaStream_t st = a.stream;
    cudaError_t e;
    uint32_t launches = 0;

    if ((e = cudaMemsetAsync(scal, 0, 64, st)) != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(muacc, 0, size_t(d) * 8, st)) != cudaSuccess) return e;
    if (!cosine) {
        launch_colmean(a.X, n, d, muacc, mu, a.sm_count, st);
        launches += 2;
    } else {
        if ((e = cudaMemsetAsync(mu, 0, size_t(d) * 4, st)) != cudaSuccess) return e;
    }
    center_stats_kernel<<<a.sm_count * 8, 256, 0, st>>>(a.X, n, d, mu, maxabs, sorted ? skey : nullptr, sidx,
                                                        vec4_rows(a.X, d));
    if (sorted) {
        if ((e = cub::DeviceRadixSort::SortPairs(stemp, stemp_bytes, skey, skey2, sidx, perm, int(n), 0, 32, st)) !=
            cudaSuccess)
            return e;
        invert_perm_kernel<<<a.sm_count * 4, 256, 0, st>>>(perm, n, rowpos);
        launches += 3;
    }
    PrepOut po{xh, alpha, rho, xnorm, gmax};
    prep_kernel<<<a.sm_count * 8, 256, 0, st>>>(a.X, n, d, npad, kc, mu, maxabs, cosine, sorted ? perm : nullptr, po);
    chunk_min_kernel<<<(npad / 32 * 32 + 255) / 256, 256, 0, st>>>(alpha, npad / 32, bmin);
    launches += 3;
    if (sorted) {  // query rows back in input order for the A operand
        gather_rows_kernel<<<a.sm_count * 4, 256, 0, st>>>(xh, npad, kc, nullptr, a.row_begin, nrows, qpad, rowpos,
                                                           xq_planes);
        ++launches;
    }
    if ((e = cudaGetLastError()) != cudaSuccess) return e;

    // Column groups: a group's fp16 reference tiles (BN x d x 2 B each) must
    // stay L2-resident while every CTA streams them (126 MB L2; keep ~40 MB).
    const uint32_t bn = cfg.kpl == 128 ? 128 : 256;
    const uint64_t tile_bytes = uint64_t(bn) * kc * 128;
    const uint32_t ntiles = (n + bn - 1) / bn;
    uint32_t group_tiles = uint32_t((40ull << 20) / tile_bytes);
    if (group_tiles < 1) group_tiles = 1;
    if (group_tiles > ntiles) group_tiles = ntiles;
    const char* dbg = getenv("KNN_B200_DEBUG_SWEEP");
    // sorted: the A operand is the compact input-order copy of the call's rows
    const uint32_t sr0 = sorted ? 0 : a.row_begin, sr1 = sorted ? nrows : a.row_end;
    const uint8_t* xa_rows = sorted ? xq_planes : xh;
    const uint32_t npad_a = sorted ? qpad : npad;
    SweepParams sp{xh,   alpha,  n,       npad,    kc, sr0, sr1, group_tiles, dbg ? atoi(dbg) : 0,
                   cand, xa_rows, npad_a, nullptr, nullptr, nullptr, 0, bmin};
    // (whole problems with k <= 10 take the triangle sweep before reaching
    // here: run_tensor_path -> run_tri_loopback, tri_shard.cuh)
    if (a.ev_sweep0) cudaEventRecord(a.ev_sweep0, st);
    // CTA pairs (default; KNN_B200_PAIR=0 disables) need whole 256-row
    // pairs of blocks inside the padded planes.  At C2 they halve the
    // L2->SM operand traffic and cut the sweep ~3%.
    const char* pe = getenv("KNN_B200_PAIR");
    const bool pair = !(pe && atoi(pe) == 0) && kc <= uint32_t(TS_MAX_RES_KC) && cfg.nseg == 2 &&
                      (cfg.kpl == 12 || cfg.kpl == 16) && sr0 % 256 == 0 && sr0 + (nrows + 255) / 256 * 256 <= npad_a;
    if (pair) {
        e = cfg.kpl == 12 ? launch_sweep_pair<12, 256, 8>(sp, nrows, st)
                          : launch_sweep_pair<16, 256, 8>(sp, nrows, st);
        if (e != cudaSuccess) return e;
    } else if ((e = launch_sweep(cfg, kc <= uint32_t(TS_MAX_RES_KC), sp, nrows, st)) != cudaSuccess) {
        return e;
    }
    ++launches;
    if (a.ev_sweep1) cudaEventRecord(a.ev_sweep1, st);
    if (sorted) {
        remap_kernel<<<a.sm_count * 8, 256, 0, st>>>(cand, size_t(nrows) * kp, perm, n);
        ++launches;
    }

    RescoreParams rp{a.X,  n,         d,          a.klist,  kp,       a.row_begin, a.row_end, cand,
                     alpha, rho,      xnorm,      gmax,     maxabs,   a.fold,      a.out_sqrt, a.out_index,
                     a.out_dist, fb_count, fb_rows, fb_thr, rescored, 0, sorted ? rowpos : nullptr};
    {
        const char* fc = getenv("KNN_B200_FORCE_CAPTURE");
        rp.force_capture = fc && atoi(fc) != 0;
    }
    e = cosine ? launch_rescore<kCosine>(cfg, rp, nrows, st) : launch_rescore<kSqEuclidean>(cfg, rp, nrows, st);
    if (e != cudaSuccess) return e;
    ++launches;

    // Rows without a completeness proof: a second tensor pass captures the
    // whole proven band of each such row, then exact re-scoring; only rows
    // whose band overflows the capture buffer are recomputed exactly.
    if ((e = cudaMemcpyAsync(a.host_scratch, scal, 64, cudaMemcpyDeviceToHost, st)) != cudaSuccess) return e;
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
    const uint32_t nfb = *reinterpret_cast<const uint32_t*>(static_cast<const uint8_t*>(a.host_scratch) + 4);
    r.rescored = *reinterpret_cast<const unsigned long long*>(static_cast<const uint8_t*>(a.host_scratch) + 32);
    r.fallback_rows = nfb;
    if (nfb) {
        const CaptureArgs ca{xh,   alpha, rho,   xnorm, gmax,  maxabs,      bmin,    sorted ? perm : nullptr,
                             sorted ? rowpos : nullptr, n,     npad,  kc,    group_tiles, kp >= 128 ? 1024u : 512u,
                             fb_rows, fb_thr, rescored};
        if ((e = run_capture(a, ca, nfb, r, launches)) != cudaSuccess) return e;
    }
    r.launches = launches;
    return cudaSuccess;
}

}  // namespace knnb

#include "tri_shard.cuh"
