// tri_shard.cuh -- the triangle sweep sharded over ranks.
// Included at the end of tensor_path.cu (it launches that file's kernels).
//
// The paper's multi-GPU design computes every unordered pair once across
// the GPUs and merges per-GPU partial lists at the end:
// grid rows go to lanes in boustrophedon order (schedule.cpp:40-44,
// lane_of_row), a lane sweeps the upper-triangle cells of its rows
// (schedule.cpp:56-75) into lane-private heaps for BOTH endpoints
// (engine.cpp:27-56, select.cpp:60-91), and merge_all k-way merges the
// lanes' heaps row by row (merge.cpp:10-78).  Here:
//
//   rank-local   every rank holds the whole reference set (replicated by an
//                NCCL broadcast) and runs the same replicated prep (norm order,
//                fp16 planes, E4M3 planes) -- identical bits on every rank;
//   phase A      the sample pass for a contiguous slice of rows -> their
//                column-side thresholds;  exchange 1: all-gather of the
//                thresholds (2 floats per row);
//   phase O      the second column order (replicated);
//   phase B      the triangle sweep of this rank's 256-row units (boustrophedon
//                over ranks, snake over the CTA pairs): row-side lists for its
//                own rows, column-side candidates for every column appended to
//                warp logs, then binned by the owner of the column;
//   exchange 2   all-to-all of the binned column-side candidates (12 B each);
//   phase C      the owner scatters them into its rows' column-side buffers,
//                selects, and rescores its rows exactly (the merge_row of
//                merge.cpp:10-57: row side + column side, (distance, index)
//                order, one owner per row);  unproven rows take the capture
//                pass locally (it needs no exchange: every rank has all rows);
//   exchange 3   each rank's rows -> contiguous input-order shards
//                (reduce-scatter of zero-filled full arrays: every element has
//                exactly one non-zero contribution, so the sum is exact).
//
// Two drivers share the phases: run_tri_nccl (one rank per GPU, NCCL
// collectives) and run_tri_loopback (all ranks sequentially on one device,
// device copies for the exchanges) -- the latter is how the sharded program
// is tested and its per-rank time measured on a single B200.
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <vector>

namespace knnb {

// schedule.cpp:40-44: r = Y mod 2L; r < L ? r : 2L - 1 - r -- rotated by
// one rank per block of 2L units.  Each rank still takes one unit pair
// (l, 2L - 1 - l) of every block, so the tile counts balance exactly as in
// the reference; the rotation mixes the units' positions inside the second
// column order's 4-unit buckets (sorted by threshold, §3.3), whose first and
// last units hold the rows that need the capture pass.  Without it, at 8
// ranks every such unit fell to ranks 0, 3, 4 and 7 (C3: 1.4k retried rows
// each, none on the others; C5: 233 ms of capture against 24 ms).
static inline uint32_t tri_lane_of_unit(uint32_t u, uint32_t world) {
    const uint32_t r = u % (2 * world);
    const uint32_t l = r < world ? r : 2 * world - 1 - r;
    return (l + u / (2 * world)) % world;
}

// Whether the triangle sweep takes its units from the dynamic queue
// (KNN_B200_TRI_DYN=0: never; =1: always).  Default: the threshold triangle
// (C4: -14%), whose items carry no list state between column groups --
// resident and streamed query rows alike (C3, d = 1024: sweep 893 -> 830 ms
// on the last build, profiles/r02cf_knobs.txt, r02cg_knobs.txt; it measured
// +4% before the band rescore and the epilogue changes).  The list triangle
// keeps the static walk at any world size: its CTA pairs sweep each column
// group in step, so the group's tiles stay L2-resident.  Measured at C2, 8
// emulated ranks (6.6 units per pair): (unit, group) items from the queue
// made pairs wait on another pair's list state and lost that residency
// (sweep +3%); whole-unit claims for the lightest 20% of the tiles after a
// static head, +8% (profiles/r02at_*).
static bool tri_use_dyn(bool tcap, uint32_t kc) {
    (void)kc;
    if (const char* e = getenv("KNN_B200_TRI_DYN")) return atoi(e) != 0;
    return tcap;
}

// Estimated sweep cost of unit u (relative units): its U - u tiles, weighted
// up for the lowest-norm units -- rows near the centroid lie inside many
// columns' thresholds ("hubs") and append column-side candidates on most of
// their tiles.  The shape was fitted to the per-pair sweep times of C2 at 8
// emulated ranks under the plain tile-count deal
// (profiles/r02aq_cta_static.txt: decay over ~0.4% of the rows); the weight
// was then measured: 0 / 0.45 / 0.9 -> C2 at 8 ranks 37.4 / 35.5 / 35.0 ms,
// at 4 ranks 68.1 / 66.2 / 65.8 ms (profiles/r02au_*).  Only the deal
// depends on it, never the results.
static double tri_unit_cost(uint32_t u, uint32_t U) {
    static const double hub = [] {  // tuning: KNN_B200_TRI_HUB = the weight in percent (0: tiles only)
        const char* e = getenv("KNN_B200_TRI_HUB");
        return e ? std::max(0, atoi(e)) / 100.0 : 0.9;
    }();
    const double tau = std::max(1.0, 0.004 * U);
    return double(U - u) * (1.0 + hub * std::exp(-double(u) / tau));
}

// The static walk's deal of a rank's units a (ascending u: cost descending)
// to P CTA pairs: pair p walks positions p, p + P, ...  Round r hands the P
// next-heaviest units to the pairs in ascending order of their cost so far
// (LPT per round, equal unit counts: the snake deal when cost = tiles); the
// pairs that take a unit in a partial last round are then labelled 0, 1, ...
static void lpt_deal(const std::vector<uint32_t>& a, uint32_t U, uint32_t pairs_max, uint32_t* out) {
    const uint32_t m = uint32_t(a.size());
    const uint32_t P = std::max<uint32_t>(1, std::min(m, pairs_max));
    const uint32_t rounds = (m + P - 1) / P;
    std::vector<double> load(P, 0.0);
    std::vector<std::vector<uint32_t>> got(P);
    std::vector<uint32_t> order(P);
    for (uint32_t r = 0; r < rounds; ++r) {
        for (uint32_t q = 0; q < P; ++q) order[q] = q;
        std::stable_sort(order.begin(), order.end(), [&](uint32_t x, uint32_t y) { return load[x] < load[y]; });
        const uint32_t i0 = r * P, cnt = std::min(P, m - i0);
        for (uint32_t q = 0; q < cnt; ++q) {
            got[order[q]].push_back(a[i0 + q]);
            load[order[q]] += tri_unit_cost(a[i0 + q], U);
        }
    }
    std::vector<uint32_t> label;
    for (uint32_t q = 0; q < P; ++q)
        if (got[q].size() == rounds) label.push_back(q);
    for (uint32_t q = 0; q < P; ++q)
        if (got[q].size() != rounds) label.push_back(q);
    for (uint32_t l = 0; l < P; ++l)
        for (uint32_t k = 0; k < got[label[l]].size(); ++k) out[k * P + l] = got[label[l]][k];
}

// Per-rank unit lists.  Units go to ranks in boustrophedon order.  With the
// dynamic queue a rank's units stay ascending (work U - u descending): CTA
// pairs claim them heaviest first, and the units of a column group with work
// are a prefix.  Without it they are dealt to the launch's CTA pairs by
// lpt_deal.
static std::vector<std::vector<uint32_t>> tri_unit_lists(uint32_t U, uint32_t G, uint32_t pairs_max, bool dyn) {
    std::vector<std::vector<uint32_t>> asc(G), out(G);
    for (uint32_t u = 0; u < U; ++u) asc[tri_lane_of_unit(u, G)].push_back(u);
    if (dyn) return asc;
    for (uint32_t r = 0; r < G; ++r) {
        out[r].resize(asc[r].size());
        lpt_deal(asc[r], U, pairs_max, out[r].data());
    }
    return out;
}

// Host-side plan, flattened (the C ABI's knn_b200_tri_unit_plan).
void tri_unit_plan(uint32_t U, uint32_t G, uint32_t pairs_max, uint32_t* units, uint32_t* counts) {
    const auto lists = tri_unit_lists(U, G, pairs_max, tri_use_dyn(false, 1));  // the list triangle's
    uint32_t at = 0;
    for (uint32_t r = 0; r < G; ++r) {
        counts[r] = uint32_t(lists[r].size());
        for (uint32_t u : lists[r]) units[at++] = u;
    }
}

// ---- kernels -----------------------------------------------------------------

// Count the column-side pool entries per owner rank (one block per chunk).
__global__ void tri_bin_count_kernel(const uint32_t* __restrict__ lcol, const uint32_t* __restrict__ lcnt,
                                     const uint32_t* __restrict__ lnext, uint32_t nchunks,
                                     const uint32_t* __restrict__ unit_owner, uint32_t G,
                                     unsigned long long* __restrict__ cnt, unsigned int* __restrict__ overflow) {
    __shared__ uint32_t h[kTriMaxWorld];
    const uint32_t w = blockIdx.x, used = *lnext;
    if (w == 0 && threadIdx.x == 0 && used > nchunks) atomicOr(overflow, 1u);
    if (w >= min(used, nchunks)) return;
    for (uint32_t i = threadIdx.x; i < G; i += blockDim.x) h[i] = 0;
    __syncthreads();
    const uint32_t c = lcnt[w];
    const size_t base = size_t(w) * kLogChunk;
    for (uint32_t i = threadIdx.x; i < c; i += blockDim.x) atomicAdd(&h[unit_owner[lcol[base + i] >> 8]], 1u);
    __syncthreads();
    for (uint32_t o = threadIdx.x; o < G; o += blockDim.x)
        if (h[o]) atomicAdd(cnt + o, (unsigned long long)h[o]);
}

// Exclusive scan of the G counts -> segment offsets; cursors to 0.
__global__ void tri_seg_offsets_kernel(const unsigned long long* __restrict__ cnt, uint32_t G,
                                       unsigned long long* __restrict__ off, unsigned long long* __restrict__ cur) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        unsigned long long s = 0;
        for (uint32_t o = 0; o < G; ++o) {
            off[o] = s;
            cur[o] = 0;
            s += cnt[o];
        }
    }
}

// Place each entry in its owner's segment: key (y', row) and the column's
// slot among the owner's rows (unit_lidx: the unit's position in the
// owner's unit list).  Block-local ranges are reserved with one atomic per
// owner, entries placed with shared-memory atomics.
__global__ void tri_bin_place_kernel(const uint64_t* __restrict__ lkey, const uint32_t* __restrict__ lcol,
                                     const uint32_t* __restrict__ lcnt, const uint32_t* __restrict__ lnext,
                                     uint32_t nchunks, const uint32_t* __restrict__ unit_owner,
                                     const uint32_t* __restrict__ unit_lidx, uint32_t G,
                                     const unsigned long long* __restrict__ off, unsigned long long* __restrict__ cur,
                                     uint64_t* __restrict__ skey, uint32_t* __restrict__ sslot) {
    __shared__ uint32_t h[kTriMaxWorld];
    __shared__ unsigned long long b[kTriMaxWorld];
    const uint32_t w = blockIdx.x;
    if (w >= min(*lnext, nchunks)) return;
    for (uint32_t i = threadIdx.x; i < G; i += blockDim.x) h[i] = 0;
    __syncthreads();
    const uint32_t c = lcnt[w];
    const size_t base = size_t(w) * kLogChunk;
    for (uint32_t i = threadIdx.x; i < c; i += blockDim.x) atomicAdd(&h[unit_owner[lcol[base + i] >> 8]], 1u);
    __syncthreads();
    for (uint32_t o = threadIdx.x; o < G; o += blockDim.x) {
        b[o] = h[o] ? off[o] + atomicAdd(cur + o, (unsigned long long)h[o]) : 0;
        h[o] = 0;
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < c; i += blockDim.x) {
        const uint32_t col = lcol[base + i];
        const uint32_t o = unit_owner[col >> 8];
        const unsigned long long at = b[o] + atomicAdd(&h[o], 1u);
        skey[at] = lkey[base + i];
        sslot[at] = unit_lidx[col >> 8] * 256 + (col & 255);
    }
}

// One rank (no exchange): the pool straight into the per-row buffers, the
// column translated to its slot (unit_lidx: its unit's place in the list).
__global__ void tri_scatter_local_kernel(const uint64_t* __restrict__ lkey, const uint32_t* __restrict__ lcol,
                                         const uint32_t* __restrict__ lcnt, const uint32_t* __restrict__ lnext,
                                         uint32_t nchunks, const uint32_t* __restrict__ unit_lidx,
                                         uint32_t* __restrict__ ccnt, uint64_t* __restrict__ cbuf, uint32_t ccap,
                                         unsigned int* __restrict__ overflow) {
    const uint32_t w = blockIdx.x, used = *lnext;
    if (w == 0 && threadIdx.x == 0 && used > nchunks) atomicOr(overflow, 1u);
    if (w >= min(used, nchunks)) return;
    const uint32_t c = lcnt[w];
    const size_t base = size_t(w) * kLogChunk;
    for (uint32_t i = threadIdx.x; i < c; i += blockDim.x) {
        const uint32_t col = lcol[base + i];
        const uint32_t s = unit_lidx[col >> 8] * 256 + (col & 255);
        const uint32_t at = atomicAdd(ccnt + s, 1u);
        if (at < ccap) cbuf[size_t(s) * ccap + at] = lkey[base + i];
    }
}

// Received column-side entries -> the owner's per-row buffers.
__global__ void tri_scatter_flat_kernel(const uint64_t* __restrict__ rkey, const uint32_t* __restrict__ rslot,
                                        unsigned long long count, uint32_t* __restrict__ ccnt,
                                        uint64_t* __restrict__ cbuf, uint32_t ccap) {
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < count;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        const uint32_t s = rslot[i];
        const uint32_t at = atomicAdd(ccnt + s, 1u);
        if (at < ccap) cbuf[size_t(s) * ccap + at] = rkey[i];
    }
}

// The threshold triangle's per-row capture thresholds (y space) from the fp16
// sample lists: T ~ the row's k-th distance is estimated by the rank-r
// smallest y over the sample columns (r set so that the sample's r-th
// exceeds the true k-th with high probability), and the threshold admits its
// proof band: thr = proof_bound(T) - alpha.  Any
// value is correct -- the capture rescore proves each row or retries it.
// loose: the sample lists' largest y (a retry threshold for rows left with
// fewer than k candidates).
struct TcapThrArgs {
    const uint64_t* cand;  // rows [j0, j1): 2 x 16 sample keys each
    uint32_t n, j0, j1, kp, r, d;
    float unscale;         // sample y -> fp16-plane y (1 / 2^-16 for E4M3 operands)
    const float* alpha;
    const double* rho;
    const double* xnorm;
    const unsigned long long* gmax;
    const unsigned int* maxabs;
    float* thr;
    float* loose;
};

template <int FOLD>
__global__ void tcap_threshold_kernel(const TcapThrArgs t) {
    for (uint32_t j = t.j0 + blockIdx.x * blockDim.x + threadIdx.x; j < t.j1; j += gridDim.x * blockDim.x) {
        float thr = -__int_as_float(0x7f800000), lo = thr;
        if (j < t.n) {
            const uint64_t* c = t.cand + size_t(j - t.j0) * t.kp;
            uint64_t kth = kEmptyKey, last = 0;
            for (uint32_t a = 0; a < t.kp; ++a) {
                uint32_t below = 0;
                for (uint32_t b = 0; b < t.kp; ++b) below += c[b] < c[a];
                if (below == t.r - 1) kth = c[a];
                if (c[a] != kEmptyKey && c[a] > last) last = c[a];
            }
            const double al = double(t.alpha[j]);
            const int e = scale_exponent(*t.maxabs);
            // A space: s^2 D (sqeuclidean), 2 s^2 D (cosine: 2 s^2 (1 - cos))
            const double s2 = (FOLD == kCosine ? 2.0 : 1.0) * ldexp(1.0, 2 * e);
            if (kth == kEmptyKey) {
                thr = __int_as_float(0x7f800000);  // fewer than r sampled columns: admit everything
            } else {
                const double y = double(ordered_to_float(uint32_t(kth >> 32))) * t.unscale;
                const double b1 = proof_bound<FOLD>(t.d, t.maxabs, t.gmax, t.xnorm[j], t.rho[j], al,
                                                    fmax((al + y) / s2, 0.0));
                thr = __double2float_ru(b1 - al);
            }
            lo = last == 0 ? thr : fmaxf(thr, __fmul_rn(ordered_to_float(uint32_t(last >> 32)), t.unscale));
        }
        t.thr[j] = thr;
        t.loose[j] = lo;
    }
}

// ---- state ----------------------------------------------------------------

// Bump allocation inside one block; base == null only measures.
struct Carve {
    uint8_t* base = nullptr;
    size_t off = 0;
    template <class T>
    T* take(size_t count) {
        T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
        off += (count * sizeof(T) + 255) / 256 * 256;
        return p;
    }
};

// Grow-only device memory by purpose (api.cu keeps one buffer per slot).
using ShardAllocFn = ShardAlloc;
// rank r: kSlotRank0 + 4 r + {0: lists and counters, 1: send, 2: receive, 3: count matrix}
enum : int { kSlotShared = 0, kSlotScratch = 1, kSlotRank0 = 2 };
static inline int rank_slot(uint32_t rank, int which) { return kSlotRank0 + 4 * int(rank) + which; }

// Replicated state: identical on every rank (same input, same kernels).
struct TriShared {
    uint32_t n = 0, npad = 0, d = 0, kc = 0, U = 0, G = 1, S = 0;  // S: rows per all-gather slice
    bool tcap = false;    // the threshold triangle (k > 10, any d, cosine too): fp16 sample, 2 x 16 lists
    bool cosine = false;  // no norm order (every norm is 1): identity permutation
    bool dyn = false;     // the sweep takes units from the dynamic queue (tri_use_dyn)
    uint32_t stride = kTriStride, skpl = kTriSampleKpl, trank = kTriRank, sm = 0, spad = 0, skc = 0;
    bool f8 = true;
    float dscale = 1.0f;
    uint32_t group_tiles = 1, gts = 1;
    // common prep (first order = norm order)
    uint8_t* xh;
    float *alpha, *bmin, *mu;
    double *rho, *xnorm, *muacc;
    uint8_t* scal;  // maxabs @0, gmax @8
    unsigned int* maxabs;
    unsigned long long* gmax;
    float *skey, *skey2;
    uint32_t *sidx, *perm, *rowpos;
    void* stemp;
    size_t stemp_bytes = 0;
    // sample pass
    uint32_t* srows;
    uint8_t *xs, *x8;
    float *alpha_s, *bmin_s;
    float *tc2, *tl1;  // [G * S]: each rank's slice, all-gathered
    // second order
    unsigned long long *okey, *okey2;
    uint32_t *oidx, *order;
    void* otmp;
    size_t otemp = 0;
    float *tri_alpha, *tri_tc, *tri_tl, *bmin2, *tcmax;
    double *tri_rho, *tri_xnorm;
    uint32_t* tri_perm;
    uint8_t* xq2;  // the triangle's operand planes (second order)
    // unit tables
    uint32_t *unit_owner, *unit_lidx;
    uint32_t* tri_rowpos;  // input row -> second-order position (threshold triangle)
    std::vector<std::vector<uint32_t>> units_h;

    void layout(Carve& c) {
        xh = c.take<uint8_t>(size_t(kc) * npad * 128);
        alpha = c.take<float>(npad);
        bmin = c.take<float>(2 * (npad / 32));  // + bound halves
        rho = c.take<double>(npad);
        xnorm = c.take<double>(npad);
        muacc = c.take<double>(d);
        mu = c.take<float>(d);
        scal = c.take<uint8_t>(64);
        skey = c.take<float>(n);
        skey2 = c.take<float>(n);
        sidx = c.take<uint32_t>(n);
        perm = c.take<uint32_t>(n);
        rowpos = c.take<uint32_t>(n);
        stemp = c.take<uint8_t>(stemp_bytes);
        srows = c.take<uint32_t>(sm);
        xs = c.take<uint8_t>(size_t(skc) * spad * 128);
        x8 = f8 ? c.take<uint8_t>(size_t(skc) * npad * 128) : nullptr;
        alpha_s = c.take<float>(spad);
        bmin_s = c.take<float>(2 * (spad / 32));
        tc2 = c.take<float>(size_t(G) * S);
        tl1 = c.take<float>(size_t(G) * S);
        okey = c.take<unsigned long long>(n);
        okey2 = c.take<unsigned long long>(n);
        oidx = c.take<uint32_t>(n);
        order = c.take<uint32_t>(n);
        otmp = c.take<uint8_t>(otemp);
        tri_alpha = c.take<float>(npad);
        tri_tc = c.take<float>(npad);
        tri_tl = c.take<float>(npad);
        bmin2 = c.take<float>(2 * (npad / 32));
        tcmax = c.take<float>(2 * (npad / 32));
        tri_rho = c.take<double>(npad);
        tri_xnorm = c.take<double>(npad);
        tri_perm = c.take<uint32_t>(n);
        xq2 = c.take<uint8_t>(size_t(kc) * npad * 128);
        unit_owner = c.take<uint32_t>(U);
        unit_lidx = c.take<uint32_t>(U);
        tri_rowpos = c.take<uint32_t>(tcap ? n : 1);
    }
};

// One rank's persistent state (cand: phase B -> C; send/recv: the exchange).
struct TriRank {
    uint32_t rank = 0;
    uint32_t nu = 0, nslots = 0, s0 = 0, s1 = 0;
    uint32_t* units = nullptr;  // device copy of S.units_h[rank]
    uint64_t* cand = nullptr;   // nslots x 24 row-side lists
    uint64_t* cand_s = nullptr; // (s1 - s0) x 2 skpl sample lists
    uint8_t* scal = nullptr;    // fb_count @4, rescored @32, log overflow @40
    unsigned long long *scnt = nullptr, *soff = nullptr, *scur = nullptr;  // [G]
    uint32_t* fb_rows = nullptr;
    float* fb_thr = nullptr;
    // column-side pool (scratch, phase B)
    uint64_t* lkey = nullptr;
    uint32_t *lcol = nullptr, *lcnt = nullptr, *lnext = nullptr;
    uint32_t nchunks = 0;
    // send segments (by owner) and received entries
    uint64_t* skey = nullptr;
    uint32_t* sslot = nullptr;
    uint64_t* rkey = nullptr;
    uint32_t* rslot = nullptr;
    std::vector<unsigned long long> scnt_h, soff_h;  // [G]
    unsigned long long rcount = 0;
    bool overflow = false;
    TensorPathResult res;
    float ms_a = 0, ms_b = 0, ms_c = 0;
};

// ---- phases ------------------------------------------------------------------

// Replicated prep: norm order, fp16 planes + per-row terms, E4M3 planes, the
// sample columns; unit tables.  Fills S (allocating kSlotShared).
static cudaError_t tri_prep(TriShared& S, const TensorPathArgs& a, uint32_t G, ShardAllocFn alloc, void* actx,
                            bool tcap = false) {
    const uint32_t n = a.n, d = a.d;
    S.tcap = tcap;
    S.cosine = a.fold == kCosine;
    if (tcap) {
        // the sample pass estimates each row's k-th distance: every 16th
        // (k <= 47) or 32nd column, fp16 operands (E4M3 thresholds are
        // noisier: at C4 twice the rows needed a retry), 2 x 16-entry lists,
        // the rank-r value with r ~ k / stride + 2.5 sqrt(k / stride) + 1
        // (tcap_threshold_kernel)
        S.skpl = 16;
        S.f8 = false;  // tuning: KNN_B200_TCAP_E4M3=1 (C4: 2x the retried rows, sweep +0.5 s)
        S.stride = a.klist <= 47 ? 16 : 32;  // tuning: KNN_B200_TCAP_STRIDE
        if (const char* se = getenv("KNN_B200_TCAP_STRIDE")) S.stride = std::max(1, atoi(se));
        if (const char* fe = getenv("KNN_B200_TCAP_E4M3")) S.f8 = atoi(fe) != 0;
        const double m = double(a.klist) / S.stride;
        S.trank = uint32_t(std::min(32.0, std::ceil(m + 2.5 * std::sqrt(m) + 1.0)));
        // each half's list must hold the rank-r value: the shortest list that
        // does (C4: r = 7 -> 8 entries, C3: r = 9 -> 12; fewer insertions and
        // registers than 16)
        S.skpl = S.trank <= 8 ? 8u : S.trank <= 12 ? 12u : 16u;
        if (const char* ke = getenv("KNN_B200_TCAP_SAMPLE_KPL")) S.skpl = atoi(ke) == 16 ? 16u : S.skpl;
    }
    S.n = n;
    S.d = d;
    S.npad = (n + 255) / 256 * 256;
    S.kc = (d + 63) / 64;
    S.U = S.npad / 256;
    S.G = G;
    S.S = (S.U + G - 1) / G * 256;
    if (!tcap) {
        if (const char* se = getenv("KNN_B200_TRI_STRIDE")) S.stride = uint32_t(atoi(se));
        if (const char* ke = getenv("KNN_B200_TRI_SAMPLE_KPL"))
            S.skpl = atoi(ke) == 12 ? 12u : atoi(ke) == 6 ? 6u : S.skpl;
        if (const char* re = getenv("KNN_B200_TRI_RANK")) S.trank = uint32_t(atoi(re));
        S.trank = S.trank < 1 ? 1 : (S.trank > S.skpl ? S.skpl : S.trank);
        if (const char* fe = getenv("KNN_B200_TRI_E4M3")) S.f8 = atoi(fe) != 0;
    } else if (const char* re = getenv("KNN_B200_TCAP_RANK")) {
        S.trank = std::max(1u, std::min(2 * S.skpl, uint32_t(atoi(re))));
    }
    S.skc = S.f8 ? (S.kc + 1) / 2 : S.kc;
    S.sm = (n + S.stride - 1) / S.stride;
    S.spad = (S.sm + 255) / 256 * 256;
    S.dscale = S.f8 ? kE4m3Scale * kE4m3Scale : 1.0f;
    S.stemp_bytes = sort_temp_bytes(n);
    cub::DeviceRadixSort::SortPairs(nullptr, S.otemp, static_cast<const unsigned long long*>(nullptr),
                                    static_cast<unsigned long long*>(nullptr), static_cast<const uint32_t*>(nullptr),
                                    static_cast<uint32_t*>(nullptr), int(n));
    const uint64_t tile_bytes = uint64_t(256) * S.kc * 128;
    uint64_t group_bytes = 40ull << 20;  // a column group's fp16 tiles, sized to stay L2-resident
    if (const char* ge = getenv("KNN_B200_TRI_GROUP_MB")) group_bytes = uint64_t(std::max(1, atoi(ge))) << 20;
    S.group_tiles = uint32_t(std::max<uint64_t>(1, std::min<uint64_t>(group_bytes / tile_bytes, S.U)));
    S.gts = uint32_t(std::max<uint64_t>(1, std::min<uint64_t>((40ull << 20) / (uint64_t(256) * S.skc * 128),
                                                                S.spad / 256)));
    Carve c;
    S.layout(c);
    c.base = static_cast<uint8_t*>(alloc(actx, kSlotShared, c.off));
    if (!c.base) return cudaErrorMemoryAllocation;
    c.off = 0;
    S.layout(c);
    S.maxabs = reinterpret_cast<unsigned int*>(S.scal);
    S.gmax = reinterpret_cast<unsigned long long*>(S.scal + 8);
    S.dyn = tri_use_dyn(tcap, S.kc);
    S.units_h = tri_unit_lists(S.U, G, uint32_t(a.sm_count / 2), S.dyn);
    std::vector<uint32_t> owner(S.U), lidx(S.U);
    for (uint32_t r = 0; r < G; ++r)
        for (uint32_t i = 0; i < S.units_h[r].size(); ++i) {
            owner[S.units_h[r][i]] = r;
            lidx[S.units_h[r][i]] = i;
        }
    cudaStream_t st = a.stream;
    cudaError_t e;
    if ((e = cudaMemcpyAsync(S.unit_owner, owner.data(), S.U * 4, cudaMemcpyHostToDevice, st)) != cudaSuccess) return e;
    if ((e = cudaMemcpyAsync(S.unit_lidx, lidx.data(), S.U * 4, cudaMemcpyHostToDevice, st)) != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(S.scal, 0, 64, st)) != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(S.muacc, 0, size_t(d) * 8, st)) != cudaSuccess) return e;
    if (S.cosine) {  // mu = 0, every norm the same: input order
        if ((e = cudaMemsetAsync(S.mu, 0, size_t(d) * 4, st)) != cudaSuccess) return e;
        iota_stride_kernel<<<a.sm_count, 256, 0, st>>>(S.perm, n, 1);
        iota_stride_kernel<<<a.sm_count, 256, 0, st>>>(S.rowpos, n, 1);
        center_stats_kernel<<<a.sm_count * 8, 256, 0, st>>>(a.X, n, d, S.mu, S.maxabs, nullptr, nullptr,
                                                            vec4_rows(a.X, d));
    } else {
        launch_colmean(a.X, n, d, S.muacc, S.mu, a.sm_count, st);
        center_stats_kernel<<<a.sm_count * 8, 256, 0, st>>>(a.X, n, d, S.mu, S.maxabs, S.skey, S.sidx,
                                                            vec4_rows(a.X, d));
        if ((e = cub::DeviceRadixSort::SortPairs(S.stemp, S.stemp_bytes, S.skey, S.skey2, S.sidx, S.perm, int(n), 0,
                                                 32, st)) != cudaSuccess)
            return e;
        invert_perm_kernel<<<a.sm_count * 4, 256, 0, st>>>(S.perm, n, S.rowpos);
    }
    PrepOut po{S.xh, S.alpha, S.rho, S.xnorm, S.gmax};
    prep_kernel<<<a.sm_count * 8, 256, 0, st>>>(a.X, n, d, S.npad, S.kc, S.mu, S.maxabs, S.cosine ? 1 : 0, S.perm,
                                                  po);
    chunk_min_kernel<<<(S.npad / 32 * 32 + 255) / 256, 256, 0, st>>>(S.alpha, S.npad / 32, S.bmin);
    iota_stride_kernel<<<a.sm_count, 256, 0, st>>>(S.srows, S.sm, S.stride);
    if (S.f8) e4m3_planes_kernel<<<a.sm_count * 8, 256, 0, st>>>(S.xh, S.npad, S.kc, S.skc, S.x8);
    gather_rows_kernel<<<a.sm_count * 4, 256, 0, st>>>(S.f8 ? S.x8 : S.xh, S.npad, S.skc, S.srows, 0, S.sm, S.spad,
                                                       nullptr, S.xs);
    gather_alpha_kernel<<<a.sm_count, 256, 0, st>>>(S.alpha, S.srows, S.sm, S.spad, S.dscale, S.alpha_s);
    chunk_min_kernel<<<(S.spad / 32 * 32 + 255) / 256, 256, 0, st>>>(S.alpha_s, S.spad / 32, S.bmin_s);
    return cudaGetLastError();
}

// Per-rank buffers (rank_slot(r, 0)): units, lists, counters.
static cudaError_t tri_rank_init(TriShared& S, TriRank& R, uint32_t rank, const TensorPathArgs& a, ShardAllocFn alloc,
                                 void* actx) {
    R = TriRank{};
    R.rank = rank;
    R.nu = uint32_t(S.units_h[rank].size());
    R.nslots = R.nu * 256;
    R.s0 = std::min(rank * S.S, S.npad);
    R.s1 = std::min((rank + 1) * S.S, S.npad);
    R.scnt_h.assign(S.G, 0);
    R.soff_h.assign(S.G, 0);
    auto lay = [&](Carve& c) {
        R.units = c.take<uint32_t>(std::max<uint32_t>(R.nu, 1));
        R.cand = c.take<uint64_t>(S.tcap ? 1 : size_t(R.nslots) * 24 + 1);  // the threshold triangle keeps no lists
        R.cand_s = c.take<uint64_t>(size_t(R.s1 - R.s0) * 2 * S.skpl + 1);
        R.scal = c.take<uint8_t>(64);
        R.scnt = c.take<unsigned long long>(S.G);
        R.soff = c.take<unsigned long long>(S.G);
        R.scur = c.take<unsigned long long>(S.G);
        R.fb_rows = c.take<uint32_t>(R.nslots + 1);
        R.fb_thr = c.take<float>(R.nslots + 1);
    };
    Carve c;
    lay(c);
    c.base = static_cast<uint8_t*>(alloc(actx, rank_slot(rank, 0), c.off));
    if (!c.base) return cudaErrorMemoryAllocation;
    c.off = 0;
    lay(c);
    cudaError_t e;
    if (R.nu && (e = cudaMemcpyAsync(R.units, S.units_h[rank].data(), R.nu * 4, cudaMemcpyHostToDevice, a.stream)) !=
                    cudaSuccess)
        return e;
    return cudaMemsetAsync(R.scal, 0, 64, a.stream);
}

// Phase A: sample pass over sorted rows [s0, s1) -> tc2/tl1 there.
static cudaError_t tri_sample(TriShared& S, TriRank& R, const TensorPathArgs& a) {
    if (R.s1 <= R.s0) return cudaSuccess;
    cudaStream_t st = a.stream;
    SweepParams ss{S.xs,     S.alpha_s, S.sm,  S.spad, S.skc,   R.s0, std::min(R.s1, S.n), S.gts, 0,
                   R.cand_s, S.f8 ? S.x8 : S.xh, S.npad, nullptr, nullptr, nullptr, 0, S.bmin_s};
    ss.e4m3 = S.f8;
    const uint32_t rows = R.s1 - R.s0;
    const bool ares = S.skc <= uint32_t(TS_MAX_RES_KC);
    // (d > 256: the query rows stream with every reference chunk, ARES = false)
    cudaError_t e = S.skpl == 16  ? (ares ? launch_sweep_pair<16, 256, 8>(ss, rows, st)
                                          : launch_sweep_pair<16, 256, 8, false, false, false>(ss, rows, st))
                    : S.skpl == 12 ? (ares ? launch_sweep_pair<12, 256, 8>(ss, rows, st)
                                           : launch_sweep_pair<12, 256, 8, false, false, false>(ss, rows, st))
                    : S.skpl == 8  ? (ares ? launch_sweep_pair<8, 256, 8>(ss, rows, st)
                                           : launch_sweep_pair<8, 256, 8, false, false, false>(ss, rows, st))
                    : S.skpl == 6  ? launch_sweep_pair<6, 256, 8>(ss, rows, st)
                                   : launch_sweep_pair<kTriSampleKpl, 256, 8>(ss, rows, st);
    if (e != cudaSuccess) return e;
    if (S.tcap) {
        const TcapThrArgs ta{R.cand_s, S.n,   R.s0,    R.s1,   2 * S.skpl, S.trank, S.d,  1.0f / S.dscale,
                             S.alpha,  S.rho, S.xnorm, S.gmax, S.maxabs,   S.tc2,   S.tl1};
        if (S.cosine) tcap_threshold_kernel<kCosine><<<a.sm_count * 4, 256, 0, st>>>(ta);
        else tcap_threshold_kernel<kSqEuclidean><<<a.sm_count * 4, 256, 0, st>>>(ta);
    } else {
        tri_threshold_kernel<<<a.sm_count * 4, 256, 0, st>>>(R.cand_s, S.n, R.s0, R.s1, 2 * S.skpl, S.trank,
                                                              1.0f / S.dscale, S.tc2, S.tl1);
    }
    return cudaGetLastError();
}

// Phase O (replicated): thresholds sorted within norm buckets; planes and
// per-row arrays gathered into that order.
static cudaError_t tri_order(TriShared& S, const TensorPathArgs& a) {
    cudaStream_t st = a.stream;
    const uint32_t n = S.n, npad = S.npad;
    tri_order_key_kernel<<<a.sm_count * 4, 256, 0, st>>>(S.tc2, n, kTriBucket, S.okey, S.oidx);
    cudaError_t e = cub::DeviceRadixSort::SortPairs(S.otmp, S.otemp, S.okey, S.okey2, S.oidx, S.order, int(n), 0, 64, st);
    if (e != cudaSuccess) return e;
    tri_permute_kernel<<<a.sm_count * 4, 256, 0, st>>>(S.order, n, npad, S.alpha, S.rho, S.xnorm, S.tc2, S.tl1, S.perm,
                                                        S.tri_alpha, S.tri_rho, S.tri_xnorm, S.tri_tc, S.tri_tl,
                                                        S.tri_perm);
    gather_rows_kernel<<<a.sm_count * 4, 256, 0, st>>>(S.xh, npad, S.kc, S.order, 0, n, npad, nullptr, S.xq2);
    chunk_min_kernel<<<(npad / 32 * 32 + 255) / 256, 256, 0, st>>>(S.tri_alpha, npad / 32, S.bmin2);
    chunk_max_kernel<<<(npad / 32 * 32 + 255) / 256, 256, 0, st>>>(S.tri_tc, npad / 32, S.tcmax);
    if (S.tcap) invert_perm_kernel<<<a.sm_count * 4, 256, 0, st>>>(S.tri_perm, n, S.tri_rowpos);
    return cudaGetLastError();
}

// The threshold triangle with 16 epilogue warps (4 per TMEM lane quadrant,
// 64 columns each per tile) instead of 8: twice the warps to hide the
// filter's latency; it keeps no lists, so 112 registers suffice.  The
// default for resident query rows: C4 2.363-2.365 s against 2.375-2.384 s
// with 8, C3 level (profiles/r02cd_ew.txt).  KNN_B200_TCAP_EW=8: 8 warps.
static bool tcap_ew16() {
    const char* e = getenv("KNN_B200_TCAP_EW");
    return !(e && atoi(e) == 8);
}

// Phase B: the triangle sweep of this rank's units; column-side entries
// counted by owner (R.scnt_h, host) -- the caller then sizes the send
// buffers and calls tri_bin.
static cudaError_t tri_sweep(TriShared& S, TriRank& R, const TensorPathArgs& a, ShardAllocFn alloc, void* actx) {
    cudaStream_t st = a.stream;
    cudaError_t e;
    const uint32_t pairs = std::max<uint32_t>(1, std::min<uint32_t>(R.nu, uint32_t(a.sm_count / 2)));
    // the column-side pool: 3x this rank's expected volume (~64 entries per
    // row over the whole triangle; C2 uses 63).  A unit's share lies between "in
    // proportion to its pairs" and "the same for every unit" (a column's
    // candidates come from rows near it in the norm order): take the larger.
    double share_w = 0;
    for (uint32_t u : S.units_h[R.rank]) share_w += double(S.U - u);
    const double total = double(S.U) * (S.U + 1) / 2;
    const double share = std::max(total > 0 ? share_w / total : 1.0, double(R.nu) / double(S.U));
    // the threshold triangle: ~ (r x stride) captured entries per row plus
    // the proof band (tcap_threshold_kernel; C3 ~ 350, C4 ~ 220 per row), 2.5x
    const double per_row = S.tcap ? 2.5 * (double(S.trank) * S.stride + 64.0) : 3.0 * 64.0;  // C2 uses ~63
    uint64_t pool = uint64_t(per_row * double(S.n) * share) + uint64_t(2 * pairs * 8) * kLogChunk;
    if (const char* lce = getenv("KNN_B200_TRI_LOGCAP")) pool = uint64_t(atoi(lce));
    R.nchunks = uint32_t((pool + kLogChunk - 1) / kLogChunk);
    // the dynamic queue's claim counters (one per column group) and per-unit
    // list-state counters
    const uint32_t ngroups = ((S.n + 255) / 256 + S.group_tiles - 1) / S.group_tiles;
    const bool dyn = S.dyn;
    uint32_t* qctr = nullptr;
    auto lay = [&](Carve& c) {
        R.lkey = c.take<uint64_t>(size_t(R.nchunks) * kLogChunk);
        R.lcol = c.take<uint32_t>(size_t(R.nchunks) * kLogChunk);
        R.lcnt = c.take<uint32_t>(size_t(R.nchunks) + 1);
        qctr = c.take<uint32_t>(size_t(ngroups) + R.nu + 1);
    };
    Carve c;
    lay(c);
    c.base = static_cast<uint8_t*>(alloc(actx, kSlotScratch, c.off));
    if (!c.base) return cudaErrorMemoryAllocation;
    c.off = 0;
    lay(c);
    R.lnext = R.lcnt + R.nchunks;
    if ((e = cudaMemsetAsync(R.lnext, 0, 4, st)) != cudaSuccess) return e;
    if (R.nu == 0) {
        std::fill(R.scnt_h.begin(), R.scnt_h.end(), 0ull);
        return cudaSuccess;
    }
    const char* dbg = getenv("KNN_B200_DEBUG_SWEEP");
    SweepParams tp{S.xq2, S.tri_alpha, S.n,    S.npad,  S.kc, 0, S.n, S.group_tiles, dbg ? atoi(dbg) : 0,
                   R.cand, S.xq2,      S.npad, nullptr, nullptr, nullptr, 0, S.bmin2,
                   S.tri_tc, S.tcmax,  R.lkey, R.lcol,  R.lcnt, R.lnext, R.nchunks};
    tp.units = R.units;
    tp.nunits = R.nu;
    if (dyn) {
        if ((e = cudaMemsetAsync(qctr, 0, (size_t(ngroups) + R.nu) * 4, st)) != cudaSuccess) return e;
        tp.qctr = qctr;
        tp.udone = qctr + ngroups;
    }
    // profiling only: per-CTA start/end times of this rank's sweep, appended
    // to the file the variable names (rank, CTA, start ns, end ns, units)
    const char* ctaf = getenv("KNN_B200_DEBUG_CTA_TIMES");
    unsigned long long* cta_ns = nullptr;
    if (ctaf) {
        cudaMallocAsync(reinterpret_cast<void**>(&cta_ns), 2 * 8 * 2 * pairs, st);
        tp.cta_ns = cta_ns;
    }
    const bool ares = S.kc <= uint32_t(TS_MAX_RES_KC);
    if (!S.tcap) e = dyn ? launch_sweep_pair<12, 256, 8, true, false, true, true>(tp, R.nslots, st)
                         : launch_sweep_pair<12, 256, 8, true, false, true, false>(tp, R.nslots, st);
    else if (ares && tcap_ew16()) e = dyn ? launch_sweep_pair<2, 256, 16, true, true, true, true>(tp, R.nslots, st)
                                          : launch_sweep_pair<2, 256, 16, true, true, true, false>(tp, R.nslots, st);
    else if (ares) e = dyn ? launch_sweep_pair<2, 256, 8, true, true, true, true>(tp, R.nslots, st)
                           : launch_sweep_pair<2, 256, 8, true, true, true, false>(tp, R.nslots, st);
    else e = dyn ? launch_sweep_pair<2, 256, 8, true, true, false, true>(tp, R.nslots, st)
                 : launch_sweep_pair<2, 256, 8, true, true, false, false>(tp, R.nslots, st);
    if (e != cudaSuccess) return e;
    if (cta_ns) {
        std::vector<unsigned long long> t(4 * pairs);
        cudaMemcpyAsync(t.data(), cta_ns, t.size() * 8, cudaMemcpyDeviceToHost, st);
        cudaStreamSynchronize(st);
        cudaFreeAsync(cta_ns, st);
        if (FILE* f = fopen(ctaf, "a")) {
            for (uint32_t c = 0; c < 2 * pairs; ++c) {
                uint32_t nu = 0;  // (the static walk's units; the dynamic queue's are not recorded)
                for (size_t i = c / 2; !dyn && i < S.units_h[R.rank].size(); i += pairs) ++nu;
                fprintf(f, "%u %u %llu %llu %u\n", R.rank, c, t[2 * c], t[2 * c + 1], nu);
            }
            fclose(f);
        }
    }
    if (S.G == 1) {  // no exchange: only the pool's overflow matters (phase C scatters it in place)
        uint32_t* h = static_cast<uint32_t*>(a.host_scratch);
        if ((e = cudaMemcpyAsync(h, R.lnext, 4, cudaMemcpyDeviceToHost, st)) != cudaSuccess) return e;
        if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
        R.overflow = h[0] > R.nchunks;
        R.scnt_h[0] = 0;
        return cudaSuccess;
    }
    if ((e = cudaMemsetAsync(R.scnt, 0, size_t(S.G) * 8, st)) != cudaSuccess) return e;
    tri_bin_count_kernel<<<R.nchunks, 256, 0, st>>>(R.lcol, R.lcnt, R.lnext, R.nchunks, S.unit_owner, S.G, R.scnt,
                                                    reinterpret_cast<unsigned int*>(R.scal + 40));
    tri_seg_offsets_kernel<<<1, 32, 0, st>>>(R.scnt, S.G, R.soff, R.scur);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    unsigned long long* h = static_cast<unsigned long long*>(a.host_scratch);  // 64 B pinned: G <= 8 counts
    std::vector<unsigned long long> cnt(S.G);
    for (uint32_t o0 = 0; o0 < S.G; o0 += 7) {
        const uint32_t m = std::min<uint32_t>(7, S.G - o0);
        if ((e = cudaMemcpyAsync(h, R.scnt + o0, m * 8, cudaMemcpyDeviceToHost, st)) != cudaSuccess) return e;
        if ((e = cudaMemcpyAsync(h + 7, R.scal + 40, 4, cudaMemcpyDeviceToHost, st)) != cudaSuccess) return e;
        if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
        for (uint32_t i = 0; i < m; ++i) cnt[o0 + i] = h[i];
        R.overflow = R.overflow || (uint32_t(h[7]) != 0);
    }
    unsigned long long s = 0;
    for (uint32_t o = 0; o < S.G; ++o) {
        R.scnt_h[o] = cnt[o];
        R.soff_h[o] = s;
        s += cnt[o];
    }
    return cudaSuccess;
}

// Phase B, second half: place the entries into their owners' segments.
static cudaError_t tri_bin(TriShared& S, TriRank& R, const TensorPathArgs& a, ShardAllocFn alloc, void* actx) {
    unsigned long long total = 0;
    for (auto c : R.scnt_h) total += c;
    Carve c;
    c.take<uint64_t>(total + 1);
    c.take<uint32_t>(total + 1);
    uint8_t* b = static_cast<uint8_t*>(alloc(actx, rank_slot(R.rank, 1), c.off));
    if (!b) return cudaErrorMemoryAllocation;
    c.base = b;
    c.off = 0;
    R.skey = c.take<uint64_t>(total + 1);
    R.sslot = c.take<uint32_t>(total + 1);
    if (R.nu == 0) return cudaSuccess;
    tri_bin_place_kernel<<<R.nchunks, 256, 0, a.stream>>>(R.lkey, R.lcol, R.lcnt, R.lnext, R.nchunks, S.unit_owner,
                                                          S.unit_lidx, S.G, R.soff, R.scur, R.skey, R.sslot);
    return cudaGetLastError();
}

// Receive buffers for `count` entries (rank_slot(r, 2)).
static cudaError_t tri_recv_alloc(TriRank& R, unsigned long long count, ShardAllocFn alloc, void* actx) {
    Carve c;
    c.take<uint64_t>(count + 1);
    c.take<uint32_t>(count + 1);
    uint8_t* b = static_cast<uint8_t*>(alloc(actx, rank_slot(R.rank, 2), c.off));
    if (!b) return cudaErrorMemoryAllocation;
    c.base = b;
    c.off = 0;
    R.rkey = c.take<uint64_t>(count + 1);
    R.rslot = c.take<uint32_t>(count + 1);
    R.rcount = count;
    return cudaSuccess;
}

// Phase C: the owner's merge (merge.cpp:10-57) -- column-side entries into
// per-row buffers, the best kTriSel of each, and the exact rescore of row
// side + column side; unproven rows through the capture pass.  Outputs go
// to a.out_* at the rows' input positions.
static cudaError_t tcap_finish(TriShared& S, TriRank& R, const TensorPathArgs& a, ShardAllocFn alloc, void* actx);

static cudaError_t tri_finish(TriShared& S, TriRank& R, const TensorPathArgs& a, ShardAllocFn alloc, void* actx) {
    cudaStream_t st = a.stream;
    cudaError_t e;
    if (R.nu == 0) return cudaSuccess;
    if (S.tcap) return tcap_finish(S, R, a, alloc, actx);
    uint64_t* cbuf;
    uint32_t* ccnt;
    uint64_t* sel;
    uint32_t* selcnt;
    float* selbound;
    auto lay = [&](Carve& c) {
        cbuf = c.take<uint64_t>(size_t(R.nslots) * kTriCap);
        ccnt = c.take<uint32_t>(R.nslots);
        sel = c.take<uint64_t>(size_t(R.nslots) * kTriSel);
        selcnt = c.take<uint32_t>(R.nslots);
        selbound = c.take<float>(R.nslots);
    };
    Carve c;
    lay(c);
    // one rank scatters its pool directly, so the pool (kSlotScratch) must
    // outlive this allocation: use the (unused) receive slot instead
    const int slot = S.G == 1 ? rank_slot(R.rank, 2) : kSlotScratch;
    c.base = static_cast<uint8_t*>(alloc(actx, slot, c.off));
    if (!c.base) return cudaErrorMemoryAllocation;
    c.off = 0;
    lay(c);
    if ((e = cudaMemsetAsync(ccnt, 0, size_t(R.nslots) * 4, st)) != cudaSuccess) return e;
    if (S.G == 1)
        tri_scatter_local_kernel<<<R.nchunks, 256, 0, st>>>(R.lkey, R.lcol, R.lcnt, R.lnext, R.nchunks, S.unit_lidx,
                                                            ccnt, cbuf, kTriCap,
                                                            reinterpret_cast<unsigned int*>(R.scal + 40));
    else if (R.rcount)
        tri_scatter_flat_kernel<<<a.sm_count * 8, 256, 0, st>>>(R.rkey, R.rslot, R.rcount, ccnt, cbuf, kTriCap);
    remap_kernel<<<a.sm_count * 8, 256, 0, st>>>(R.cand, size_t(R.nslots) * 24, S.tri_perm, S.n);
    remap_capture_kernel<<<R.nslots, 128, 0, st>>>(cbuf, ccnt, R.nslots, kTriCap, S.tri_perm);
    tri_select_kernel<<<(R.nslots * 32 + 255) / 256, 256, 0, st>>>(cbuf, ccnt, kTriCap, R.nslots, S.tri_tc, sel, selcnt,
                                                                     selbound, R.units);
    uint32_t* fb_count = reinterpret_cast<uint32_t*>(R.scal + 4);
    unsigned long long* rescored = reinterpret_cast<unsigned long long*>(R.scal + 32);
    RescoreParams rp{a.X,        S.n,      a.d,        a.klist,     24,     0,        R.nslots, R.cand,
                     S.tri_alpha, S.tri_rho, S.tri_xnorm, S.gmax, S.maxabs, a.fold,  a.out_sqrt, a.out_index,
                     a.out_dist,  fb_count, R.fb_rows, R.fb_thr, rescored, 0,       nullptr};
    if (const char* fc = getenv("KNN_B200_FORCE_CAPTURE")) rp.force_capture = atoi(fc) != 0;
    rp.rowperm = S.tri_perm;
    rp.xbuf = sel;
    rp.xcnt = selcnt;
    rp.xbound = selbound;
    rp.xcap = S.tri_tl;
    rp.units = R.units;
    const dim3 grid((R.nslots + 7) / 8);
    rescore_kernel<kSqEuclidean, 24, 2, kTriSel><<<grid, 256, 0, st>>>(rp);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    if ((e = cudaMemcpyAsync(a.host_scratch, R.scal, 64, cudaMemcpyDeviceToHost, st)) != cudaSuccess) return e;
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
    const uint32_t nfb = *reinterpret_cast<const uint32_t*>(static_cast<const uint8_t*>(a.host_scratch) + 4);
    R.res.rescored = *reinterpret_cast<const unsigned long long*>(static_cast<const uint8_t*>(a.host_scratch) + 32);
    R.res.fallback_rows = nfb;
    R.res.launches += 6;
    if (nfb) {
        const auto tr0 = std::chrono::steady_clock::now();
        const CaptureArgs ca{S.xh,    S.alpha,  S.rho, S.xnorm, S.gmax,        S.maxabs, S.bmin, S.perm, S.rowpos,
                             S.n,     S.npad,   S.kc,  S.group_tiles, 512u, R.fb_rows, R.fb_thr, rescored};
        if ((e = run_capture(a, ca, nfb, R.res, R.res.launches)) != cudaSuccess) return e;
        if (getenv("KNN_B200_DEBUG_FB")) {  // profiling only: per-rank capture rows and time
            cudaStreamSynchronize(st);
            fprintf(stderr, "[tri_finish] rank %u capture %u rows, %.2f ms\n", R.rank, nfb,
                    std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tr0).count());
        }
    }
    return cudaSuccess;
}

// ---- drivers -------------------------------------------------------------------

static float ev_ms(cudaEvent_t x, cudaEvent_t y) {
    float m = 0;
    cudaEventElapsedTime(&m, x, y);
    return m;
}

// All ranks, one after another, on a.stream's device; the exchanges are
// device copies.  a.out_* (n x klist) receive every row.  rank_ms (optional,
// world x 4): per rank [replicated prep + order, phase A, phase B, phase C]
// in ms (CUDA events); exchange volume per rank in xbytes (optional, world).
cudaError_t run_tri_loopback(const TensorPathArgs& a, uint32_t G, ShardAllocFn alloc, void* actx,
                             TensorPathResult& r, float* rank_ms, unsigned long long* xbytes, bool* overflow,
                             bool tcap) {
    cudaStream_t st = a.stream;
    cudaError_t e;
    TriShared S;
    std::vector<TriRank> R(G);
    cudaEvent_t ev[8];
    for (auto& x : ev) cudaEventCreate(&x);
    auto done = [&](cudaError_t err) {
        for (auto& x : ev) cudaEventDestroy(x);
        return err;
    };
    cudaEventRecord(ev[0], st);
    if ((e = tri_prep(S, a, G, alloc, actx, tcap)) != cudaSuccess) return done(e);
    for (uint32_t g = 0; g < G; ++g)
        if ((e = tri_rank_init(S, R[g], g, a, alloc, actx)) != cudaSuccess) return done(e);
    cudaEventRecord(ev[1], st);
    if (a.ev_sweep0) cudaEventRecord(a.ev_sweep0, st);  // the sweep phase: sample pass + order + triangle
    std::vector<float> ms_a(G), ms_b(G), ms_c(G);
    for (uint32_t g = 0; g < G; ++g) {  // phase A; exchange 1 is implicit (shared tc2/tl1)
        cudaEventRecord(ev[2], st);
        if ((e = tri_sample(S, R[g], a)) != cudaSuccess) return done(e);
        cudaEventRecord(ev[3], st);
        cudaEventSynchronize(ev[3]);
        ms_a[g] = ev_ms(ev[2], ev[3]);
    }
    cudaEventRecord(ev[4], st);
    if ((e = tri_order(S, a)) != cudaSuccess) return done(e);
    cudaEventRecord(ev[5], st);
    bool ovf = false;
    for (uint32_t g = 0; g < G; ++g) {  // phase B (the logs are per-rank scratch, binned at once)
        cudaEventRecord(ev[2], st);
        if ((e = tri_sweep(S, R[g], a, alloc, actx)) != cudaSuccess) return done(e);
        if (G > 1 && (e = tri_bin(S, R[g], a, alloc, actx)) != cudaSuccess) return done(e);
        cudaEventRecord(ev[3], st);
        cudaEventSynchronize(ev[3]);
        ms_b[g] = ev_ms(ev[2], ev[3]);
        ovf = ovf || R[g].overflow;
    }
    if (a.ev_sweep1) cudaEventRecord(a.ev_sweep1, st);
    if (overflow) *overflow = ovf;
    if (ovf) return done(cudaSuccess);  // the caller redoes the call without the triangle
    if (getenv("KNN_B200_DEBUG_SWEEP_ONLY")) {  // profiling only: phase timings up to the sweep, no results
        if (rank_ms)
            for (uint32_t g = 0; g < G; ++g) {
                rank_ms[4 * g + 0] = ev_ms(ev[0], ev[1]) + ev_ms(ev[4], ev[5]);
                rank_ms[4 * g + 1] = ms_a[g];
                rank_ms[4 * g + 2] = ms_b[g];
                rank_ms[4 * g + 3] = 0;
            }
        return done(cudaSuccess);
    }
    // exchange 2: rank o receives segment [g -> o] of every rank g, in rank order
    for (uint32_t o = 0; o < G && G > 1; ++o) {
        unsigned long long cnt = 0;
        for (uint32_t g = 0; g < G; ++g) cnt += R[g].scnt_h[o];
        if ((e = tri_recv_alloc(R[o], cnt, alloc, actx)) != cudaSuccess) return done(e);
        unsigned long long at = 0;
        for (uint32_t g = 0; g < G; ++g) {
            const unsigned long long m = R[g].scnt_h[o];
            if (!m) continue;
            if ((e = cudaMemcpyAsync(R[o].rkey + at, R[g].skey + R[g].soff_h[o], m * 8, cudaMemcpyDeviceToDevice,
                                     st)) != cudaSuccess)
                return done(e);
            if ((e = cudaMemcpyAsync(R[o].rslot + at, R[g].sslot + R[g].soff_h[o], m * 4, cudaMemcpyDeviceToDevice,
                                     st)) != cudaSuccess)
                return done(e);
            at += m;
        }
        if (xbytes) {  // bytes rank o sends to its peers
            unsigned long long sent = 0;
            for (uint32_t p = 0; p < G; ++p)
                if (p != o) sent += R[o].scnt_h[p] * 12;
            xbytes[o] = sent;
        }
    }
    for (uint32_t g = 0; g < G; ++g) {  // phase C
        cudaEventRecord(ev[2], st);
        if ((e = tri_finish(S, R[g], a, alloc, actx)) != cudaSuccess) return done(e);
        cudaEventRecord(ev[3], st);
        cudaEventSynchronize(ev[3]);
        ms_c[g] = ev_ms(ev[2], ev[3]);
        r.rescored += R[g].res.rescored;
        r.fallback_rows += R[g].res.fallback_rows;
        r.exact_rows += R[g].res.exact_rows;
        r.launches += R[g].res.launches;
    }
    r.launches += 20 + 6 * G;
    const float ms_rep = ev_ms(ev[0], ev[1]) + ev_ms(ev[4], ev[5]);
    if (rank_ms)
        for (uint32_t g = 0; g < G; ++g) {
            rank_ms[4 * g + 0] = ms_rep;
            rank_ms[4 * g + 1] = ms_a[g];
            rank_ms[4 * g + 2] = ms_b[g];
            rank_ms[4 * g + 3] = ms_c[g];
        }
    return done(cudaSuccess);
}

static cudaError_t nccl_err(ncclResult_t x) { return x == ncclSuccess ? cudaSuccess : cudaErrorUnknown; }

// One rank of G (one GPU each) over an NCCL communicator.  a.out_* are full
// n x klist arrays (padded to G * ceil(n / G) rows); on return this rank's
// rows hold its results and every other row is 0 -- the caller's
// reduce-scatter then leaves each rank with its contiguous shard.
// *overflow: some rank's column-side logs overflowed (all ranks agree).
cudaError_t run_tri_nccl(const TensorPathArgs& a, ncclComm_t comm, uint32_t rank, uint32_t G, ShardAllocFn alloc,
                         void* actx, TensorPathResult& r, bool* overflow, bool tcap) {
    cudaStream_t st = a.stream;
    cudaError_t e;
    TriShared S;
    TriRank R;
    if ((e = tri_prep(S, a, G, alloc, actx, tcap)) != cudaSuccess) return e;
    if ((e = tri_rank_init(S, R, rank, a, alloc, actx)) != cudaSuccess) return e;
    if (a.ev_sweep0) cudaEventRecord(a.ev_sweep0, st);  // the sweep phase: sample pass + order + triangle
    if ((e = tri_sample(S, R, a)) != cudaSuccess) return e;
    // exchange 1: every rank's threshold slice (S rows) to every rank, in place
    if ((e = nccl_err(ncclGroupStart())) != cudaSuccess) return e;
    ncclAllGather(S.tc2 + size_t(rank) * S.S, S.tc2, S.S, ncclFloat32, comm, st);
    ncclAllGather(S.tl1 + size_t(rank) * S.S, S.tl1, S.S, ncclFloat32, comm, st);
    if ((e = nccl_err(ncclGroupEnd())) != cudaSuccess) return e;
    if ((e = tri_order(S, a)) != cudaSuccess) return e;
    if ((e = tri_sweep(S, R, a, alloc, actx)) != cudaSuccess) return e;
    if (G == 1) {  // one rank: the pool goes straight to the merge (no exchange 2)
        if (a.ev_sweep1) cudaEventRecord(a.ev_sweep1, st);
        *overflow = R.overflow;
        if (R.overflow) return cudaSuccess;
        if ((e = tri_finish(S, R, a, alloc, actx)) != cudaSuccess) return e;
        r = R.res;
        r.launches += 20;
        return cudaSuccess;
    }
    if ((e = tri_bin(S, R, a, alloc, actx)) != cudaSuccess) return e;
    if (a.ev_sweep1) cudaEventRecord(a.ev_sweep1, st);
    // exchange 2a: the G x (G + 1) count matrix (last column: overflow flag)
    std::vector<unsigned long long> mine(G + 1), all(size_t(G) * (G + 1));
    for (uint32_t o = 0; o < G; ++o) mine[o] = R.scnt_h[o];
    mine[G] = R.overflow ? 1 : 0;
    auto* dm = static_cast<unsigned long long*>(alloc(actx, rank_slot(rank, 3), size_t(G) * (G + 1) * 8));
    if (!dm) return cudaErrorMemoryAllocation;
    if ((e = cudaMemcpyAsync(dm + size_t(rank) * (G + 1), mine.data(), (G + 1) * 8, cudaMemcpyHostToDevice, st)) !=
        cudaSuccess)
        return e;
    if ((e = nccl_err(ncclAllGather(dm + size_t(rank) * (G + 1), dm, G + 1, ncclUint64, comm, st))) != cudaSuccess)
        return e;
    if ((e = cudaMemcpyAsync(all.data(), dm, all.size() * 8, cudaMemcpyDeviceToHost, st)) != cudaSuccess) return e;
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
    bool ovf = false;
    for (uint32_t g = 0; g < G; ++g) ovf = ovf || all[size_t(g) * (G + 1) + G] != 0;
    *overflow = ovf;
    if (ovf) return cudaSuccess;
    unsigned long long rc = 0;
    std::vector<unsigned long long> roff(G);
    for (uint32_t g = 0; g < G; ++g) {
        roff[g] = rc;
        rc += all[size_t(g) * (G + 1) + rank];
    }
    if ((e = tri_recv_alloc(R, rc, alloc, actx)) != cudaSuccess) return e;
    // exchange 2b: all-to-all of the column-side entries (keys, then slots)
    if ((e = nccl_err(ncclGroupStart())) != cudaSuccess) return e;
    for (uint32_t p = 0; p < G; ++p) {
        const unsigned long long sc = R.scnt_h[p], rcnt = all[size_t(p) * (G + 1) + rank];
        if (sc) {
            ncclSend(R.skey + R.soff_h[p], sc * 8, ncclUint8, int(p), comm, st);
            ncclSend(R.sslot + R.soff_h[p], sc * 4, ncclUint8, int(p), comm, st);
        }
        if (rcnt) {
            ncclRecv(R.rkey + roff[p], rcnt * 8, ncclUint8, int(p), comm, st);
            ncclRecv(R.rslot + roff[p], rcnt * 4, ncclUint8, int(p), comm, st);
        }
    }
    if ((e = nccl_err(ncclGroupEnd())) != cudaSuccess) return e;
    if ((e = tri_finish(S, R, a, alloc, actx)) != cudaSuccess) return e;
    r = R.res;
    r.launches += 26;
    return cudaSuccess;
}

// ---- the threshold triangle (one GPU) ---------------------------------------

// Whole problems with 10 < min(k, n-1) <= 128 (and past the size crossover):
// every unordered pair once, both endpoints against fixed thresholds from an
// fp16 sample pass (no lists), each row's captured candidates rescored
// exactly with the band-capture proof; rows it cannot prove get a second
// capture pass with the threshold their candidates imply.
bool tcap_eligible(uint32_t n, uint32_t d, uint32_t klist) {
    const char* te = getenv("KNN_B200_TCAP");
    if (te && strcmp(te, "0") == 0) return false;
    const bool force = te && strcmp(te, "force") == 0;
    (void)d;
    return klist > 10 && klist <= 128 && (force ? n >= 512 : n >= 262144);
}

static uint32_t tcap_cap(uint32_t klist) {
    if (const char* e = getenv("KNN_B200_TCAP_CAP")) return uint32_t(std::max(64, std::min(2048, atoi(e))));
    (void)klist;
    return 1024u;  // C4 (k = 32): 512 sent 2x more rows to the retry pass
}

// Slot s of a rank's rows (second-order position units[s / 256] * 256 +
// s % 256): its input row (or ~0 for padding) and its capture threshold.
__global__ void tcap_slots_kernel(const uint32_t* __restrict__ units, uint32_t nslots, uint32_t n,
                                  const uint32_t* __restrict__ tri_perm, const float* __restrict__ tri_tc,
                                  uint32_t* __restrict__ rows, float* __restrict__ thr) {
    for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < nslots; s += gridDim.x * blockDim.x) {
        const uint32_t pos = units[s >> 8] * 256 + (s & 255);
        rows[s] = pos < n ? tri_perm[pos] : 0xffffffffu;
        thr[s] = pos < n ? tri_tc[pos] : 0.0f;
    }
}

// Phase C of the threshold triangle: this rank's rows' captured candidates
// (pool entries (y, other endpoint) -> per-row buffers), the exact capture
// rescore with its proof, and a second capture pass for the rows it retries.
static cudaError_t tcap_finish(TriShared& S, TriRank& R, const TensorPathArgs& a, ShardAllocFn alloc, void* actx) {
    cudaStream_t st = a.stream;
    cudaError_t e;
    const uint32_t cap = tcap_cap(a.klist);
    uint64_t* cbuf;
    uint32_t *ccnt, *rows, *fb_count, *big;
    float* thr;
    auto lay = [&](Carve& c) {
        cbuf = c.take<uint64_t>(size_t(R.nslots) * cap);
        ccnt = c.take<uint32_t>(R.nslots);
        rows = c.take<uint32_t>(R.nslots);
        thr = c.take<float>(R.nslots);
        fb_count = c.take<uint32_t>(16);  // [0]: retried rows, [8]: second-pass bands
        big = c.take<uint32_t>(R.nslots);
    };
    Carve c;
    lay(c);
    const int slot = S.G == 1 ? rank_slot(R.rank, 2) : kSlotScratch;  // one rank: the pool is still live
    c.base = static_cast<uint8_t*>(alloc(actx, slot, c.off));
    if (!c.base) return cudaErrorMemoryAllocation;
    c.off = 0;
    lay(c);
    if ((e = cudaMemsetAsync(ccnt, 0, size_t(R.nslots) * 4, st)) != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(fb_count, 0, 64, st)) != cudaSuccess) return e;
    if (S.G == 1)
        tri_scatter_local_kernel<<<R.nchunks, 256, 0, st>>>(R.lkey, R.lcol, R.lcnt, R.lnext, R.nchunks, S.unit_lidx,
                                                            ccnt, cbuf, cap,
                                                            reinterpret_cast<unsigned int*>(R.scal + 40));
    else if (R.rcount)
        tri_scatter_flat_kernel<<<a.sm_count * 8, 256, 0, st>>>(R.rkey, R.rslot, R.rcount, ccnt, cbuf, cap);
    remap_capture_kernel<<<R.nslots, 128, 0, st>>>(cbuf, ccnt, R.nslots, cap, S.tri_perm);
    tcap_slots_kernel<<<a.sm_count * 4, 256, 0, st>>>(R.units, R.nslots, S.n, S.tri_perm, S.tri_tc, rows, thr);
    unsigned long long* rescored = reinterpret_cast<unsigned long long*>(R.scal + 32);
    Rescore2Params r2{a.X,  S.n, a.d,        a.klist,     0,          rows,     R.nslots, ccnt,
                      cbuf, cap, a.out_sqrt, a.out_index, a.out_dist, fb_count, R.fb_rows, rescored,
                      thr,  S.tri_rowpos, S.tri_alpha, S.tri_rho, S.tri_xnorm, S.gmax, S.maxabs};
    r2.retry_thr = R.fb_thr;
    r2.loose = S.tri_tl;
    r2.big = big;
    r2.nbig = fb_count + 8;
    // the typical band: the sample's rank-r window plus the proof band (~64)
    const uint32_t expect = S.trank * S.stride + 64;
    e = a.fold == kCosine ? launch_rescore_capture<kCosine>(r2, R.nslots, st, expect)
                          : launch_rescore_capture<kSqEuclidean>(r2, R.nslots, st, expect);
    if (e != cudaSuccess) return e;
    uint32_t* h = static_cast<uint32_t*>(a.host_scratch);
    if ((e = cudaMemcpyAsync(h, fb_count, 4, cudaMemcpyDeviceToHost, st)) != cudaSuccess) return e;
    if ((e = cudaMemcpyAsync(h + 2, rescored, 8, cudaMemcpyDeviceToHost, st)) != cudaSuccess) return e;
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
    const uint32_t nretry = h[0];
    R.res.rescored = *reinterpret_cast<const unsigned long long*>(h + 2);
    R.res.fallback_rows = nretry;
    R.res.launches += 5;
    // profiling only: per-rank retried rows and the retry pass's time
    const bool dbg_fb = getenv("KNN_B200_DEBUG_FB") != nullptr;
    const auto tr0 = std::chrono::steady_clock::now();
    if (nretry == 0) {
        if (dbg_fb) fprintf(stderr, "[tcap_finish] rank %u retried 0\n", R.rank);
        return cudaSuccess;
    }
    // second capture pass: the retried rows against their implied thresholds,
    // with room for wider bands (rows that filled their first buffer)
    const CaptureArgs ca{S.xh, S.alpha, S.rho, S.xnorm, S.gmax, S.maxabs, S.bmin, S.cosine ? nullptr : S.perm,
                         S.cosine ? nullptr : S.rowpos, S.n, S.npad, S.kc, S.group_tiles, 2048u, R.fb_rows,
                         R.fb_thr, rescored};
    e = run_capture(a, ca, nretry, R.res, R.res.launches);
    if (dbg_fb) {
        cudaStreamSynchronize(st);
        fprintf(stderr, "[tcap_finish] rank %u retried %u, retry pass %.2f ms\n", R.rank, nretry,
                std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tr0).count());
    }
    return e;
}

}  // namespace knnb
