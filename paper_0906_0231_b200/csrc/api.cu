// api.cu -- the C ABI (include/knn_b200.h): contexts, workspace, dispatch.
//
// Mirrors the control flow of knn::solve_knn (src/engine.cpp:13-68) on the
// device: argument checks -> validation (before any compute) -> Phase 1+2
// fused sweep per row shard -> results.  The reference's per-lane HeapStore +
// merge_all (engine.cpp:27-59) has no counterpart: each query row is owned by
// exactly one CTA, so its list is final when the sweep ends.
#include <cuda_runtime.h>
#include <fcntl.h>
#include <nccl.h>
#include <stdint.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <map>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <type_traits>
#include <vector>

#include "../../include/knn_b200.h"
#include "common.cuh"
#include "kernels.h"

namespace {

thread_local std::string g_last_error;

struct Status {
    int code;
    std::string msg;
};

struct KnnError {
    int code;
    std::string msg;
};

[[noreturn]] void fail(int code, const std::string& msg) { throw KnnError{code, msg}; }

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) fail(KNN_B200_ERR_INTERNAL, std::string(what) + ": " + cudaGetErrorString(e));
}

template <typename Fn>
int guarded(Fn&& fn) {
    try {
        fn();
        return KNN_B200_OK;
    } catch (const KnnError& e) {
        g_last_error = e.msg;
        return e.code;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return KNN_B200_ERR_INTERNAL;
    }
}

struct DevBuf {
    void* ptr = nullptr;
    size_t bytes = 0;
    void* get(size_t want) {
        if (want > bytes) {
            if (ptr) cudaFree(ptr);
            ptr = nullptr;
            bytes = 0;
            cuda_check(cudaMalloc(&ptr, want ? want : 16), "cudaMalloc workspace");
            bytes = want ? want : 16;
        }
        return ptr;
    }
    void release() {
        if (ptr) cudaFree(ptr);
        ptr = nullptr;
        bytes = 0;
    }
};

std::string fmt_value(float v) {
    // std::to_string(float) formatting, as the reference message uses.
    return std::to_string(v);
}

}  // namespace

// Pinned staging for host buffers the caller did not pin (the drop-in's
// Dataset is a std::vector): kStageThreads host threads each own two pinned
// chunks and a copy stream; a thread memcpys chunk c into one buffer while
// the DMA of the other is in flight, so the copy runs at the PCIe rate
// instead of the driver's pageable path (C2: 1 GB in ~90 ms -> ~20 ms).
constexpr int kStageThreads = 16;  // lanes allocated at most; 12 used by default
constexpr int kStageThreadsDefault = 12;
constexpr size_t kStageChunkDefault = size_t(4) << 20;
constexpr size_t kStageMin = size_t(16) << 20;  // smaller copies: plain cudaMemcpyAsync
struct StageLane {
    void* buf[2] = {nullptr, nullptr};
    cudaStream_t st = nullptr;
    cudaEvent_t ev[2] = {nullptr, nullptr};
    cudaEvent_t done = nullptr;
};

struct knn_b200_ctx {
    int device = 0;
    int sm_count = 148;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev[6] = {};  // [0..3] call phases, [4..5] around the sweep kernel
    DevBuf vectors, staged, flags, out_index, out_dist, tensor_ws, exact_ws, capture_ws;
    // Recorded on the working stream at the end of every call; the next call's
    // stream waits on it first, so a call on another stream never touches the
    // workspace while the previous call's kernels are still in flight.
    cudaEvent_t busy = nullptr;
    bool busy_recorded = false;
    // sharded triangle (tri_shard.cuh): grow-only buffers by slot, the full
    // padded result arrays before the reduce-scatter, and the communicator
    std::map<int, DevBuf> shard_ws;
    DevBuf full_index, full_dist, shard_index, shard_dist;
    ncclComm_t comm = nullptr;
    int comm_rank = 0, comm_world = 1;
    bool comm_owned = false;
    unsigned long long* host_flags = nullptr;  // pinned
    StageLane stage[kStageThreads];
    cudaEvent_t stage_go = nullptr;
    bool stage_ready = false;
    int stage_n = kStageThreadsDefault;     // tuning: KNN_B200_STAGE_THREADS
    size_t stage_chunk = kStageChunkDefault;  // tuning: KNN_B200_STAGE_CHUNK_MB
    std::mutex mu;
};

namespace {

void stage_init(knn_b200_ctx* ctx) {
    if (ctx->stage_ready) return;
    if (const char* e = getenv("KNN_B200_STAGE_THREADS")) ctx->stage_n = std::max(1, std::min(atoi(e), kStageThreads));
    if (const char* e = getenv("KNN_B200_STAGE_CHUNK_MB")) ctx->stage_chunk = size_t(std::max(1, atoi(e))) << 20;
    cuda_check(cudaEventCreateWithFlags(&ctx->stage_go, cudaEventDisableTiming), "stage event");
    for (int t = 0; t < ctx->stage_n; ++t) {
        StageLane& l = ctx->stage[t];
        for (int b = 0; b < 2; ++b) {
            cuda_check(cudaHostAlloc(&l.buf[b], ctx->stage_chunk, cudaHostAllocDefault), "cudaHostAlloc staging");
            cuda_check(cudaEventCreateWithFlags(&l.ev[b], cudaEventDisableTiming), "stage event");
        }
        cuda_check(cudaStreamCreateWithFlags(&l.st, cudaStreamNonBlocking), "stage stream");
        cuda_check(cudaEventCreateWithFlags(&l.done, cudaEventDisableTiming), "stage event");
    }
    ctx->stage_ready = true;
}

void stage_free(knn_b200_ctx* ctx) {
    if (!ctx->stage_ready) return;
    for (auto& l : ctx->stage) {
        for (int b = 0; b < 2; ++b) {
            if (l.buf[b]) cudaFreeHost(l.buf[b]);
            if (l.ev[b]) cudaEventDestroy(l.ev[b]);
        }
        if (l.st) cudaStreamDestroy(l.st);
        if (l.done) cudaEventDestroy(l.done);
    }
    cudaEventDestroy(ctx->stage_go);
    ctx->stage_ready = false;
}

bool host_pinned(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

// One host<->device copy: `dst` and `src` are the host and device sides
// as the direction says.
struct CopySeg {
    void* dst;
    const void* src;
    size_t bytes;
};

// Copy host buffers to or from device memory, ordered on `s` (it starts
// after the work already queued on s, and work queued on s afterwards sees
// the data).  Pinned or small host buffers go straight to the DMA engine;
// pageable ones through the staging lanes, all segments' chunks dealt over
// the lanes together (the two output arrays share one pipelined pass).  D2H
// returns with the data in host memory.
void host_copy_segs(knn_b200_ctx* ctx, const std::vector<CopySeg>& segs, bool h2d, cudaStream_t s,
                    int threads = 0) {
    std::vector<CopySeg> staged;
    bool direct_d2h = false;
    for (const CopySeg& g : segs) {
        if (g.bytes == 0) continue;
        const void* host = h2d ? g.src : g.dst;
        if (g.bytes < kStageMin || host_pinned(host)) {
            cuda_check(cudaMemcpyAsync(g.dst, g.src, g.bytes, h2d ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost, s),
                       h2d ? "H2D" : "D2H");
            direct_d2h |= !h2d;
        } else {
            staged.push_back(g);
        }
    }
    if (staged.empty()) {
        if (direct_d2h) cuda_check(cudaStreamSynchronize(s), "D2H sync");
        return;
    }
    stage_init(ctx);
    threads = threads > 0 ? std::min(threads, ctx->stage_n) : ctx->stage_n;
    size_t total = 0;
    for (const CopySeg& g : staged) total += g.bytes;
    // H2D uses the lane buffers whole.  D2H is shorter (C2: 80 MB), so its
    // chunks shrink until every lane pipelines at least four of them.
    size_t chunk = ctx->stage_chunk;
    if (!h2d) {
        const size_t want = (total / (size_t(threads) * 4) + 4095) / 4096 * 4096;
        chunk = std::max<size_t>(size_t(256) << 10, std::min(chunk, want));
    }
    struct Chunk {
        char* dst;
        const char* src;
        size_t len;
    };
    std::vector<Chunk> chunks;
    for (const CopySeg& g : staged)
        for (size_t off = 0; off < g.bytes; off += chunk)
            chunks.push_back({static_cast<char*>(g.dst) + off, static_cast<const char*>(g.src) + off,
                              std::min(chunk, g.bytes - off)});
    const size_t nchunks = chunks.size();
    cuda_check(cudaEventRecord(ctx->stage_go, s), "stage event");
    std::vector<cudaError_t> errs(threads, cudaSuccess);
    auto work = [&](int t) {
        StageLane& l = ctx->stage[t];
        cudaError_t e = cudaSetDevice(ctx->device);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(l.st, ctx->stage_go, 0);
        size_t i = 0;
        const Chunk* prev = nullptr;
        for (size_t c = t; c < nchunks && e == cudaSuccess; c += threads, ++i) {
            const int b = int(i & 1);
            const Chunk& k = chunks[c];
            if (h2d) {
                if (i >= 2) e = cudaEventSynchronize(l.ev[b]);  // the DMA that last read buf[b]
                if (e != cudaSuccess) break;
                std::memcpy(l.buf[b], k.src, k.len);
                e = cudaMemcpyAsync(k.dst, l.buf[b], k.len, cudaMemcpyHostToDevice, l.st);
                if (e == cudaSuccess) e = cudaEventRecord(l.ev[b], l.st);
            } else {
                e = cudaMemcpyAsync(l.buf[b], k.src, k.len, cudaMemcpyDeviceToHost, l.st);
                if (e == cudaSuccess) e = cudaEventRecord(l.ev[b], l.st);
                if (e == cudaSuccess && prev) {  // the previous chunk out of the other buffer
                    e = cudaEventSynchronize(l.ev[b ^ 1]);
                    if (e == cudaSuccess) std::memcpy(prev->dst, l.buf[b ^ 1], prev->len);
                }
                prev = &k;
            }
        }
        if (!h2d && e == cudaSuccess && prev) {
            e = cudaEventSynchronize(l.ev[(i - 1) & 1]);
            if (e == cudaSuccess) std::memcpy(prev->dst, l.buf[(i - 1) & 1], prev->len);
        }
        if (e == cudaSuccess) e = cudaEventRecord(l.done, l.st);
        errs[t] = e;
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < threads; ++t) pool.emplace_back(work, t);
    work(0);
    for (auto& th : pool) th.join();
    for (auto e : errs) cuda_check(e, h2d ? "staged H2D" : "staged D2H");
    for (int t = 0; t < threads; ++t) cuda_check(cudaStreamWaitEvent(s, ctx->stage[t].done, 0), "stage join");
    if (direct_d2h) cuda_check(cudaStreamSynchronize(s), "D2H sync");
}

void host_copy(knn_b200_ctx* ctx, void* dst, const void* src, size_t bytes, bool h2d, cudaStream_t s,
               int threads = 0) {
    host_copy_segs(ctx, {CopySeg{dst, src, bytes}}, h2d, s, threads);
}

// A file's byte range [off, off + bytes) to device memory, ordered on `s`:
// the staging lanes pread chunks into their pinned buffers and DMA them, so
// the read runs in parallel and overlaps the copies (the reference reads the
// whole file into a std::vector first, io.cpp:35-46).
void file_to_device(knn_b200_ctx* ctx, int fd, uint64_t off, void* dst, size_t bytes, cudaStream_t s,
                    const std::string& path) {
    if (bytes == 0) return;
    stage_init(ctx);
    const int threads = ctx->stage_n;
    const size_t chunk = ctx->stage_chunk;
    const size_t nchunks = (bytes + chunk - 1) / chunk;
    cuda_check(cudaEventRecord(ctx->stage_go, s), "stage event");
    std::vector<cudaError_t> errs(threads, cudaSuccess);
    std::vector<int> ioerr(threads, 0);
    auto work = [&](int t) {
        StageLane& l = ctx->stage[t];
        cudaError_t e = cudaSetDevice(ctx->device);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(l.st, ctx->stage_go, 0);
        size_t i = 0;
        for (size_t c = t; c < nchunks && e == cudaSuccess && !ioerr[t]; c += threads, ++i) {
            const int b = int(i & 1);
            const size_t pos = c * chunk, len = std::min(chunk, bytes - pos);
            if (i >= 2) e = cudaEventSynchronize(l.ev[b]);  // the DMA that last read buf[b]
            if (e != cudaSuccess) break;
            size_t got = 0;
            while (got < len) {
                const ssize_t r = pread(fd, static_cast<char*>(l.buf[b]) + got, len - got, off_t(off + pos + got));
                if (r <= 0) {
                    ioerr[t] = 1;
                    break;
                }
                got += size_t(r);
            }
            if (ioerr[t]) break;
            e = cudaMemcpyAsync(static_cast<char*>(dst) + pos, l.buf[b], len, cudaMemcpyHostToDevice, l.st);
            if (e == cudaSuccess) e = cudaEventRecord(l.ev[b], l.st);
        }
        if (e == cudaSuccess) e = cudaEventRecord(l.done, l.st);
        errs[t] = e;
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < threads; ++t) pool.emplace_back(work, t);
    work(0);
    for (auto& th : pool) th.join();
    for (int t = 0; t < threads; ++t) {
        cuda_check(errs[t], "file staging");
        if (ioerr[t]) fail(KNN_B200_ERR_IO, "failed to read '" + path + "'");
    }
    for (int t = 0; t < threads; ++t) cuda_check(cudaStreamWaitEvent(s, ctx->stage[t].done, 0), "stage join");
}

// KNNV header (io.cpp:64-88): magic "KNNV", u32 version (kFormatVersion = 1),
// u32 n, u32 d, little endian, then n x d f32; the reference's messages.
struct KnnvHeader {
    uint32_t n, d;
};
KnnvHeader read_knnv_header(int fd, const std::string& path) {
    struct stat sb;
    if (fstat(fd, &sb) != 0) fail(KNN_B200_ERR_IO, "failed to read '" + path + "'");
    const uint64_t size = uint64_t(sb.st_size);
    if (size < 16) fail(KNN_B200_ERR_IO, "'" + path + "' is too short to hold a dataset header");
    unsigned char h[16];
    if (pread(fd, h, 16, 0) != 16) fail(KNN_B200_ERR_IO, "failed to read '" + path + "'");
    if (std::memcmp(h, "KNNV", 4) != 0) fail(KNN_B200_ERR_IO, "'" + path + "' is not a dataset file (bad magic)");
    auto u32 = [&](int o) {
        return uint32_t(h[o]) | uint32_t(h[o + 1]) << 8 | uint32_t(h[o + 2]) << 16 | uint32_t(h[o + 3]) << 24;
    };
    if (u32(4) != 1)
        fail(KNN_B200_ERR_IO, "'" + path + "' has unsupported format version " + std::to_string(u32(4)));
    KnnvHeader hd{u32(8), u32(12)};
    const uint64_t expect = 16 + uint64_t(hd.n) * hd.d * 4;
    if (size != expect)
        fail(KNN_B200_ERR_IO, "'" + path + "' holds " + std::to_string(size) + " bytes but the header implies " +
                                  std::to_string(expect));
    return hd;
}

struct Fd {
    int fd;
    explicit Fd(const std::string& path) : fd(open(path.c_str(), O_RDONLY)) {
        if (fd < 0) fail(KNN_B200_ERR_IO, "cannot open '" + path + "' for reading");
    }
    ~Fd() { close(fd); }
};

const char* metric_name(int metric) {
    switch (metric) {
    case KNN_B200_METRIC_HELLINGER: return "hellinger";
    case KNN_B200_METRIC_SQEUCLIDEAN: return "sqeuclidean";
    case KNN_B200_METRIC_COSINE: return "cosine";
    case KNN_B200_METRIC_EUCLIDEAN: return "euclidean";
    case KNN_B200_METRIC_MANHATTAN: return "manhattan";
    case KNN_B200_METRIC_ROOT_SQUARES: return "root_of_squares";
    default: return "?";
    }
}

// The device fold of a metric id (kernels: common.cuh).
int fold_of(int metric) {
    switch (metric) {
    case KNN_B200_METRIC_COSINE: return knnb::kCosine;
    case KNN_B200_METRIC_MANHATTAN: return knnb::kManhattan;
    case KNN_B200_METRIC_ROOT_SQUARES: return knnb::kRootSquares;
    default: return knnb::kSqEuclidean;  // sqeuclidean, euclidean, sqrt-staged hellinger
    }
}

// Folds the TENSOR filter's completeness proof covers.
bool tensor_fold(int metric) { return metric <= KNN_B200_METRIC_EUCLIDEAN; }

void check_args(uint32_t n, uint32_t d, uint32_t k, int metric, int arith) {
    // engine.cpp:15 (k), schedule.cpp:12 (n), dataset.cpp:13-19 (n, d)
    if (k < 1) fail(KNN_B200_ERR_CONFIG, "k must be at least 1");
    if (n < 2) fail(KNN_B200_ERR_CONFIG, "n must be at least 2, got " + std::to_string(n));
    if (d < 1) fail(KNN_B200_ERR_CONFIG, "dataset dimension must be at least 1");
    if (metric < 0 || metric > 5) fail(KNN_B200_ERR_CONFIG, "unknown metric id " + std::to_string(metric));
    if (arith < 0 || arith > 2) fail(KNN_B200_ERR_CONFIG, "unknown arithmetic policy " + std::to_string(arith));
    // any k: lists longer than the fused kernels hold (kExactMaxK) take the
    // sort-based EXACT path (exact_bigk.cu), as HeapStore holds min(k, n-1)
    // for any k (heap.cpp:66-70)
}

struct Counters {
    uint32_t launches = 0;
    uint64_t distance_evals = 0;
    uint64_t rescored = 0;
    uint32_t fallback_rows = 0;
    uint32_t exact_rows = 0;
    int arith_used = KNN_B200_ARITH_EXACT;
};

// Device validation of the whole reference set (host copy of two flags; this
// synchronises, as the reference validates before its timer, engine.cpp:23).
void validate_device(knn_b200_ctx* ctx, const float* X, uint32_t n, uint32_t d, int metric,
                     cudaStream_t stream, Counters& ctr) {
    auto* flags = static_cast<unsigned long long*>(ctx->flags.get(2 * sizeof(unsigned long long)));
    cuda_check(cudaMemsetAsync(flags, 0xff, 2 * sizeof(unsigned long long), stream), "memset flags");
    const uint64_t count = uint64_t(n) * d;
    cuda_check(knnb::launch_validate(X, count, metric == KNN_B200_METRIC_HELLINGER, flags, ctx->sm_count,
                                     stream),
               "validate launch");
    ++ctr.launches;
    cuda_check(cudaMemcpyAsync(ctx->host_flags, flags, 2 * sizeof(unsigned long long),
                               cudaMemcpyDeviceToHost, stream),
               "flags D2H");
    cuda_check(cudaStreamSynchronize(stream), "validate sync");
    const unsigned long long bad_nf = ctx->host_flags[0], bad_dom = ctx->host_flags[1];
    const unsigned long long none = ~0ull;
    if (bad_nf != none) {
        // dataset.cpp:25-27
        fail(KNN_B200_ERR_VALIDATION, "non-finite coordinate " + std::to_string(bad_nf % d) + " in vector " +
                                          std::to_string(bad_nf / d));
    }
    if (bad_dom != none) {
        float v = 0;
        cuda_check(cudaMemcpy(&v, X + bad_dom, sizeof(float), cudaMemcpyDeviceToHost), "value D2H");
        // distance.cpp:41-45
        fail(KNN_B200_ERR_VALIDATION, "coordinate " + std::to_string(bad_dom % d) + " of vector " +
                                          std::to_string(bad_dom / d) + " (value " + fmt_value(v) +
                                          ") is outside the domain of " + metric_name(metric));
    }
}

void* shard_alloc(void* c, int slot, size_t bytes);

// Validation + staging + the row-shard sweep, all enqueued on `stream`.
void solve_rows_core(knn_b200_ctx* ctx, const float* X, uint32_t n, uint32_t d, uint32_t k, int metric,
                     int arith, uint32_t row_begin, uint32_t row_end, uint32_t* out_index, float* out_dist,
                     cudaStream_t stream, Counters& ctr) {
    validate_device(ctx, X, n, d, metric, stream, ctr);
    if (row_end == row_begin) return;  // an empty shard: validated, nothing to compute
    const float* Xs = X;
    if (metric == KNN_B200_METRIC_HELLINGER) {
        float* staged = static_cast<float*>(ctx->staged.get(size_t(n) * d * sizeof(float)));
        cuda_check(knnb::launch_stage_sqrt(X, staged, uint64_t(n) * d, ctx->sm_count, stream), "stage launch");
        ++ctr.launches;
        Xs = staged;
    }
    const uint32_t klist = std::min(k, n - 1);
    const int fold = fold_of(metric);
    const int out_sqrt = metric == KNN_B200_METRIC_EUCLIDEAN;
    if (klist > knnb::kExactMaxK) {  // long lists: sort-based EXACT path
        ctr.arith_used = KNN_B200_ARITH_EXACT;
        ctr.distance_evals += uint64_t(row_end - row_begin) * n;
        void* ws = ctx->exact_ws.get(knnb::exact_bigk_workspace_bytes(row_end - row_begin, n, 0));
        cuda_check(cudaEventRecord(ctx->ev[4], stream), "event");
        cuda_check(knnb::launch_exact_bigk(fold, 0, Xs, n, d, klist, row_begin, row_end, out_index, out_dist,
                                           out_sqrt, ws, ctx->sm_count, stream),
                   "exact long-list launch");
        cuda_check(cudaEventRecord(ctx->ev[5], stream), "event");
        ctr.launches += 3 * ((row_end - row_begin + knnb::exact_bigk_batch_rows(row_end - row_begin, n) - 1) /
                             knnb::exact_bigk_batch_rows(row_end - row_begin, n));
        return;
    }
    const uint32_t kp = knnb::tensor_kp_for(klist);
    // AUTO: the tensor filter pays off once the sweep dominates its fixed
    // prologue; both policies return identical bits.
    // (the custom-functor folds run EXACT whatever the policy asks: the
    // filter's proof covers the sqeuclidean and cosine forms only)
    const bool tensor = kp != 0 && tensor_fold(metric) &&
                        (arith == KNN_B200_ARITH_TENSOR || (arith == KNN_B200_ARITH_AUTO && n >= 4096));
    ctr.distance_evals += uint64_t(row_end - row_begin) * n;
    if (tensor) {
        ctr.arith_used = KNN_B200_ARITH_TENSOR;
        knnb::TensorPathArgs ta{};
        ta.X = Xs;
        ta.n = n;
        ta.d = d;
        ta.klist = klist;
        ta.kp = kp;
        ta.row_begin = row_begin;
        ta.row_end = row_end;
        ta.fold = fold;
        ta.out_sqrt = out_sqrt;
        ta.out_index = out_index;
        ta.out_dist = out_dist;
        // the rectangular sweep's workspace, allocated only if that path runs
        // (whole problems take a triangle, which uses the slot buffers)
        ta.alloc_ws = [](void* c, size_t bytes) -> void* {
            try {
                return static_cast<knn_b200_ctx*>(c)->tensor_ws.get(bytes);
            } catch (...) {
                return nullptr;
            }
        };
        ta.host_scratch = ctx->host_flags + 4;
        ta.exact_scratch = ctx->exact_ws.get(std::max<size_t>(
            16, knnb::exact_scratch_bytes(row_end - row_begin, n, klist, ctx->sm_count)));
        ta.sm_count = ctx->sm_count;
        ta.stream = stream;
        ta.ev_sweep0 = ctx->ev[4];
        ta.ev_sweep1 = ctx->ev[5];
        ta.alloc2 = [](void* c, size_t bytes) -> void* {
            try {
                return static_cast<knn_b200_ctx*>(c)->capture_ws.get(bytes);
            } catch (...) {
                return nullptr;
            }
        };
        ta.alloc2_ctx = ctx;
        ta.shard_alloc = shard_alloc;
        ta.shard_ctx = ctx;
        knnb::TensorPathResult tr;
        cuda_check(knnb::run_tensor_path(ta, tr), "tensor path");
        ctr.launches += tr.launches;
        ctr.rescored += tr.rescored;
        ctr.fallback_rows += tr.fallback_rows;
        ctr.exact_rows += tr.exact_rows;
        return;
    }
    ctr.arith_used = KNN_B200_ARITH_EXACT;
    cuda_check(cudaEventRecord(ctx->ev[4], stream), "event");
    void* xs = ctx->exact_ws.get(std::max<size_t>(16, knnb::exact_scratch_bytes(row_end - row_begin, n, klist,
                                                                                   ctx->sm_count)));
    cuda_check(knnb::launch_exact_fused(fold, Xs, n, d, klist, nullptr, row_begin, row_end, out_index, out_dist,
                                        out_sqrt, 0, xs, ctx->sm_count, stream),
               "exact sweep launch");
    cuda_check(cudaEventRecord(ctx->ev[5], stream), "event");
    ++ctr.launches;
}

// KNN_DOUBLE_ACCUM rows: validation + staging + the FP64 EXACT sweep of query
// rows [row_begin, row_end), enqueued on `stream`.
void solve_rows_core_f64(knn_b200_ctx* ctx, const float* X, uint32_t n, uint32_t d, uint32_t k, int metric,
                         uint32_t row_begin, uint32_t row_end, uint32_t* out_index, double* out_dist,
                         cudaStream_t stream, Counters& ctr) {
    validate_device(ctx, X, n, d, metric, stream, ctr);
    if (row_end == row_begin) return;
    const float* Xs = X;
    if (metric == KNN_B200_METRIC_HELLINGER) {
        float* staged = static_cast<float*>(ctx->staged.get(size_t(n) * d * sizeof(float)));
        cuda_check(knnb::launch_stage_sqrt(X, staged, uint64_t(n) * d, ctx->sm_count, stream), "stage launch");
        ++ctr.launches;
        Xs = staged;
    }
    const int fold = fold_of(metric);
    const uint32_t klist = std::min(k, n - 1);
    ctr.arith_used = KNN_B200_ARITH_EXACT;
    ctr.distance_evals += uint64_t(row_end - row_begin) * n;
    cuda_check(cudaEventRecord(ctx->ev[4], stream), "event");
    if (klist > knnb::kExactMaxK) {
        void* ws = ctx->exact_ws.get(knnb::exact_bigk_workspace_bytes(row_end - row_begin, n, 1));
        cuda_check(knnb::launch_exact_bigk(fold, 1, Xs, n, d, klist, row_begin, row_end, out_index, out_dist,
                                           metric == KNN_B200_METRIC_EUCLIDEAN, ws, ctx->sm_count, stream),
                   "exact f64 long-list launch");
    } else {
        cuda_check(knnb::launch_exact_f64(fold, Xs, n, d, klist, row_begin, row_end, out_index, out_dist,
                                          metric == KNN_B200_METRIC_EUCLIDEAN, stream),
                   "exact f64 sweep launch");
    }
    cuda_check(cudaEventRecord(ctx->ev[5], stream), "event");
    ++ctr.launches;
}

// ---- sharded triangle (tri_shard.cuh) ----------------------

void* shard_alloc(void* c, int slot, size_t bytes) {
    try {
        return static_cast<knn_b200_ctx*>(c)->shard_ws[slot].get(bytes);
    } catch (...) {
        return nullptr;
    }
}

void* capture_alloc(void* c, size_t bytes) {
    try {
        return static_cast<knn_b200_ctx*>(c)->capture_ws.get(bytes);
    } catch (...) {
        return nullptr;
    }
}

// The TENSOR-path arguments of a whole-problem triangle solve whose results
// land in full n-row arrays out_index / out_dist.
knnb::TensorPathArgs tri_args(knn_b200_ctx* ctx, const float* Xs, uint32_t n, uint32_t d, uint32_t klist, int metric,
                              uint32_t* out_index, float* out_dist, cudaStream_t stream) {
    knnb::TensorPathArgs ta{};
    ta.X = Xs;
    ta.n = n;
    ta.d = d;
    ta.klist = klist;
    ta.kp = knnb::tensor_kp_for(klist);
    ta.row_begin = 0;
    ta.row_end = n;
    ta.fold = fold_of(metric);
    ta.out_sqrt = metric == KNN_B200_METRIC_EUCLIDEAN;
    ta.out_index = out_index;
    ta.out_dist = out_dist;
    ta.host_scratch = ctx->host_flags + 4;
    ta.exact_scratch = ctx->exact_ws.get(std::max<size_t>(16, knnb::exact_scratch_bytes(n, n, klist, ctx->sm_count)));
    ta.sm_count = ctx->sm_count;
    ta.stream = stream;
    ta.ev_sweep0 = ctx->ev[4];
    ta.ev_sweep1 = ctx->ev[5];
    ta.alloc2 = capture_alloc;
    ta.alloc2_ctx = ctx;
    return ta;
}

// Which triangle a whole problem takes: 0 none, 1 the list triangle (k <= 10),
// 2 the threshold triangle (10 < k <= 128).
int tri_selected(uint32_t n, uint32_t d, uint32_t klist, int metric, int arith) {
    if (arith == KNN_B200_ARITH_EXACT || klist > knnb::kExactMaxK || !tensor_fold(metric)) return 0;
    if (knnb::tensor_kp_for(klist) != 0 &&
        knnb::tri_eligible(n, d, klist, metric == KNN_B200_METRIC_COSINE ? knnb::kCosine : knnb::kSqEuclidean))
        return 1;
    return knnb::tcap_eligible(n, d, klist) ? 2 : 0;
}

// Rows of rank `rank` of `world`: [R rank, R (rank + 1)) clipped to n, R = ceil(n / world).
void shard_rows(uint32_t n, int rank, int world, uint32_t& r0, uint32_t& r1) {
    const uint32_t R = uint32_t((uint64_t(n) + world - 1) / world);
    r0 = uint32_t(std::min<uint64_t>(uint64_t(R) * rank, n));
    r1 = uint32_t(std::min<uint64_t>(uint64_t(r0) + R, n));
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) fail(KNN_B200_ERR_INTERNAL, std::string(what) + ": " + ncclGetErrorString(r));
}

// One rank of a sharded solve on an NCCL communicator (world > 1): the whole
// problem is solved across the ranks, this rank's contiguous shard of rows
// (shard_rows) lands in out_index / out_dist (device).  Triangle-eligible
// problems compute each unordered pair once across all ranks
// (run_tri_nccl + a reduce-scatter of the rows); everything else -- and a
// triangle whose column-side logs overflow -- solves its row shard directly
// (rectangular sweep: each pair of the shard against all n).
void solve_sharded_core(knn_b200_ctx* ctx, ncclComm_t comm, int rank, int world, const float* X, uint32_t n,
                        uint32_t d, uint32_t k, int metric, int arith, uint32_t* out_index, float* out_dist,
                        cudaStream_t stream, Counters& ctr) {
    uint32_t r0, r1;
    shard_rows(n, rank, world, r0, r1);
    const uint32_t klist = std::min(k, n - 1);
    const int mode = tri_selected(n, d, klist, metric, arith);
    if (!mode) {
        solve_rows_core(ctx, X, n, d, k, metric, arith, r0, r1, out_index, out_dist, stream, ctr);
        return;
    }
    validate_device(ctx, X, n, d, metric, stream, ctr);
    const float* Xs = X;
    if (metric == KNN_B200_METRIC_HELLINGER) {
        float* staged = static_cast<float*>(ctx->staged.get(size_t(n) * d * sizeof(float)));
        cuda_check(knnb::launch_stage_sqrt(X, staged, uint64_t(n) * d, ctx->sm_count, stream), "stage launch");
        ++ctr.launches;
        Xs = staged;
    }
    const uint32_t R = uint32_t((uint64_t(n) + world - 1) / world);
    const size_t full = size_t(R) * world * klist;  // rows padded to world x R for the reduce-scatter
    auto* fi = static_cast<uint32_t*>(ctx->full_index.get(full * 4));
    auto* fd = static_cast<float*>(ctx->full_dist.get(full * 4));
    cuda_check(cudaMemsetAsync(fi, 0, full * 4, stream), "memset");
    cuda_check(cudaMemsetAsync(fd, 0, full * 4, stream), "memset");
    knnb::TensorPathArgs ta = tri_args(ctx, Xs, n, d, klist, metric, fi, fd, stream);
    knnb::TensorPathResult tr;
    bool overflow = false;
    cuda_check(knnb::run_tri_nccl(ta, comm, uint32_t(rank), uint32_t(world), shard_alloc, ctx, tr, &overflow,
                                  mode == 2),
               "sharded triangle");
    ctr.arith_used = KNN_B200_ARITH_TENSOR;
    ctr.launches += tr.launches;
    ctr.rescored += tr.rescored;
    ctr.fallback_rows += tr.fallback_rows;
    ctr.exact_rows += tr.exact_rows;
    ctr.distance_evals += uint64_t(n) * (n - 1) / 2 / world;  // about this rank's share of the pairs
    if (overflow) {  // pathological data: every rank solves its rows with the rectangular sweep
        solve_rows_core(ctx, X, n, d, k, metric, arith == KNN_B200_ARITH_AUTO ? KNN_B200_ARITH_TENSOR : arith, r0, r1,
                        out_index, out_dist, stream, ctr);
        return;
    }
    // exchange 3: rows to their contiguous shards.  Every element of the
    // full arrays is written by exactly one rank and 0 elsewhere; u32 + 0 and
    // f32 + (+0) are exact (no result is -0.0), so a sum is the gather.
    const size_t rc = size_t(R) * klist;
    auto* si = static_cast<uint32_t*>(ctx->shard_index.get(rc * 4 + 4));
    auto* sd = static_cast<float*>(ctx->shard_dist.get(rc * 4 + 4));
    nccl_check(ncclGroupStart(), "ncclGroupStart");
    nccl_check(ncclReduceScatter(fi, si, rc, ncclUint32, ncclSum, comm, stream), "ncclReduceScatter");
    nccl_check(ncclReduceScatter(fd, sd, rc, ncclFloat32, ncclSum, comm, stream), "ncclReduceScatter");
    nccl_check(ncclGroupEnd(), "ncclGroupEnd");
    const size_t mine = size_t(r1 - r0) * klist;
    if (mine) {
        cuda_check(cudaMemcpyAsync(out_index, si, mine * 4, cudaMemcpyDeviceToDevice, stream), "D2D");
        cuda_check(cudaMemcpyAsync(out_dist, sd, mine * 4, cudaMemcpyDeviceToDevice, stream), "D2D");
    }
}

void fill_stats(knn_b200_stats* st, const Counters& ctr, uint64_t pairs, int ndev) {
    if (!st) return;
    st->pair_evaluations = pairs;
    st->distance_evals = ctr.distance_evals;
    st->rescored = ctr.rescored;
    st->fallback_rows = ctr.fallback_rows;
    st->exact_rows = ctr.exact_rows;
    st->kernel_launches = ctr.launches;
    st->arith_used = ctr.arith_used;
    st->n_devices = ndev;
}

// Order a call after the context's previous one (which may have left
// kernels in flight on another stream) and mark its end on `s`.
void begin_call(knn_b200_ctx* ctx, cudaStream_t s) {
    if (ctx->busy_recorded) cuda_check(cudaStreamWaitEvent(s, ctx->busy, 0), "wait for the previous call");
}
void end_call(knn_b200_ctx* ctx, cudaStream_t s) {
    cuda_check(cudaEventRecord(ctx->busy, s), "record call end");
    ctx->busy_recorded = true;
}

float elapsed_ms(cudaEvent_t a, cudaEvent_t b) {
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    return ms;
}

}  // namespace

extern "C" {

int knn_b200_abi_version(void) { return KNN_B200_ABI_VERSION; }

const char* knn_b200_last_error(void) { return g_last_error.c_str(); }

int knn_b200_device_count(int* out_count) {
    return guarded([&] {
        int n = 0;
        cudaError_t e = cudaGetDeviceCount(&n);
        if (e != cudaSuccess) n = 0;
        int ok = 0;
        for (int i = 0; i < n; ++i) {
            cudaDeviceProp p;
            if (cudaGetDeviceProperties(&p, i) == cudaSuccess && p.major == 10) ++ok;
        }
        *out_count = ok;
    });
}

int knn_b200_create(int device, knn_b200_ctx** out_ctx) {
    return guarded([&] {
        *out_ctx = nullptr;
        int ndev = 0;
        cuda_check(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount (no CUDA device; there is no CPU fallback)");
        if (device < 0 || device >= ndev)
            fail(KNN_B200_ERR_CONFIG, "device " + std::to_string(device) + " out of range (" +
                                          std::to_string(ndev) + " visible)");
        cudaDeviceProp p;
        cuda_check(cudaGetDeviceProperties(&p, device), "cudaGetDeviceProperties");
        if (p.major != 10)
            fail(KNN_B200_ERR_INTERNAL, std::string("device ") + p.name + " is sm_" + std::to_string(p.major) +
                                            std::to_string(p.minor) + "; this build targets sm_100a only");
        auto* ctx = new knn_b200_ctx();
        ctx->device = device;
        ctx->sm_count = p.multiProcessorCount;
        cuda_check(cudaSetDevice(device), "cudaSetDevice");
        cuda_check(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking), "cudaStreamCreate");
        for (auto& e : ctx->ev) cuda_check(cudaEventCreate(&e), "cudaEventCreate");
        cuda_check(cudaEventCreateWithFlags(&ctx->busy, cudaEventDisableTiming), "cudaEventCreate");
        cuda_check(cudaMallocHost(&ctx->host_flags, 16 * sizeof(unsigned long long)), "cudaMallocHost");
        *out_ctx = ctx;
    });
}

void knn_b200_destroy(knn_b200_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    ctx->vectors.release();
    ctx->staged.release();
    ctx->flags.release();
    ctx->out_index.release();
    ctx->out_dist.release();
    ctx->tensor_ws.release();
    ctx->exact_ws.release();
    ctx->capture_ws.release();
    for (auto& kv : ctx->shard_ws) kv.second.release();
    ctx->full_index.release();
    ctx->full_dist.release();
    ctx->shard_index.release();
    ctx->shard_dist.release();
    if (ctx->comm && ctx->comm_owned) ncclCommDestroy(ctx->comm);
    if (ctx->host_flags) cudaFreeHost(ctx->host_flags);
    stage_free(ctx);
    for (auto& e : ctx->ev)
        if (e) cudaEventDestroy(e);
    if (ctx->busy) cudaEventDestroy(ctx->busy);
    if (ctx->stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
}

int knn_b200_solve(knn_b200_ctx* ctx, const float* host_vectors, uint32_t n, uint32_t d, uint32_t k,
                   int metric, int arith, uint32_t* out_index, float* out_dist, knn_b200_stats* stats) {
    return guarded([&] {
        if (!ctx) fail(KNN_B200_ERR_CONFIG, "null context");
        check_args(n, d, k, metric, arith);
        std::lock_guard<std::mutex> lock(ctx->mu);
        const auto t0 = std::chrono::steady_clock::now();
        cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
        const uint32_t klist = std::min(k, n - 1);
        const size_t vec_bytes = size_t(n) * d * sizeof(float);
        const size_t out_elems = size_t(n) * klist;
        float* X = static_cast<float*>(ctx->vectors.get(vec_bytes));
        auto* oi = static_cast<uint32_t*>(ctx->out_index.get(out_elems * sizeof(uint32_t)));
        auto* od = static_cast<float*>(ctx->out_dist.get(out_elems * sizeof(float)));
        Counters ctr;
        cudaStream_t s = ctx->stream;
        begin_call(ctx, s);
        cuda_check(cudaEventRecord(ctx->ev[0], s), "event");
        host_copy(ctx, X, host_vectors, vec_bytes, true, s);
        cuda_check(cudaEventRecord(ctx->ev[1], s), "event");
        solve_rows_core(ctx, X, n, d, k, metric, arith, 0, n, oi, od, s, ctr);
        cuda_check(cudaEventRecord(ctx->ev[2], s), "event");
        cuda_check(cudaEventSynchronize(ctx->ev[2]), "solve sync");
        const auto t_d2h = std::chrono::steady_clock::now();
        host_copy_segs(ctx, {{out_index, oi, out_elems * sizeof(uint32_t)}, {out_dist, od, out_elems * sizeof(float)}},
                       false, s);
        end_call(ctx, s);
        cuda_check(cudaStreamSynchronize(s), "solve sync");
        if (stats) {
            fill_stats(stats, ctr, uint64_t(n) * (n - 1) / 2, 1);
            stats->h2d_ms = elapsed_ms(ctx->ev[0], ctx->ev[1]);
            stats->kernel_ms = elapsed_ms(ctx->ev[1], ctx->ev[2]);
            stats->d2h_ms = float(std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_d2h).count());
            stats->sweep_ms = elapsed_ms(ctx->ev[4], ctx->ev[5]);
            stats->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        }
    });
}

int knn_b200_solve_f64(knn_b200_ctx* ctx, const float* host_vectors, uint32_t n, uint32_t d, uint32_t k,
                       int metric, uint32_t* out_index, double* out_dist, knn_b200_stats* stats) {
    return guarded([&] {
        if (!ctx) fail(KNN_B200_ERR_CONFIG, "null context");
        check_args(n, d, k, metric, KNN_B200_ARITH_EXACT);
        std::lock_guard<std::mutex> lock(ctx->mu);
        const auto t0 = std::chrono::steady_clock::now();
        cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
        const uint32_t klist = std::min(k, n - 1);
        const size_t vec_bytes = size_t(n) * d * sizeof(float);
        const size_t out_elems = size_t(n) * klist;
        float* X = static_cast<float*>(ctx->vectors.get(vec_bytes));
        auto* oi = static_cast<uint32_t*>(ctx->out_index.get(out_elems * sizeof(uint32_t)));
        auto* od = static_cast<double*>(ctx->out_dist.get(out_elems * sizeof(double)));
        Counters ctr;
        cudaStream_t s = ctx->stream;
        begin_call(ctx, s);
        cuda_check(cudaEventRecord(ctx->ev[0], s), "event");
        host_copy(ctx, X, host_vectors, vec_bytes, true, s);
        cuda_check(cudaEventRecord(ctx->ev[1], s), "event");
        solve_rows_core_f64(ctx, X, n, d, k, metric, 0, n, oi, od, s, ctr);
        cuda_check(cudaEventRecord(ctx->ev[2], s), "event");
        cuda_check(cudaEventSynchronize(ctx->ev[2]), "solve sync");
        const auto t_d2h = std::chrono::steady_clock::now();
        host_copy_segs(ctx,
                       {{out_index, oi, out_elems * sizeof(uint32_t)}, {out_dist, od, out_elems * sizeof(double)}},
                       false, s);
        end_call(ctx, s);
        cuda_check(cudaStreamSynchronize(s), "solve sync");
        if (stats) {
            fill_stats(stats, ctr, uint64_t(n) * (n - 1) / 2, 1);
            stats->h2d_ms = elapsed_ms(ctx->ev[0], ctx->ev[1]);
            stats->kernel_ms = elapsed_ms(ctx->ev[1], ctx->ev[2]);
            stats->d2h_ms = float(std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_d2h).count());
            stats->sweep_ms = elapsed_ms(ctx->ev[4], ctx->ev[5]);
            stats->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        }
    });
}

int knn_b200_generate_device(knn_b200_ctx* ctx, float* dev_out, uint64_t count, uint64_t seed, void* stream) {
    return guarded([&] {
        if (!ctx) fail(KNN_B200_ERR_CONFIG, "null context");
        cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        cuda_check(knnb::launch_generate(dev_out, count, seed, ctx->sm_count, s), "generate launch");
    });
}

int knn_b200_solve_rows_device(knn_b200_ctx* ctx, const float* dev_vectors, uint32_t n, uint32_t d, uint32_t k,
                               int metric, int arith, uint32_t row_begin, uint32_t row_end,
                               uint32_t* dev_out_index, float* dev_out_dist, void* stream,
                               knn_b200_stats* stats) {
    return guarded([&] {
        if (!ctx) fail(KNN_B200_ERR_CONFIG, "null context");
        check_args(n, d, k, metric, arith);
        if (row_begin > row_end || row_end > n)
            fail(KNN_B200_ERR_CONFIG, "row range [" + std::to_string(row_begin) + ", " + std::to_string(row_end) +
                                          ") outside [0, " + std::to_string(n) + ")");
        std::lock_guard<std::mutex> lock(ctx->mu);
        const auto t0 = std::chrono::steady_clock::now();
        cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        Counters ctr;
        begin_call(ctx, s);
        if (stats) cuda_check(cudaEventRecord(ctx->ev[1], s), "event");
        solve_rows_core(ctx, dev_vectors, n, d, k, metric, arith, row_begin, row_end, dev_out_index,
                        dev_out_dist, s, ctr);
        end_call(ctx, s);
        if (stats) {
            cuda_check(cudaEventRecord(ctx->ev[2], s), "event");
            cuda_check(cudaStreamSynchronize(s), "solve sync");
            uint64_t pairs = 0;  // unordered pairs {x, y} with at least one endpoint in the shard
            const uint64_t rows = row_end - row_begin;
            pairs = rows * (n - 1) - rows * (rows - 1) / 2;
            fill_stats(stats, ctr, pairs, 1);
            stats->h2d_ms = 0;
            stats->d2h_ms = 0;
            stats->kernel_ms = elapsed_ms(ctx->ev[1], ctx->ev[2]);
            stats->sweep_ms = elapsed_ms(ctx->ev[4], ctx->ev[5]);
            stats->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        }
    });
}

int knn_b200_knnv_header(const char* path, uint32_t* out_n, uint32_t* out_d) {
    return guarded([&] {
        const std::string p = path ? path : "";
        Fd f(p);
        const KnnvHeader h = read_knnv_header(f.fd, p);
        *out_n = h.n;
        *out_d = h.d;
    });
}

int knn_b200_load_knnv_device(knn_b200_ctx* ctx, const char* path, float* dev_out, uint64_t capacity,
                              uint32_t* out_n, uint32_t* out_d, void* stream) {
    return guarded([&] {
        if (!ctx) fail(KNN_B200_ERR_CONFIG, "null context");
        const std::string p = path ? path : "";
        std::lock_guard<std::mutex> lock(ctx->mu);
        cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
        Fd f(p);
        const KnnvHeader h = read_knnv_header(f.fd, p);
        const uint64_t count = uint64_t(h.n) * h.d;
        // the Dataset constructor's checks (dataset.cpp:13-29), prefixed with
        // the path as load_dataset does (io.cpp:92-96)
        if (h.n < 2)
            fail(KNN_B200_ERR_VALIDATION, "'" + p + "': dataset needs at least 2 vectors, got " + std::to_string(h.n));
        if (h.d < 1) fail(KNN_B200_ERR_VALIDATION, "'" + p + "': dataset dimension must be at least 1");
        if (count > capacity)
            fail(KNN_B200_ERR_CONFIG, "'" + p + "' holds " + std::to_string(count) + " floats, the buffer " +
                                          std::to_string(capacity));
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        begin_call(ctx, s);
        file_to_device(ctx, f.fd, 16, dev_out, size_t(count) * 4, s, p);
        Counters ctr;
        try {
            validate_device(ctx, dev_out, h.n, h.d, KNN_B200_METRIC_SQEUCLIDEAN, s, ctr);
        } catch (const KnnError& e) {
            end_call(ctx, s);
            if (e.code == KNN_B200_ERR_VALIDATION) fail(e.code, "'" + p + "': " + e.msg);
            throw;
        }
        end_call(ctx, s);
        *out_n = h.n;
        *out_d = h.d;
    });
}

int knn_b200_debug_tc_dots(knn_b200_ctx* ctx, const void* dev_a_f16, uint32_t m, const void* dev_b_f16, uint32_t n,
                           uint32_t d, float* dev_out, void* stream) {
    return guarded([&] {
        if (!ctx) fail(KNN_B200_ERR_CONFIG, "null context");
        cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
        cuda_check(knnb::launch_tc_dots(dev_a_f16, m, dev_b_f16, n, d, dev_out, static_cast<cudaStream_t>(stream)),
                   "tc dots launch");
    });
}

int knn_b200_tri_unit_plan(uint32_t units, uint32_t world, uint32_t pairs_max, uint32_t* out_units,
                           uint32_t* out_counts) {
    return guarded([&] {
        if (world < 1 || world > knnb::kTriMaxWorld || pairs_max < 1)
            fail(KNN_B200_ERR_CONFIG, "bad world " + std::to_string(world) + " / pairs " + std::to_string(pairs_max));
        knnb::tri_unit_plan(units, world, pairs_max, out_units, out_counts);
    });
}

int knn_b200_comm_unique_id(void* out_id) {
    return guarded([&] {
        ncclUniqueId id;
        nccl_check(ncclGetUniqueId(&id), "ncclGetUniqueId");
        std::memcpy(out_id, &id, sizeof(id));
    });
}

int knn_b200_comm_init(knn_b200_ctx* ctx, const void* id, int rank, int world) {
    return guarded([&] {
        if (!ctx) fail(KNN_B200_ERR_CONFIG, "null context");
        if (world < 1 || rank < 0 || rank >= world || world > int(knnb::kTriMaxWorld))
            fail(KNN_B200_ERR_CONFIG, "bad rank " + std::to_string(rank) + " of " + std::to_string(world));
        std::lock_guard<std::mutex> lock(ctx->mu);
        cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
        if (ctx->comm && ctx->comm_owned) ncclCommDestroy(ctx->comm);
        ctx->comm = nullptr;
        ncclUniqueId uid;
        std::memcpy(&uid, id, sizeof(uid));
        nccl_check(ncclCommInitRank(&ctx->comm, world, uid, rank), "ncclCommInitRank");
        ctx->comm_rank = rank;
        ctx->comm_world = world;
        ctx->comm_owned = true;
    });
}

int knn_b200_comm_broadcast(knn_b200_ctx* ctx, void* dev_buf, uint64_t bytes, int root, void* stream) {
    return guarded([&] {
        if (!ctx || !ctx->comm) fail(KNN_B200_ERR_CONFIG, "context has no communicator (knn_b200_comm_init)");
        cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
        nccl_check(ncclBroadcast(dev_buf, dev_buf, bytes, ncclUint8, root, ctx->comm, static_cast<cudaStream_t>(stream)),
                   "ncclBroadcast");
    });
}

int knn_b200_solve_sharded_device(knn_b200_ctx* ctx, const float* dev_vectors, uint32_t n, uint32_t d, uint32_t k,
                                  int metric, int arith, uint32_t* dev_out_index, float* dev_out_dist, void* stream,
                                  knn_b200_stats* stats) {
    return guarded([&] {
        if (!ctx) fail(KNN_B200_ERR_CONFIG, "null context");
        check_args(n, d, k, metric, arith);
        std::lock_guard<std::mutex> lock(ctx->mu);
        const auto t0 = std::chrono::steady_clock::now();
        cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        Counters ctr;
        begin_call(ctx, s);
        if (stats) cuda_check(cudaEventRecord(ctx->ev[1], s), "event");
        const int world = ctx->comm ? ctx->comm_world : 1;
        if (!ctx->comm)
            solve_rows_core(ctx, dev_vectors, n, d, k, metric, arith, 0, n, dev_out_index, dev_out_dist, s, ctr);
        else  // (a communicator of one rank runs the same collectives, degenerate)
            solve_sharded_core(ctx, ctx->comm, ctx->comm_rank, world, dev_vectors, n, d, k, metric, arith,
                               dev_out_index, dev_out_dist, s, ctr);
        end_call(ctx, s);
        if (stats) {
            cuda_check(cudaEventRecord(ctx->ev[2], s), "event");
            cuda_check(cudaStreamSynchronize(s), "solve sync");
            fill_stats(stats, ctr, uint64_t(n) * (n - 1) / 2, world);
            stats->h2d_ms = 0;
            stats->d2h_ms = 0;
            stats->kernel_ms = elapsed_ms(ctx->ev[1], ctx->ev[2]);
            stats->sweep_ms = elapsed_ms(ctx->ev[4], ctx->ev[5]);
            stats->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        }
    });
}

int knn_b200_debug_solve_sharded_loopback(knn_b200_ctx* ctx, const float* dev_vectors, uint32_t n, uint32_t d,
                                          uint32_t k, int metric, int world, uint32_t* dev_out_index,
                                          float* dev_out_dist, void* stream, knn_b200_stats* stats,
                                          float* rank_ms, uint64_t* rank_xbytes) {
    return guarded([&] {
        if (!ctx) fail(KNN_B200_ERR_CONFIG, "null context");
        check_args(n, d, k, metric, KNN_B200_ARITH_TENSOR);
        if (world < 1 || world > int(knnb::kTriMaxWorld)) fail(KNN_B200_ERR_CONFIG, "bad world " + std::to_string(world));
        const uint32_t klist = std::min(k, n - 1);
        const int mode = tri_selected(n, d, klist, metric, KNN_B200_ARITH_TENSOR);
        if (!mode)
            fail(KNN_B200_ERR_CONFIG, "problem does not take a triangle sweep (see tri_eligible, tcap_eligible)");
        std::lock_guard<std::mutex> lock(ctx->mu);
        const auto t0 = std::chrono::steady_clock::now();
        cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        Counters ctr;
        begin_call(ctx, s);
        cuda_check(cudaEventRecord(ctx->ev[1], s), "event");
        validate_device(ctx, dev_vectors, n, d, metric, s, ctr);
        const float* Xs = dev_vectors;
        if (metric == KNN_B200_METRIC_HELLINGER) {
            float* staged = static_cast<float*>(ctx->staged.get(size_t(n) * d * sizeof(float)));
            cuda_check(knnb::launch_stage_sqrt(dev_vectors, staged, uint64_t(n) * d, ctx->sm_count, s), "stage launch");
            Xs = staged;
        }
        knnb::TensorPathArgs ta = tri_args(ctx, Xs, n, d, klist, metric, dev_out_index, dev_out_dist, s);
        knnb::TensorPathResult tr;
        bool overflow = false;
        cuda_check(knnb::run_tri_loopback(ta, uint32_t(world), shard_alloc, ctx, tr, rank_ms,
                                          reinterpret_cast<unsigned long long*>(rank_xbytes), &overflow, mode == 2),
                   "sharded triangle (loopback)");
        ctr.arith_used = KNN_B200_ARITH_TENSOR;
        ctr.launches += tr.launches;
        ctr.rescored += tr.rescored;
        ctr.fallback_rows += tr.fallback_rows;
        ctr.exact_rows += tr.exact_rows;
        if (overflow)
            solve_rows_core(ctx, dev_vectors, n, d, k, metric, KNN_B200_ARITH_TENSOR, 0, n, dev_out_index,
                            dev_out_dist, s, ctr);
        end_call(ctx, s);
        cuda_check(cudaEventRecord(ctx->ev[2], s), "event");
        cuda_check(cudaStreamSynchronize(s), "solve sync");
        if (stats) {
            fill_stats(stats, ctr, uint64_t(n) * (n - 1) / 2, world);
            stats->reserved = overflow ? 1 : 0;
            stats->kernel_ms = elapsed_ms(ctx->ev[1], ctx->ev[2]);
            stats->sweep_ms = elapsed_ms(ctx->ev[4], ctx->ev[5]);
            stats->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        }
    });
}

}  // extern "C"

namespace {

// One process-wide context per device, reused across calls and guarded by a
// mutex so concurrent solve_knn calls serialise.  DistT =
// float runs the float policies; double runs the KNN_DOUBLE_ACCUM sweep.
std::mutex pool_mu;                // guards `pool`, shared by both distance types
std::vector<knn_b200_ctx*> pool;  // one context per device, created on first use

// NCCL communicators over devices 0..m-1 for the single-process multi-GPU
// solve (ncclCommInitAll), created on first use per device count.
std::map<uint32_t, std::vector<ncclComm_t>> multi_comms;  // guarded by pool_mu

template <typename DistT>
int solve_multi_impl(const float* host_vectors, uint32_t n, uint32_t d, uint32_t k, int metric, int arith,
                     uint32_t n_gpus, uint32_t* out_index, DistT* out_dist, knn_b200_stats* stats) {
    return guarded([&] {
        check_args(n, d, k, metric, arith);
        if (n_gpus < 1) fail(KNN_B200_ERR_CONFIG, "n_lanes must be at least 1");
        int ndev = 0;
        cuda_check(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount (no CUDA device; there is no CPU fallback)");
        const uint32_t use = std::min<uint32_t>(std::min<uint32_t>(n_gpus, uint32_t(ndev)), n);
        std::lock_guard<std::mutex> lock(pool_mu);
        if (pool.size() < size_t(ndev)) pool.resize(ndev, nullptr);
        for (uint32_t g = 0; g < use; ++g) {
            if (!pool[g]) {
                knn_b200_ctx* c = nullptr;
                const int rc = knn_b200_create(int(g), &c);
                if (rc != KNN_B200_OK) fail(rc, g_last_error);
                pool[g] = c;
            }
        }
        std::vector<ncclComm_t>* comms = nullptr;
        if (use > 1) {
            auto it = multi_comms.find(use);
            if (it == multi_comms.end()) {
                std::vector<ncclComm_t> cs(use);
                std::vector<int> devs(use);
                for (uint32_t g = 0; g < use; ++g) devs[g] = int(g);
                nccl_check(ncclCommInitAll(cs.data(), int(use), devs.data()), "ncclCommInitAll");
                it = multi_comms.emplace(use, std::move(cs)).first;
            }
            comms = &it->second;
        }
        const auto t0 = std::chrono::steady_clock::now();
        const uint32_t klist = std::min(k, n - 1);
        std::vector<KnnError> errs(use, KnnError{0, {}});
        std::mutex watch_mu;
        std::condition_variable watch_cv;
        bool failed = false, finished = false;
        std::vector<Counters> ctrs(use);
        std::vector<float> kms(use, 0.f), hms(use, 0.f), dms(use, 0.f), sms(use, 0.f);
        // One host thread per GPU (engine.cpp:37-56).  The reference set goes
        // to device 0 once (pinned staging lanes) and is replicated by one
        // NCCL broadcast; each device then solves its contiguous shard of rows
        // (shard_rows) -- float distances through the sharded triangle where
        // eligible -- and copies it straight into the caller's arrays.
        auto lane = [&](uint32_t g) {
            try {
                knn_b200_ctx* ctx = pool[g];
                std::lock_guard<std::mutex> cl(ctx->mu);
                cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
                uint32_t r0, r1;
                shard_rows(n, int(g), int(use), r0, r1);
                const size_t vec_bytes = size_t(n) * d * sizeof(float);
                const size_t out_elems = size_t(r1 - r0) * klist;
                float* X = static_cast<float*>(ctx->vectors.get(vec_bytes));
                auto* oi = static_cast<uint32_t*>(ctx->out_index.get(std::max<size_t>(out_elems, 1) * 4));
                auto* od = static_cast<DistT*>(ctx->out_dist.get(std::max<size_t>(out_elems, 1) * sizeof(DistT)));
                cudaStream_t s = ctx->stream;
                begin_call(ctx, s);
                cuda_check(cudaEventRecord(ctx->ev[0], s), "event");
                if (g == 0) host_copy(ctx, X, host_vectors, vec_bytes, true, s);
                if (comms)
                    nccl_check(ncclBroadcast(X, X, vec_bytes, ncclUint8, 0, (*comms)[g], s), "ncclBroadcast");
                cuda_check(cudaEventRecord(ctx->ev[1], s), "event");
                if constexpr (std::is_same_v<DistT, double>)
                    solve_rows_core_f64(ctx, X, n, d, k, metric, r0, r1, oi, od, s, ctrs[g]);
                else if (comms)
                    solve_sharded_core(ctx, (*comms)[g], int(g), int(use), X, n, d, k, metric, arith, oi, od, s,
                                       ctrs[g]);
                else
                    solve_rows_core(ctx, X, n, d, k, metric, arith, r0, r1, oi, od, s, ctrs[g]);
                cuda_check(cudaEventRecord(ctx->ev[2], s), "event");
                cuda_check(cudaEventSynchronize(ctx->ev[2]), "solve sync");
                const auto t_d2h = std::chrono::steady_clock::now();
                if (out_elems) {
                    const int st_threads = std::max(1, kStageThreadsDefault / int(use));
                    host_copy_segs(ctx,
                                   {{out_index + size_t(r0) * klist, oi, out_elems * 4},
                                    {out_dist + size_t(r0) * klist, od, out_elems * sizeof(DistT)}},
                                   false, s, st_threads);
                }
                end_call(ctx, s);
                cuda_check(cudaStreamSynchronize(s), "solve sync");
                hms[g] = elapsed_ms(ctx->ev[0], ctx->ev[1]);
                kms[g] = elapsed_ms(ctx->ev[1], ctx->ev[2]);
                dms[g] = float(std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_d2h).count());
                sms[g] = elapsed_ms(ctx->ev[4], ctx->ev[5]);
            } catch (const KnnError& e) {
                errs[g] = e;
            } catch (const std::exception& e) {
                errs[g] = KnnError{KNN_B200_ERR_INTERNAL, e.what()};
            }
            if (errs[g].code) {  // wake the watchdog: the other lanes may be waiting on this one in a collective
                std::lock_guard<std::mutex> wl(watch_mu);
                failed = true;
                watch_cv.notify_all();
            }
        };
        // The lanes' collectives wait for every rank: a lane that fails (an
        // allocation, a CUDA error) would leave the others spinning in NCCL
        // kernels.  The watchdog aborts the communicators on the first lane
        // error, which ends those kernels; the lanes then return errors, are
        // joined, and the first error is rethrown (engine.cpp:53-56).  The
        // aborted communicators are dropped; the next call makes new ones.
        std::thread watchdog;
        bool aborted = false;
        if (comms)
            watchdog = std::thread([&] {
                std::unique_lock<std::mutex> wl(watch_mu);
                watch_cv.wait(wl, [&] { return failed || finished; });
                if (failed) {
                    for (ncclComm_t c : *comms) ncclCommAbort(c);
                    aborted = true;
                }
            });
        std::vector<std::thread> threads;
        for (uint32_t g = 1; g < use; ++g) threads.emplace_back(lane, g);
        lane(0);
        for (auto& t : threads) t.join();
        if (watchdog.joinable()) {
            {
                std::lock_guard<std::mutex> wl(watch_mu);
                finished = true;
                watch_cv.notify_all();
            }
            watchdog.join();
        }
        if (aborted) multi_comms.erase(use);
        // engine.cpp:53-56: rethrow the first lane error after joining.
        for (const auto& e : errs)
            if (e.code) throw e;
        if (stats) {
            Counters tot;
            for (const auto& c : ctrs) {
                tot.launches += c.launches;
                tot.distance_evals += c.distance_evals;
                tot.rescored += c.rescored;
                tot.fallback_rows += c.fallback_rows;
                tot.exact_rows += c.exact_rows;
                tot.arith_used = c.arith_used;
            }
            fill_stats(stats, tot, uint64_t(n) * (n - 1) / 2, int(use));
            stats->h2d_ms = *std::max_element(hms.begin(), hms.end());
            stats->kernel_ms = *std::max_element(kms.begin(), kms.end());
            stats->d2h_ms = *std::max_element(dms.begin(), dms.end());
            stats->sweep_ms = *std::max_element(sms.begin(), sms.end());
            stats->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        }
    });
}

}  // namespace

extern "C" {

int knn_b200_solve_multi(const float* host_vectors, uint32_t n, uint32_t d, uint32_t k, int metric, int arith,
                         uint32_t n_gpus, uint32_t* out_index, float* out_dist, knn_b200_stats* stats) {
    return solve_multi_impl<float>(host_vectors, n, d, k, metric, arith, n_gpus, out_index, out_dist, stats);
}

int knn_b200_solve_multi_f64(const float* host_vectors, uint32_t n, uint32_t d, uint32_t k, int metric,
                             uint32_t n_gpus, uint32_t* out_index, double* out_dist, knn_b200_stats* stats) {
    return solve_multi_impl<double>(host_vectors, n, d, k, metric, KNN_B200_ARITH_EXACT, n_gpus, out_index,
                                    out_dist, stats);
}

}  // extern "C"
