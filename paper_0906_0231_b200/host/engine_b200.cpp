// engine_b200.cpp -- drop-in definition of knn::solve_knn on the B200 C ABI.
//
// Replaces the reference's src/engine.cpp:13-68 at link time: same signature
// (include/knn/engine.hpp:37-38), same option checks and plan
// (engine.cpp:15-22), same validation-before-timer (engine.cpp:23-25), same
// EngineResult fields (engine.hpp:25-31).  Compiled against the reference's
// public headers; everything else it needs (make_plan, auto_gsize,
// validate_dataset) comes from the rest of the reference library, which the
// caller links unchanged.  The compute runs on the GPU through
// include/knn_b200.h; there is no CPU fallback.
//
// n_lanes -> GPUs used = min(n_lanes, visible sm_100 devices); results are
// lane-independent bit for bit, as the reference promises (engine.hpp:33-36).
// The arithmetic policy is chosen out of band (EngineOptions has no field):
// KNN_B200_ARITH=auto|exact|tensor, default auto.  All policies return the
// same bits.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <thread>
#include <type_traits>
#include <vector>

#include "knn/engine.hpp"
#include "knn/errors.hpp"
#include "knn/rng.hpp"
#include "knn_b200.h"

namespace knn {

// dist_t is float in the default build and double with KNN_DOUBLE_ACCUM
// (types.hpp:9-13); the double build runs knn_b200_solve_f64 (EXACT policy,
// FP64 accumulation, bit-identical to the reference's double build).
static_assert(std::is_same_v<dist_t, float> || std::is_same_v<dist_t, double>);

namespace {

// Host restatements of the device folds a custom functor may turn out to be
// (common.cuh fold_step / fold_finalize; exact_f64.cu for dist_t = double).
// This TU is compiled with -ffp-contract=off, so each is separately rounded
// exactly like the device code.
dist_t device_fold_sqeuclidean(const float* u, const float* v, std::uint32_t d) {
    dist_t acc = 0;
    for (std::uint32_t j = 0; j < d; ++j) {
        const float t = u[j] - v[j];
        acc = acc + dist_t(t) * dist_t(t);
    }
    return acc;
}

dist_t device_fold_cosine(const float* u, const float* v, std::uint32_t d) {
    dist_t acc = 0;
    for (std::uint32_t j = 0; j < d; ++j) acc = acc + dist_t(u[j]) * dist_t(v[j]);
    return dist_t(1) - acc;
}

dist_t device_fold_manhattan(const float* u, const float* v, std::uint32_t d) {
    dist_t acc = 0;
    for (std::uint32_t j = 0; j < d; ++j) acc = acc + dist_t(std::fabs(u[j] - v[j]));
    return acc;
}

dist_t device_fold_root_squares(const float* u, const float* v, std::uint32_t d) {
    return dist_t(std::sqrt(device_fold_sqeuclidean(u, v, d)));
}

// A custom functor is a host function pointer (distance.hpp:68-77); the GPU
// cannot call it.  It runs on the GPU only if it IS one of the device folds,
// bit for bit: the functor is probed on random vectors -- as the reference's
// registry probes symmetry (distance.cpp:117-136) -- and compared with each
// restatement above.  Anything else is rejected with ConfigError (no CPU
// fallback).  The name is not trusted: a "cosine" with another initial value,
// sign convention or float-rounded product in the double build is rejected.
bool functor_matches(const CumulativeDistance& f, dist_t (*fold)(const float*, const float*, std::uint32_t)) {
    if (!f.step) return false;
    const metrics::Erased m{f.initial, f.step, f.finalize};
    SplitMix64 rng(0x6b2f7a11d3c05e93ull);
    constexpr std::uint32_t kMaxDim = 128;
    float u[kMaxDim], v[kMaxDim];
    for (std::uint32_t trial = 0; trial < 256; ++trial) {
        const std::uint32_t d = 1 + (trial * 7) % kMaxDim;
        // value mixes: [0,1) and [-1,1) (the data's range), and full 24-bit
        // mantissas with exponents spread over 2^-2..2^2 and 2^-5..2^5, whose
        // partial sums need rounding even in double -- a fold that rounds
        // differently (another order, sign convention or widening) shows there
        for (std::uint32_t j = 0; j < d; ++j) {
            float x[2];
            for (float& a : x) {
                const std::uint32_t mode = trial % 4;
                if (mode == 0) {
                    a = rng.next_unit_float();
                } else if (mode == 1) {
                    a = 2.0f * rng.next_unit_float() - 1.0f;
                } else {
                    const std::uint64_t r = rng.next();
                    const int spread = mode == 2 ? 2 : 5;
                    const float m = float((r >> 40) | (1u << 23)) * 0x1.0p-24f;  // [0.5, 1), 24 bits
                    const int e = int((r >> 8) % std::uint64_t(2 * spread + 1)) - spread;
                    a = std::ldexp(m, e) * ((r & 1) ? -1.0f : 1.0f);
                }
            }
            u[j] = x[0];
            v[j] = x[1];
        }
        const dist_t want = fold(u, v, d);
        const dist_t got = fold_distance(m, u, v, d);
        if (std::memcmp(&want, &got, sizeof(dist_t)) != 0) return false;
    }
    return true;
}

int gpu_metric(const CumulativeDistance& f) {
    switch (f.kind) {
    case MetricKind::hellinger:
        return KNN_B200_METRIC_HELLINGER;
    case MetricKind::sqeuclidean:
        return KNN_B200_METRIC_SQEUCLIDEAN;
    case MetricKind::custom:
        if (functor_matches(f, device_fold_sqeuclidean)) return KNN_B200_METRIC_SQEUCLIDEAN;
        if (functor_matches(f, device_fold_cosine)) return KNN_B200_METRIC_COSINE;
        if (functor_matches(f, device_fold_manhattan)) return KNN_B200_METRIC_MANHATTAN;
        if (functor_matches(f, device_fold_root_squares)) return KNN_B200_METRIC_ROOT_SQUARES;
        break;
    }
    throw ConfigError("distance functor '" + f.name +
                      "' is a host function pointer that matches none of the GPU engine's folds "
                      "(sqeuclidean, cosine = 1 - sum u*v, manhattan = sum |u - v|, sqrt of sqeuclidean); "
                      "it cannot run on the GPU engine");
}

int arith_from_env() {
    const char* v = std::getenv("KNN_B200_ARITH");
    if (!v || !*v || std::strcmp(v, "auto") == 0) return KNN_B200_ARITH_AUTO;
    if (std::strcmp(v, "exact") == 0) return KNN_B200_ARITH_EXACT;
    if (std::strcmp(v, "tensor") == 0) return KNN_B200_ARITH_TENSOR;
    throw ConfigError(std::string("KNN_B200_ARITH must be auto, exact or tensor, got '") + v + "'");
}

[[noreturn]] void rethrow_status(int rc) {
    const std::string msg = knn_b200_last_error();
    switch (rc) {
    case KNN_B200_ERR_CONFIG:
        throw ConfigError(msg);
    case KNN_B200_ERR_VALIDATION:
        throw ValidationError(msg);
    default:
        throw std::runtime_error("B200 engine: " + msg);
    }
}

// Default build: float distances, one host thread per GPU (n_lanes).
int gpu_solve(const Dataset& ds, const EngineOptions& opt, int metric, int arith, std::uint32_t lanes,
              std::uint32_t* index, float* dist, knn_b200_stats* st) {
    return knn_b200_solve_multi(ds.values().data(), ds.size(), ds.dim(), opt.k, metric, arith, lanes, index,
                                dist, st);
}

// KNN_DOUBLE_ACCUM build: double distances, the same lanes (FP64 EXACT sweep).
[[maybe_unused]] int gpu_solve(const Dataset& ds, const EngineOptions& opt, int metric, int arith,
                               std::uint32_t lanes, std::uint32_t* index, double* dist, knn_b200_stats* st) {
    if (arith == KNN_B200_ARITH_TENSOR)
        throw ConfigError("KNN_DOUBLE_ACCUM builds run the exact policy only (KNN_B200_ARITH=tensor)");
    return knn_b200_solve_multi_f64(ds.values().data(), ds.size(), ds.dim(), opt.k, metric, lanes, index, dist,
                                    st);
}

}  // namespace

EngineResult solve_knn(const Dataset& ds, const CumulativeDistance& f, const EngineOptions& opt) {
    if (opt.k < 1) throw ConfigError("k must be at least 1");
    if (opt.buf_size < 1) throw ConfigError("buf_size must be at least 1");
    if (opt.workers < 1) throw ConfigError("workers must be at least 1");

    const std::uint32_t gsize = opt.gsize != 0 ? opt.gsize : auto_gsize(ds.size(), opt.bsize);
    const GridPlan plan = make_plan(ds.size(), gsize, opt.bsize, opt.c1, opt.c2, opt.n_lanes);
    validate_dataset(f, ds);
    const int metric = gpu_metric(f);
    const int arith = arith_from_env();

    const auto t0 = std::chrono::steady_clock::now();

    const std::uint32_t n = ds.size();
    const std::uint32_t klist = std::min(opt.k, n - 1);
    // caller-owned outputs of the C ABI: not zero-filled (every element is written)
    std::unique_ptr<std::uint32_t[]> index(new std::uint32_t[std::size_t(n) * klist]);
    std::unique_ptr<dist_t[]> dist(new dist_t[std::size_t(n) * klist]);
    knn_b200_stats st{};

    // EngineResult owns one std::vector per row (engine.hpp:25-31): at C2
    // that is 1M heap allocations.  The GPU call blocks its thread for the
    // whole solve (H2D, sweeps, D2H), so it runs on a helper thread while this
    // one and a few more allocate the rows; only the copy of the values is
    // left for after it returns (C2: 49 ms of the drop-in's time before).
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const std::uint32_t nthreads = n < 65536 ? 1u : std::min<std::uint32_t>(16u, hw);
    auto parallel_rows = [&](auto&& body) {
        std::vector<std::thread> pool;
        for (std::uint32_t t = 1; t < nthreads; ++t)
            pool.emplace_back(body, std::uint32_t(std::uint64_t(n) * t / nthreads),
                              std::uint32_t(std::uint64_t(n) * (t + 1) / nthreads));
        body(0u, std::uint32_t(std::uint64_t(n) / nthreads));
        for (auto& th : pool) th.join();
    };
    int rc = KNN_B200_ERR_INTERNAL;
    std::exception_ptr solve_error;
    std::thread solver([&] {
        try {
            rc = gpu_solve(ds, opt, metric, arith, plan.n_lanes, index.get(), dist.get(), &st);
        } catch (...) {
            solve_error = std::current_exception();
        }
    });
    EngineResult result;
    try {
        result.lists.resize(n);
        parallel_rows([&](std::uint32_t r0, std::uint32_t r1) {
            for (std::uint32_t i = r0; i < r1; ++i) {
                result.lists[i].query = i;
                result.lists[i].neighbors.resize(klist);
            }
        });
    } catch (...) {
        solver.join();
        throw;
    }
    solver.join();
    if (solve_error) std::rethrow_exception(solve_error);
    if (rc != KNN_B200_OK) rethrow_status(rc);
    parallel_rows([&](std::uint32_t r0, std::uint32_t r1) {
        for (std::uint32_t i = r0; i < r1; ++i) {
            Neighbor* out = result.lists[i].neighbors.data();
            const std::size_t base = std::size_t(i) * klist;
            for (std::uint32_t j = 0; j < klist; ++j) out[j] = Neighbor{dist[base + j], index[base + j]};
        }
    });
    result.seconds =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    result.plan = plan;
    // Semantic counters (test_engine.cpp:65-68): every unordered pair is
    // covered once and offered to both endpoints.  The filter/flush counters
    // of the CPU funnel have no GPU analogue and stay 0.
    result.pair_evaluations = st.pair_evaluations;
    result.select_stats.offered = 2 * st.pair_evaluations;
    return result;
}

}  // namespace knn
