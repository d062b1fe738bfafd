// ref_capi.cpp -- C shim over the UNMODIFIED reference tknn library.
//
// TEST INFRASTRUCTURE ONLY (see oracle/knn_oracle.c header).  Compiled by
// oracle/Makefile together with the reference's own sources, read in place
// from /root/reference/proj/src, into oracle/_ref/libtknn_ref_capi.so.  It
// lets the Python tests and bench.py's reference arm call the reference
// itself through ctypes:
//   ref_brute_force  -> knn::brute_force_knn   (src/oracle.cpp:10-42)
//   ref_solve_knn    -> knn::solve_knn          (src/engine.cpp:13-68)
//   ref_generate     -> knn::generate_dataset   (src/io.cpp:57-62)
//   ref_rows_topk    -> fold_distance + NeighborHeap per sampled row
//                       (include/knn/distance.hpp:98-105, src/heap.cpp:18-64)
// Metric ids: 0 hellinger, 1 sqeuclidean (built-ins), 2 cosine (a custom fold
// registered through knn::register_distance).
// Return codes mirror the CLI exit codes (tools/main.cpp:225-240):
// 0 ok, 2 ConfigError, 3 ValidationError, 4 anything else.

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "knn/dataset.hpp"
#include "knn/distance.hpp"
#include "knn/engine.hpp"
#include "knn/errors.hpp"
#include <cmath>

#include "knn/heap.hpp"
#include "knn/io.hpp"
#include "knn/oracle.hpp"

namespace {

thread_local std::string g_err;

const knn::CumulativeDistance& cosine_fold() {
    static const knn::CumulativeDistance& f = [] () -> const knn::CumulativeDistance& {
        knn::CumulativeDistance c;
        c.name = "cosine";
        c.initial = 0;
        c.step = +[](float u, float v, knn::dist_t acc) { return acc + knn::dist_t(u) * knn::dist_t(v); };
        c.finalize = +[](knn::dist_t acc) { return knn::dist_t(1) - acc; };
        c.kind = knn::MetricKind::custom;
        return knn::register_distance(c);
    }();
    return f;
}

// The custom functors of the reference's own tests, registered through the
// reference's registry: test_distance.cpp:134-145 and :166-178.
const knn::CumulativeDistance& manhattan_fold() {
    static const knn::CumulativeDistance& f = [] () -> const knn::CumulativeDistance& {
        knn::CumulativeDistance c;
        c.name = "manhattan";
        c.initial = 0;
        c.step = +[](float u, float v, knn::dist_t acc) { return acc + knn::dist_t(std::fabs(u - v)); };
        return knn::register_distance(c);
    }();
    return f;
}

const knn::CumulativeDistance& root_squares_fold() {
    static const knn::CumulativeDistance& f = [] () -> const knn::CumulativeDistance& {
        knn::CumulativeDistance c;
        c.name = "root_of_squares";
        c.initial = 0;
        c.step = +[](float u, float v, knn::dist_t acc) {
            const float t = u - v;
            return acc + knn::dist_t(t) * knn::dist_t(t);
        };
        c.finalize = +[](knn::dist_t acc) { return knn::dist_t(std::sqrt(acc)); };
        return knn::register_distance(c);
    }();
    return f;
}

const knn::CumulativeDistance& metric_by_id(int metric) {
    switch (metric) {
    case 0: return knn::distance_by_name("hellinger");
    case 1: return knn::distance_by_name("sqeuclidean");
    case 2: return cosine_fold();
    case 3: return manhattan_fold();
    case 4: return root_squares_fold();
    default: throw knn::ConfigError("unknown metric id " + std::to_string(metric));
    }
}

template <typename Fn>
int guarded(Fn&& fn) {
    try {
        fn();
        return 0;
    } catch (const knn::ConfigError& e) {
        g_err = e.what();
        return 2;
    } catch (const knn::ValidationError& e) {
        g_err = e.what();
        return 3;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 4;
    }
}

void flatten(const std::vector<knn::NeighborList>& lists, std::uint32_t cap,
             std::uint32_t* idx, float* dist) {
    for (std::size_t i = 0; i < lists.size(); ++i) {
        const auto& nb = lists[i].neighbors;
        for (std::uint32_t j = 0; j < cap; ++j) {
            idx[i * cap + j] = j < nb.size() ? nb[j].index : 0xffffffffu;
            dist[i * cap + j] = j < nb.size() ? float(nb[j].distance) : 0.0f;
        }
    }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_generate(std::uint32_t n, std::uint32_t d, std::uint64_t seed, float* out) {
    return guarded([&] {
        const knn::Dataset ds = knn::generate_dataset(n, d, seed);
        std::memcpy(out, ds.values().data(), ds.values().size() * sizeof(float));
    });
}

int ref_brute_force(const float* x, std::uint32_t n, std::uint32_t d, std::uint32_t k,
                    int metric, std::uint32_t* idx, float* dist, std::uint64_t* pairs,
                    double* seconds) {
    return guarded([&] {
        const knn::CumulativeDistance& f = metric_by_id(metric);
        knn::Dataset ds(n, d, std::vector<float>(x, x + std::size_t(n) * d));
        const knn::OracleResult r = knn::brute_force_knn(ds, f, k);
        flatten(r.lists, std::min(k, n - 1), idx, dist);
        if (pairs) *pairs = r.pair_evaluations;
        if (seconds) *seconds = r.seconds;
    });
}

#if defined(KNN_DOUBLE_ACCUM)
// The reference's KNN_DOUBLE_ACCUM build (types.hpp:9-13): brute_force_knn
// with double distances, returned without narrowing.
int ref_brute_force_f64(const float* x, std::uint32_t n, std::uint32_t d, std::uint32_t k,
                        int metric, std::uint32_t* idx, double* dist) {
    return guarded([&] {
        const knn::CumulativeDistance& f = metric_by_id(metric);
        knn::Dataset ds(n, d, std::vector<float>(x, x + std::size_t(n) * d));
        const knn::OracleResult r = knn::brute_force_knn(ds, f, k);
        const std::uint32_t cap = std::min(k, n - 1);
        for (std::size_t i = 0; i < r.lists.size(); ++i)
            for (std::uint32_t j = 0; j < cap; ++j) {
                idx[i * cap + j] = r.lists[i].neighbors[j].index;
                dist[i * cap + j] = r.lists[i].neighbors[j].distance;
            }
    });
}
#endif

int ref_solve_knn(const float* x, std::uint32_t n, std::uint32_t d, std::uint32_t k,
                  int metric, std::uint32_t n_lanes, std::uint32_t gsize,
                  std::uint32_t* idx, float* dist, std::uint64_t* pairs, double* seconds) {
    return guarded([&] {
        const knn::CumulativeDistance& f = metric_by_id(metric);
        knn::Dataset ds(n, d, std::vector<float>(x, x + std::size_t(n) * d));
        knn::EngineOptions opt;
        opt.k = k;
        opt.n_lanes = n_lanes;
        opt.gsize = gsize;
        const knn::EngineResult r = knn::solve_knn(ds, f, opt);
        if (idx && dist) flatten(r.lists, std::min(k, n - 1), idx, dist);
        if (pairs) *pairs = r.pair_evaluations;
        if (seconds) *seconds = r.seconds;
    });
}

// Exact lists for a subset of query rows with the reference's own fold and
// bounded heap, `threads` std::threads over rows. No Dataset copy: the fold
// reads the caller's buffer directly (validation is the caller's business).
int ref_rows_topk(const float* x, std::uint32_t n, std::uint32_t d, std::uint32_t k,
                  int metric, const std::uint32_t* rows, std::uint32_t nrows,
                  std::uint32_t threads, std::uint32_t* idx, float* dist) {
    return guarded([&] {
        if (k < 1) throw knn::ConfigError("k must be at least 1");
        const knn::CumulativeDistance& f = metric_by_id(metric);
        const std::uint32_t cap = std::min(k, n - 1);
        std::atomic<std::uint32_t> next{0};
        auto work = [&] {
            knn::dispatch_metric(f, [&](auto m) {
                for (;;) {
                    const std::uint32_t r = next.fetch_add(1);
                    if (r >= nrows) break;
                    const std::uint32_t q = rows[r];
                    knn::NeighborHeap h(cap);
                    const float* vq = x + std::size_t(q) * d;
                    for (std::uint32_t i = 0; i < n; ++i) {
                        if (i == q) continue;
                        const float* vi = x + std::size_t(i) * d;
                        const knn::dist_t dd = i > q ? knn::fold_distance(m, vi, vq, d)
                                                     : knn::fold_distance(m, vq, vi, d);
                        h.push({dd, i});
                    }
                    const auto sorted = h.drain_sorted();
                    for (std::uint32_t t = 0; t < cap; ++t) {
                        idx[std::size_t(r) * cap + t] = sorted[t].index;
                        dist[std::size_t(r) * cap + t] = float(sorted[t].distance);
                    }
                }
            });
        };
        std::vector<std::thread> pool;
        for (std::uint32_t t = 1; t < std::max(1u, threads); ++t) pool.emplace_back(work);
        work();
        for (auto& t : pool) t.join();
    });
}

}  // extern "C"
