// bench_dropin.cpp -- time the C++ drop-in knn::solve_knn end to end.
//
// The reference's public entry point (include/knn/engine.hpp:37-38) linked
// against the B200 drop-in (engine_b200.cpp): the caller's Dataset is a
// pageable std::vector, the result is EngineResult.lists, one NeighborList
// (a std::vector) per row -- exactly what a user of the reference gets.  The
// timed region is the whole solve_knn call, K times after W warm-ups, on the
// host's steady clock; the dataset is generate_dataset(n, d, seed)
// (io.cpp:57-62), built before the timer.
//
//   bench_dropin n d k seed steps warmup [lanes]   -> one JSON line
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "knn/distance.hpp"
#include "knn/engine.hpp"
#include "knn/io.hpp"

int main(int argc, char** argv) {
    if (argc < 7) {
        std::fprintf(stderr, "usage: %s n d k seed steps warmup [lanes]\n", argv[0]);
        return 2;
    }
    const std::uint32_t n = std::uint32_t(std::strtoul(argv[1], nullptr, 10));
    const std::uint32_t d = std::uint32_t(std::strtoul(argv[2], nullptr, 10));
    const std::uint32_t k = std::uint32_t(std::strtoul(argv[3], nullptr, 10));
    const std::uint64_t seed = std::strtoull(argv[4], nullptr, 10);
    const int steps = std::atoi(argv[5]), warmup = std::atoi(argv[6]);
    const std::uint32_t lanes = argc > 7 ? std::uint32_t(std::atoi(argv[7])) : 1;
    const knn::Dataset ds = knn::generate_dataset(n, d, seed);
    knn::EngineOptions opt;
    opt.k = k;
    opt.n_lanes = lanes;
    const knn::CumulativeDistance& f = knn::distance_by_name("sqeuclidean");
    double engine_s = 0;
    std::size_t rows = 0;
    for (int i = 0; i < warmup; ++i) rows = knn::solve_knn(ds, f, opt).lists.size();
    const auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < steps; ++i) {
        const knn::EngineResult r = knn::solve_knn(ds, f, opt);
        engine_s += r.seconds;
        rows = r.lists.size();
    }
    const double total = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    std::printf("{\"ms_per_step\": %.3f, \"engine_seconds_per_step\": %.6f, \"rows\": %zu, \"n\": %u, \"d\": %u, "
                "\"k\": %u, \"lanes\": %u, \"steps\": %d}\n",
                1e3 * total / steps, engine_s / steps, rows, n, d, k, lanes, steps);
    return 0;
}
