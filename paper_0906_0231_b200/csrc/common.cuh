// common.cuh -- shared device helpers for the B200 k-NN kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace knnb {

// Device folds.  kHellinger and kSqEuclidean are the reference built-ins
// (Hellinger arrives sqrt-staged and folds like kSqEuclidean); the others
// restate custom functors of the reference's registry that a drop-in caller
// may register (distance.hpp:68-77): cosine, manhattan
// (acc + |u - v|, test_distance.cpp:134-145) and root-of-squares
// (sqeuclidean with finalize sqrt, test_distance.cpp:166-178).  The last two
// run on the EXACT policy only.
enum Metric : int { kHellinger = 0, kSqEuclidean = 1, kCosine = 2, kManhattan = 3, kRootSquares = 4 };

// (distance, index) packed into one u64 whose unsigned order is the
// reference's Neighbor order (include/knn/heap.hpp:21-24): distance first,
// smaller index on ties.  The float is mapped to an order-preserving u32
// (negative values, possible for cosine, flip all bits).  -0.0 is
// canonicalised to +0.0 first because the reference compares with float
// `<`/`!=`, where the two are equal and the index decides.
__host__ __device__ __forceinline__ uint32_t float_to_ordered(float f) {
#ifdef __CUDA_ARCH__
    uint32_t b = __float_as_uint(f + 0.0f);
#else
    union { float f; uint32_t u; } c;
    c.f = f + 0.0f;
    uint32_t b = c.u;
#endif
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

__host__ __device__ __forceinline__ float ordered_to_float(uint32_t o) {
    const uint32_t b = (o & 0x80000000u) ? (o & 0x7fffffffu) : ~o;
#ifdef __CUDA_ARCH__
    return __uint_as_float(b);
#else
    union { float f; uint32_t u; } c;
    c.u = b;
    return c.f;
#endif
}

__host__ __device__ __forceinline__ uint64_t make_key(float dist, uint32_t index) {
    return (uint64_t(float_to_ordered(dist)) << 32) | index;
}

constexpr uint64_t kEmptyKey = ~0ull;

// One step of the reference fold on staged coordinates, with every operation
// separately rounded (no FMA contraction), distance.hpp:49-52 / :59-62.
// Hellinger arrives here with both coordinates already sqrt-staged.
template <int METRIC>
__device__ __forceinline__ float fold_step(float u, float v, float acc) {
    if constexpr (METRIC == kCosine) {
        return __fadd_rn(acc, __fmul_rn(u, v));
    } else if constexpr (METRIC == kManhattan) {
        return __fadd_rn(acc, fabsf(__fsub_rn(u, v)));
    } else {
        const float t = __fsub_rn(u, v);
        return __fadd_rn(acc, __fmul_rn(t, t));
    }
}

// Packed element-wise sub/mul (sm_100 FADD2 / FMUL2): each element is the
// same IEEE round-to-nearest operation as __fsub_rn / __fmul_rn, two per
// instruction.  The accumulating adds stay scalar and in fold order, so the
// folds below are bit-identical to fold_step with a third fewer instructions.
__device__ __forceinline__ void sub2_rn(float a0, float a1, float b0, float b1, float& r0, float& r1) {
    asm("{\n\t.reg .b64 x, y, r;\n\tmov.b64 x, {%2, %3};\n\tmov.b64 y, {%4, %5};\n\t"
        "sub.rn.f32x2 r, x, y;\n\tmov.b64 {%0, %1}, r;\n\t}"
        : "=f"(r0), "=f"(r1)
        : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}
__device__ __forceinline__ void mul2_rn(float a0, float a1, float b0, float b1, float& r0, float& r1) {
    asm("{\n\t.reg .b64 x, y, r;\n\tmov.b64 x, {%2, %3};\n\tmov.b64 y, {%4, %5};\n\t"
        "mul.rn.f32x2 r, x, y;\n\tmov.b64 {%0, %1}, r;\n\t}"
        : "=f"(r0), "=f"(r1)
        : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}

// The fold's per-coordinate term (u, v) -> t for two coordinates at once.
template <int METRIC>
__device__ __forceinline__ void fold_terms2(float u0, float u1, float v0, float v1, float& t0, float& t1) {
    if constexpr (METRIC == kCosine) {
        mul2_rn(u0, u1, v0, v1, t0, t1);
    } else if constexpr (METRIC == kManhattan) {
        sub2_rn(u0, u1, v0, v1, t0, t1);
        t0 = fabsf(t0);
        t1 = fabsf(t1);
    } else {
        sub2_rn(u0, u1, v0, v1, t0, t1);
        mul2_rn(t0, t1, t0, t1, t0, t1);
    }
}

// Two independent folds one step each: acc0 += term(u0, v0), acc1 += term(u1, v1).
template <int METRIC>
__device__ __forceinline__ void fold_step2(float u0, float u1, float v0, float v1, float& acc0, float& acc1) {
    float t0, t1;
    fold_terms2<METRIC>(u0, u1, v0, v1, t0, t1);
    acc0 = __fadd_rn(acc0, t0);
    acc1 = __fadd_rn(acc1, t1);
}

// One fold, two consecutive coordinates (j, j + 1): the adds in order.
template <int METRIC>
__device__ __forceinline__ float fold_step_x2(float u0, float u1, float v0, float v1, float acc) {
    float t0, t1;
    fold_terms2<METRIC>(u0, u1, v0, v1, t0, t1);
    return __fadd_rn(__fadd_rn(acc, t0), t1);
}

template <int METRIC>
__device__ __forceinline__ float fold_finalize(float acc) {
    if constexpr (METRIC == kCosine) {
        return __fsub_rn(1.0f, acc);
    } else if constexpr (METRIC == kRootSquares) {
        return __fsqrt_rn(acc);
    } else {
        return acc;
    }
}

}  // namespace knnb
