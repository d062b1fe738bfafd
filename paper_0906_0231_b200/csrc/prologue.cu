// prologue.cu -- HBM-bound passes that run before the distance sweep.
//
//   validate : every coordinate finite (Dataset ctor, src/dataset.cpp:23-29)
//              and inside the metric's domain (Hellinger coord_valid x >= 0,
//              src/distance.cpp:18, checked by validate_dataset :57-59).  The
//              first offending flat index is found with atomicMin so the
//              error message names the same vector/coordinate the reference's
//              sequential scan would.
//   stage    : Hellinger's sqrt staging (include/knn/distance.hpp:47), applied
//              once per coordinate with IEEE sqrtf (correctly rounded, so
//              step over raw values == step_staged over staged values).
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "kernels.h"

namespace knnb {

__global__ void validate_kernel(const float* __restrict__ X, uint64_t count, int check_nonneg,
                                unsigned long long* __restrict__ first_nonfinite,
                                unsigned long long* __restrict__ first_domain) {
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += stride) {
        const float v = X[i];
        if (!isfinite(v)) atomicMin(first_nonfinite, (unsigned long long)i);
        else if (check_nonneg && !(v >= 0.0f)) atomicMin(first_domain, (unsigned long long)i);
    }
}

__global__ void stage_sqrt_kernel(const float* __restrict__ X, float* __restrict__ Y, uint64_t count,
                                  int vec) {
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    const uint64_t n4 = vec ? count / 4 : 0;
    const float4* X4 = reinterpret_cast<const float4*>(X);
    float4* Y4 = reinterpret_cast<float4*>(Y);
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += stride) {
        float4 v = X4[i];
        v.x = __fsqrt_rn(v.x);
        v.y = __fsqrt_rn(v.y);
        v.z = __fsqrt_rn(v.z);
        v.w = __fsqrt_rn(v.w);
        Y4[i] = v;
    }
    for (uint64_t i = n4 * 4 + uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += stride)
        Y[i] = __fsqrt_rn(X[i]);
}

// Reference generate_dataset (io.cpp:57-62) with the SplitMix64 of
// rng.hpp:13-23.  The generator state after i+1 calls is seed + (i+1)*gamma,
// so every element is independent and the device output is bit-identical to
// the host stream.
__global__ void generate_kernel(float* __restrict__ out, uint64_t count, uint64_t seed) {
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += stride) {
        uint64_t z = seed + (i + 1) * 0x9e3779b97f4a7c15ull;
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        z = z ^ (z >> 31);
        out[i] = __fmul_rn(float(uint32_t(z >> 40)), 0x1.0p-24f);
    }
}

static unsigned grid_for(uint64_t count, int sm_count) {
    const uint64_t want = (count + 255) / 256;
    const uint64_t cap = uint64_t(sm_count) * 8;
    return unsigned(want < cap ? (want ? want : 1) : cap);
}

cudaError_t launch_validate(const float* X, uint64_t count, int check_nonneg,
                            unsigned long long* flags, int sm_count, cudaStream_t stream) {
    validate_kernel<<<grid_for(count, sm_count), 256, 0, stream>>>(X, count, check_nonneg, flags,
                                                                    flags + 1);
    return cudaGetLastError();
}

cudaError_t launch_stage_sqrt(const float* X, float* Y, uint64_t count, int sm_count,
                              cudaStream_t stream) {
    // X and Y come from cudaMalloc / the caller's device buffer; the float4
    // path needs 16-byte alignment, checked here.
    const int vec = ((reinterpret_cast<uintptr_t>(X) | reinterpret_cast<uintptr_t>(Y)) & 15u) == 0;
    stage_sqrt_kernel<<<grid_for(vec ? count / 4 + 1 : count, sm_count), 256, 0, stream>>>(X, Y, count,
                                                                                           vec);
    return cudaGetLastError();
}

cudaError_t launch_generate(float* out, uint64_t count, uint64_t seed, int sm_count, cudaStream_t stream) {
    generate_kernel<<<grid_for(count, sm_count), 256, 0, stream>>>(out, count, seed);
    return cudaGetLastError();
}

}  // namespace knnb
