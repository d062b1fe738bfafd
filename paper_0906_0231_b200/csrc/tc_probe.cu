// tc_probe.cu -- raw tcgen05 dot products, for measuring the accumulation
// error the TENSOR policy's completeness proof allows for.
//
// The proof bounds the tensor core's FP32 accumulation of exact fp16 products
// by c * d * 2^-23 * ||a|| ||b|| with c = kTcSafety = 4.  This kernel runs the
// sweep's own instruction -- tcgen05.mma.cta_group::1.kind::f16, M = 128,
// N = 256, K = 16 per instruction, 64-wide K chunks in SWIZZLE_128B K-major
// shared memory, FP32 accumulator in TMEM -- on caller-given fp16 rows and
// returns every dot, so tests can compare them with exact (fp64) dots on
// adversarial inputs and report how much of c is used.  Test/measurement
// infrastructure of the proof, not a solve path.
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "kernels.h"
#include "sm100_ptx.cuh"

namespace knnb {

namespace {

constexpr int TP_M = 128, TP_N = 256;

// One CTA: rows [128 bx, +128) of A against rows [256 by, +256) of B, all of
// K; out[i][j] = sum_k A[i][k] B[j][k] as the tensor core accumulates it.
__global__ void __launch_bounds__(128, 1)
tc_dot_kernel(const __half* __restrict__ A, uint32_t m, const __half* __restrict__ B, uint32_t n, uint32_t d,
              float* __restrict__ out) {
    extern __shared__ uint8_t tp_smem_raw[];  // A chunk | B chunk, 1024-aligned
    uint8_t* sa = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(tp_smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sb = sa + TP_M * 128;
    __shared__ uint64_t bar;
    __shared__ uint32_t tmem_slot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t r0 = blockIdx.x * TP_M, c0 = blockIdx.y * TP_N;
    if (threadIdx.x == 0) {
        ptx::mbar_init(ptx::smem_u32(&bar), 1);
        ptx::fence_mbar_init();
    }
    if (warp == 0) ptx::tmem_alloc(ptx::smem_u32(&tmem_slot), TP_N);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = tmem_slot;
    constexpr uint32_t idesc = ptx::idesc_f16_f32(TP_M, TP_N);
    uint32_t phase = 0;
    for (uint32_t k0 = 0; k0 < d; k0 += 64) {
        // stage the 64-wide K chunk in the SW128 K-major layout: row r's
        // 16-byte unit u sits at r * 128 + ((u ^ (r & 7)) << 4); K past d is 0
        auto stage = [&](const __half* src, uint32_t rows, uint32_t row0, uint32_t nmax, uint8_t* dst) {
            for (uint32_t i = threadIdx.x; i < rows * 8; i += blockDim.x) {
                const uint32_t r = i >> 3, u = i & 7;
                uint32_t w[4] = {0, 0, 0, 0};
                for (int q = 0; q < 8; ++q) {
                    const uint32_t k = k0 + u * 8 + q;
                    const uint16_t h = (row0 + r < nmax && k < d)
                                           ? __half_as_ushort(src[size_t(row0 + r) * d + k]) : uint16_t(0);
                    w[q >> 1] |= uint32_t(h) << (16 * (q & 1));
                }
                *reinterpret_cast<uint4*>(dst + r * 128 + ((u ^ (r & 7)) << 4)) = make_uint4(w[0], w[1], w[2], w[3]);
            }
        };
        stage(A, TP_M, r0, m, sa);
        stage(B, TP_N, c0, n, sb);
        ptx::fence_proxy_async_smem();  // generic-proxy smem writes -> visible to the tensor core
        __syncthreads();
        if (threadIdx.x == 0) {
            ptx::tc_fence_after();
#pragma unroll
            for (uint32_t kk = 0; kk < 4; ++kk)
                ptx::mma_f16_ss(tmem, ptx::sw128_kmajor_desc(ptx::smem_u32(sa) + 32 * kk),
                                ptx::sw128_kmajor_desc(ptx::smem_u32(sb) + 32 * kk), idesc, (k0 | kk) != 0);
            ptx::mma_commit(ptx::smem_u32(&bar));
        }
        ptx::mbar_wait(ptx::smem_u32(&bar), phase);  // the chunk's MMAs are done: smem may be restaged
        phase ^= 1;
        ptx::tc_fence_after();
    }
    // TMEM lane = row (warp w: rows 32 w .. 32 w + 31), column = B row
    const uint32_t row = r0 + warp * 32 + lane;
    for (uint32_t c = 0; c < TP_N; c += 32) {
        uint32_t v[32];
        ptx::tmem_ld_32x32b_x32(tmem + (uint32_t(warp * 32) << 16) + c, v);
        ptx::tmem_wait_ld();
        if (row < m)
            for (int j = 0; j < 32; ++j)
                if (c0 + c + j < n) out[size_t(row) * n + c0 + c + j] = __uint_as_float(v[j]);
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem, TP_N);
    }
}

}  // namespace

cudaError_t launch_tc_dots(const void* a_f16, uint32_t m, const void* b_f16, uint32_t n, uint32_t d, float* out,
                           cudaStream_t stream) {
    if (m == 0 || n == 0 || d == 0) return cudaSuccess;
    const dim3 grid((m + TP_M - 1) / TP_M, (n + TP_N - 1) / TP_N);
    const int smem = (TP_M + TP_N) * 128 + 1024;
    cudaError_t e = cudaFuncSetAttribute(tc_dot_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    tc_dot_kernel<<<grid, 128, smem, stream>>>(static_cast<const __half*>(a_f16), m, static_cast<const __half*>(b_f16),
                                            n, d, out);
    return cudaGetLastError();
}

}  // namespace knnb
