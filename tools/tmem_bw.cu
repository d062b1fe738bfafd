// TMEM read bandwidth microbenchmark (dev tool, not product code).
// One CTA per SM allocates 512 TMEM columns; NW warps (warp w reads lane
// quadrant w % 4) repeatedly tcgen05.ld 32x32b.x32 (+ wait::ld) over their
// share of the columns.  Prints bytes per clock per SM for NW = 4, 8, 12, 16
// and for 1, 2 or 4 loads in flight per wait.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/tmem_bw tools/tmem_bw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "../paper_0906_0231_b200/csrc/sm100_ptx.cuh"

using namespace knnb;

template <int INFL>
__global__ void tmem_bw_kernel(int reps, unsigned long long* cycles, uint32_t* sink) {
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if (warp == 0) ptx::tmem_alloc(ptx::smem_u32(&slot), 512);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = slot;
    const int quad = warp & 3, per_quad = nw / 4, sub = warp >> 2;
    const uint32_t cols = 512 / per_quad;  // this warp's columns
    const uint32_t base = tmem + (uint32_t(quad * 32) << 16) + sub * cols;
    uint32_t acc = 0;
    __syncthreads();
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
        for (uint32_t c = 0; c < cols; c += 32 * INFL) {
            uint32_t v[INFL][32];
#pragma unroll
            for (int i = 0; i < INFL; ++i) ptx::tmem_ld_32x32b_x32(base + c + 32 * i, v[i]);
            ptx::tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < INFL; ++i)
#pragma unroll
                for (int j = 0; j < 32; ++j) acc ^= v[i][j];
        }
    }
    __syncthreads();
    const long long t1 = clock64();
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
    if (acc == 0x12345678u) sink[0] = acc;
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem, 512);
    }
}

template <int INFL>
static void run(int nw, int reps) {
    unsigned long long* cyc;
    uint32_t* sink;
    cudaMalloc(&cyc, 148 * 8);
    cudaMalloc(&sink, 4);
    tmem_bw_kernel<INFL><<<148, 32 * nw>>>(reps, cyc, sink);
    tmem_bw_kernel<INFL><<<148, 32 * nw>>>(reps, cyc, sink);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[148];
    cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < 148; ++i) avg += double(h[i]) / 148;
    const double bytes = double(reps) * 128 * 512 * 4;  // whole 128 x 512 fp32 TMEM per rep
    printf("warps %2d in-flight %d: %.1f B/clk/SM (%s)\n", nw, INFL, bytes / avg, cudaGetErrorString(e));
    cudaFree(cyc);
    cudaFree(sink);
}

int main() {
    const int reps = 2000;
    for (int nw : {4, 8, 16}) {
        run<1>(nw, reps);
        run<2>(nw, reps);
        if (nw <= 8) run<4>(nw, reps);
    }
    return 0;
}
