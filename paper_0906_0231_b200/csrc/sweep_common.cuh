// sweep_common.cuh -- per-row candidate lists shared by the tensor sweeps.
#pragma once

#include <stdint.h>

#include "common.cuh"

namespace knnb {

// Per-row candidate list: KPL unsorted (y, index) entries in shared memory --
// a [KPL][LIST_ROWS] float array and a [KPL][LIST_ROWS] index array, so the
// 32 lanes of a warp touch consecutive words -- plus its maximum, the
// admission threshold (the reference's heap root, heap.hpp:86-90).  The list
// keeps the KPL smallest y with ties broken arbitrarily: the completeness
// proof only needs "every column outside the list has y >= the list maximum".
// Replacing the maximum and rescanning costs KPL independent shared loads and
// runs warp-convergently: a warp pays once per column any of its rows admits.
struct ListMax {
    float a;
    uint32_t slot;
};

__device__ __forceinline__ float lds_f32(uint32_t addr) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
    return v;
}

__device__ __forceinline__ void sts_f32(uint32_t addr, float v) {
    asm volatile("st.shared.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}

__device__ __forceinline__ void sts_u32(uint32_t addr, uint32_t v) {
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}

template <int KPL, uint32_t STRIDE>
__device__ __forceinline__ ListMax list_rescan(uint32_t a_base) {
    // pass 1: maximum (independent loads, a max tree); pass 2: its slot
    float m = lds_f32(a_base);
#pragma unroll 32
    for (int i = 1; i < KPL; ++i) m = fmaxf(m, lds_f32(a_base + i * STRIDE));
    uint32_t slot = 0;
#pragma unroll 32
    for (int i = KPL - 1; i >= 0; --i) slot = (lds_f32(a_base + i * STRIDE) == m) ? uint32_t(i) : slot;
    return ListMax{m, slot};
}

template <int KPL, uint32_t STRIDE>
__device__ __noinline__ ListMax list_replace_max(uint32_t a_base, uint32_t i_base, uint32_t slot, float a,
                                                 uint32_t col) {
    sts_f32(a_base + slot * STRIDE, a);
    sts_u32(i_base + slot * STRIDE, col);
    return list_rescan<KPL, STRIDE>(a_base);
}

}  // namespace knnb
