// Tensor-memory-accelerator (TMA) plane loads for the stencil kernels: a
// tile plane of a full-grid f64 vector (tile + one-cell halo, box 68 x VH x 1
// cells) lands in shared memory with one cp.async.bulk.tensor issued by one
// thread, completing on an mbarrier. Out-of-domain cells of the box are
// zero-filled by the hardware (the outside of the domain is zero in every
// solver vector), so the halo needs no bounds logic.
#pragma once

#include <cuda.h>

#include "common.cuh"

namespace nb2 {

// Tensor maps of every solver vector a stencil kernel reads with TMA: d
// (Dtmp), the direction ring slots, the two x buffers. Passed by value as a
// __grid_constant__ kernel parameter; rebuilt when a buffer moves.
constexpr int kMapD = 0, kMapRing = 1, kMapX0 = 1 + kRing, kMapX1 = 2 + kRing, kNumMaps = 3 + kRing;
struct TmaMaps {
    CUtensorMap m[kNumMaps];
};

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
// one arrival (the issuing thread) plus the bytes the loads will deliver
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// generic-proxy accesses of shared memory before this point are ordered
// before later async-proxy (TMA) writes to it
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int x, int y, int z, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];\n" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<unsigned long long>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_prefetch_map(const CUtensorMap* map) {
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<unsigned long long>(map)) : "memory");
}

}  // namespace nb2
