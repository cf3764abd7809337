// mbarrier helpers shared by the ring kernels (dedisp.cu, dedisp_h16.cu): a slot's `full`
// and `empty` barriers count warp arrivals; waits spin on try_wait.parity with acquire
// semantics, arrivals release the arriving warp's prior shared-memory writes.
#pragma once

#include <cstdint>

namespace pgb {
namespace {

__device__ __forceinline__ uint32_t sh_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void ring_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sh_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void ring_inval(uint64_t* bar) {
    asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(sh_addr(bar)) : "memory");
}
__device__ __forceinline__ void ring_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(sh_addr(bar)) : "memory");
}
__device__ __forceinline__ void ring_wait(uint64_t* bar, uint32_t parity) {
    const uint32_t a = sh_addr(bar);
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(a), "r"(parity)
            : "memory");
    }
}

}  // namespace
}  // namespace pgb
