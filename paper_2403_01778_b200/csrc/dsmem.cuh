// Point-to-point messages between the CTAs of one thread-block cluster: a
// value is stored into the same shared-memory slot of another CTA with
// st.async, which counts its bytes on that CTA's mbarrier (transaction
// count); the receiver arms the barrier with the bytes it expects and waits
// on its phase.  No cluster barrier: the complete_tx has release semantics at
// cluster scope (it orders the sender's earlier memory operations), the
// receiver's try_wait acquires.  Used by the Bunch-Kaufman panel (bk.cu) and
// the single-cluster Lanczos kernel (lanczos.cu).
#pragma once

#include <cstdint>

namespace r1 {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init1(uint64_t* bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_init_fence() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// v -> the same shared-memory slot of CTA `rank`, counted on its mbarrier `bar`
__device__ __forceinline__ void send8(const void* slot, double v, const uint64_t* bar, int rank) {
    uint32_t ra, rb;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(slot)), "r"(rank));
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(smem_u32(bar)), "r"(rank));
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(ra), "d"(v),
                 "r"(rb)
                 : "memory");
}

// one arrival that also expects `bytes` of messages on `bar` (this phase)
__device__ __forceinline__ void expect_bytes(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void wait_parity(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "R1_MBAR_WAIT_%=:\n"
        " mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra R1_MBAR_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

}  // namespace r1
