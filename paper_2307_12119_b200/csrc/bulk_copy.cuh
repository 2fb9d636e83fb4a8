// bulk_copy.cuh — 1-D TMA bulk copies (cp.async.bulk) global -> shared with an
// mbarrier transaction count, for the row passes' per-warp input staging: one
// lane requests a whole row (several contiguous segments) for the NEXT work
// item while the warp computes the current one, so the row's HBM latency is
// hidden without holding registers (SASS: UBLKCP, SYNCS.ARRIVE.TRANS64).
#pragma once

#include <cstdint>

namespace gtb {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// One arrival (the issuing lane) completes the phase once `bytes` have landed.
__device__ __forceinline__ void mbar_init(uint64_t* mb, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(mb)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* mb, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(mb)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* mb, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(mb)),
        "r"(parity)
        : "memory");
}

// Orders this thread's earlier generic-proxy shared accesses (after a
// __syncwarp, the whole warp's) before the async-proxy writes that follow.
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// bytes: multiple of 16; src, dst: 16-byte aligned.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* mb) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(mb))
        : "memory");
}

}  // namespace gtb
