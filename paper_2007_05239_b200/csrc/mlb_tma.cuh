// Asynchronous global -> shared staging for sm_100a.
//
//  * tma_load_1d: one-dimensional bulk copy through the Tensor Memory
//    Accelerator (cp.async.bulk ... mbarrier::complete_tx, SASS UBLKCP),
//    completion tracked by an mbarrier; for contiguous, 16-byte aligned
//    tables (twiddles, spatial kernels, grid slabs).
//  * cp_async8 / cp_async16: per-element LDGSTS copies for strided tiles; the
//    issuing thread does not block until cp_async_wait_all().
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace mlb {

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_addr(bar)),
        "r"(phase)
        : "memory");
}

// bytes: multiple of 16; src/dst 16-byte aligned
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
            smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}

// Stage n_bytes (rounded up to 16; the source allocation must cover it) from
// global to shared with chunked bulk copies issued by one thread; every
// thread of the CTA waits.  `bar` must be initialised (count 1) and fenced.
__device__ __forceinline__ void tma_stage(void* dst, const void* src, uint32_t n_bytes, uint64_t* bar,
                                          uint32_t phase) {
    const uint32_t total = (n_bytes + 15u) & ~15u;
    if (threadIdx.x == 0) {
        mbar_arrive_expect_tx(bar, total);
        constexpr uint32_t kChunkBytes = 32768;
        for (uint32_t off = 0; off < total; off += kChunkBytes) {
            const uint32_t b = (total - off < kChunkBytes) ? (total - off) : kChunkBytes;
            tma_load_1d(static_cast<char*>(dst) + off, static_cast<const char*>(src) + off, b, bar);
        }
    }
    mbar_wait(bar, phase);
}

__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_addr(dst)), "l"(src) : "memory");
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_addr(dst)), "l"(src) : "memory");
}

__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait_group() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

}  // namespace mlb
