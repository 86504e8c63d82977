// Bulk-copy (TMA, cp.async.bulk) + mbarrier helpers for sm_100a (inline PTX).
// Used to stage contiguous tiles (matrix tiles, MAS subdomain inverses) in
// shared memory ahead of use, so the bytes in flight per SM are bounded by
// shared memory instead of registers.
#pragma once

#include <cstdint>

namespace adipc_gpu {

__device__ __forceinline__ std::uint32_t smem_u32(const void* p) {
    return static_cast<std::uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(std::uint64_t* bar, std::uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

// make mbarrier initialisation visible to the async (TMA) proxy
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }

// order this thread's prior generic-proxy smem accesses before subsequent
// async-proxy writes (re-filling a buffer that was just read)
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ void mbar_arrive_expect_tx(std::uint64_t* bar, std::uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

// global -> shared bulk copy completing `bytes` of transaction on `bar`.
// src, dst 16-byte aligned, bytes a multiple of 16.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, std::uint32_t bytes, std::uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// same, with an L2 evict-first hint (data read exactly once per pass)
__device__ __forceinline__ void bulk_g2s_evict_first(void* dst, const void* src, std::uint32_t bytes,
                                                     std::uint64_t* bar) {
    std::uint64_t policy;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}

// same, with an L2 evict-last hint (small operands re-read every iteration)
__device__ __forceinline__ void bulk_g2s_evict_last(void* dst, const void* src, std::uint32_t bytes,
                                                    std::uint64_t* bar) {
    std::uint64_t policy;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(policy));
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}

// L2 cache policies for explicit residency control of streamed operands
__device__ __forceinline__ std::uint64_t policy_evict_last() {
    std::uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ std::uint64_t policy_evict_first() {
    std::uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ double ld_nc_policy(const double* ptr, std::uint64_t pol) {
    double v;
    asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(ptr), "l"(pol));
    return v;
}
__device__ __forceinline__ std::uint32_t ld_nc_policy(const std::uint32_t* ptr, std::uint64_t pol) {
    std::uint32_t v;
    asm volatile("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(ptr), "l"(pol));
    return v;
}

// Read-only gather that the compiler may not sink below later code (volatile
// asm statements keep their relative order): used to put all the gathers of a
// block in flight at once instead of one dependent round trip after another.
__device__ __forceinline__ double ldg_issue(const double* ptr) {
    double v;
    asm volatile("ld.global.nc.f64 %0, [%1];" : "=d"(v) : "l"(ptr));
    return v;
}

__device__ __forceinline__ std::int32_t ldg_issue(const std::int32_t* ptr) {
    std::int32_t v;
    asm volatile("ld.global.nc.s32 %0, [%1];" : "=r"(v) : "l"(ptr));
    return v;
}
__device__ __forceinline__ std::int64_t ldg_issue(const std::int64_t* ptr) {
    std::int64_t v;
    asm volatile("ld.global.nc.s64 %0, [%1];" : "=l"(v) : "l"(ptr));
    return v;
}

// Fire-and-forget fp64 add to global memory. Spelled out as `red` because
// nvcc emits ATOMG (with a return path through L1) instead of REDG for
// atomicAdd in kernels that also use a returning atomic + fence (the
// last-block-done reductions): measured 81 vs 59 us for the cfg5 SpMV.
__device__ __forceinline__ void red_add(double* ptr, double v) {
    asm volatile("red.global.add.f64 [%0], %1;" ::"l"(ptr), "d"(v));
}

// 256-bit read-only gather (sm_100: LDG.E.256) of a slot padded to 4 doubles
__device__ __forceinline__ void ldg_v4(const double* ptr, double& a, double& b, double& c, double& d) {
    asm volatile("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(ptr));
}

__device__ __forceinline__ void mbar_wait(std::uint64_t* bar, std::uint32_t parity) {
    std::uint32_t done;
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    } while (!done);
}

}  // namespace adipc_gpu
