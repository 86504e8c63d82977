// Exclusive prefix sums over device arrays (reduce-then-scan, 3 launches).
// Used for row offsets, unique-block offsets and compaction; all integer, so
// the result is exact and order-independent.
#pragma once

#include "common.cuh"

namespace adipc_gpu {
namespace {  // internal linkage: every TU that scans gets its own kernels

constexpr int kScanThreads = 512;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;

template <class T>
__device__ __forceinline__ std::int64_t block_exclusive_scan(std::int64_t v, std::int64_t* sm, std::int64_t* total) {
    // warp inclusive scan
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    std::int64_t x = v;
    for (int o = 1; o < 32; o <<= 1) {
        std::int64_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) sm[w] = x;
    __syncthreads();
    if (w == 0) {
        const int nw = blockDim.x >> 5;
        std::int64_t s = lane < nw ? sm[lane] : 0;
        for (int o = 1; o < 32; o <<= 1) {
            std::int64_t y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        if (lane < nw) sm[lane] = s;
    }
    __syncthreads();
    const std::int64_t warp_off = w > 0 ? sm[w - 1] : 0;
    if (total) *total = sm[(blockDim.x >> 5) - 1];
    return warp_off + x - v;
}

template <class T>
__global__ void k_scan_tiles(const T* __restrict__ in, std::int64_t n, std::int64_t* __restrict__ out,
                             std::int64_t* __restrict__ tile_sums) {
    __shared__ std::int64_t sm[32];
    const std::int64_t base = static_cast<std::int64_t>(blockIdx.x) * kScanTile + threadIdx.x * kScanItems;
    std::int64_t v[kScanItems];
    std::int64_t local = 0;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        const std::int64_t idx = base + i;
        v[i] = idx < n ? static_cast<std::int64_t>(in[idx]) : 0;
        local += v[i];
    }
    std::int64_t total;
    std::int64_t off = block_exclusive_scan<T>(local, sm, &total);
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        const std::int64_t idx = base + i;
        if (idx < n) out[idx] = off;
        off += v[i];
    }
    if (threadIdx.x == 0) tile_sums[blockIdx.x] = total;
}

__global__ void k_scan_tile_sums(std::int64_t* __restrict__ sums, std::int64_t n_tiles, std::int64_t* __restrict__ grand) {
    __shared__ std::int64_t sm[32];
    std::int64_t carry = 0;
    for (std::int64_t base = 0; base < n_tiles; base += blockDim.x) {
        const std::int64_t i = base + threadIdx.x;
        const std::int64_t v = i < n_tiles ? sums[i] : 0;
        std::int64_t total;
        const std::int64_t ex = block_exclusive_scan<std::int64_t>(v, sm, &total);
        if (i < n_tiles) sums[i] = carry + ex;
        carry += total;
        __syncthreads();
    }
    if (threadIdx.x == 0) *grand = carry;
}

__global__ void k_scan_add(std::int64_t* __restrict__ out, std::int64_t n, const std::int64_t* __restrict__ tile_offs,
                           const std::int64_t* __restrict__ grand) {
    const std::int64_t base = static_cast<std::int64_t>(blockIdx.x) * kScanTile;
    const std::int64_t add = tile_offs[blockIdx.x];
    for (int i = threadIdx.x; i < kScanTile; i += blockDim.x) {
        const std::int64_t idx = base + i;
        if (idx < n) out[idx] += add;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) out[n] = *grand;
}

// out[0..n] = exclusive scan of in[0..n), out[n] = total. `scratch` must hold
// ceil(n / kScanTile) + 1 int64.
template <class T>
inline void exclusive_scan(const T* in, std::int64_t n, std::int64_t* out, DBuf<std::int64_t>& scratch,
                           cudaStream_t st) {
    const std::int64_t tiles = ceil_div(n, kScanTile) > 0 ? ceil_div(n, kScanTile) : 1;
    scratch.reserve(tiles + 1);
    k_scan_tiles<T><<<tiles, kScanThreads, 0, st>>>(in, n, out, scratch.p);
    ADIPC_LAUNCH_CHECK();
    k_scan_tile_sums<<<1, 1024, 0, st>>>(scratch.p, tiles, scratch.p + tiles);
    ADIPC_LAUNCH_CHECK();
    k_scan_add<<<tiles, kScanThreads, 0, st>>>(out, n, scratch.p, scratch.p + tiles);
    ADIPC_LAUNCH_CHECK();
}

}  // namespace
}  // namespace adipc_gpu
