// Hessian assembly on B200: replaces sort_stream + fast_hash_reduction
// (sparse/block_coo.hpp:67-113, sparse/reduction.hpp:30-107) as called at
// solver/incremental_potential.hpp:256-257.
//
// The reference sorts 64-bit (row, col) keys with a serial 4 x 16-bit LSD
// radix sort, gathers the 72-byte blocks through the permutation, scans key
// changes serially and sums each segment left to right (deterministic mode).
// Here the same result is produced by exploiting that keys are block
// coordinates with row < n:
//   1. row histogram (atomics)                         -> row_cnt[n]
//   2. exclusive scan                                  -> row_start[n+1]
//   3. bucket scatter of (col << 32 | emission index)  -> sorted[T]
//      (atomic slot order, fixed in 4)
//   4. per-row sort of (col, index) in registers/shared memory; sorting by the
//      emission index as the low word reproduces a *stable* sort exactly
//   5. unique-col count per row + scan                 -> row_ptr / U
//   6. per unique block: sequential fp64 sum in emission order of the gathered
//      72-byte values (never materialising the sorted value copy, K2 fused
//      into K4), written straight to rows/cols/blocks.
// Step 6 reproduces the reference's deterministic mode bit for bit
// (reduction.hpp:39-53: left-to-right adds, no FMA involved); the parallel
// mode of the reference differs from it only by rounding (<= 1e-12).
#include <algorithm>
#include <vector>

#include "context.hpp"
#include "scan.cuh"

namespace adipc_gpu {

namespace {

constexpr int kWarpSortMax = 128;   // rows up to this length: one warp, register bitonic
constexpr int kCtaSortMax = 8192;   // rows up to this length: one CTA, smem bitonic
constexpr int kCtaSortThreads = 1024;
constexpr int kHugeRow = 4 * kCtaSortMax;  // longer rows: multi-CTA chunk sort + merge-path passes
constexpr int kMergeTile = 4096;           // output elements per CTA of a merge pass

// The triplet stream as the kernels see it: up to two segments (the DOF
// stream, then the reduced contact tiles appended by two_level_abd_reduce,
// incremental_potential.hpp:392-394) and optionally filter_pinned
// (incremental_potential.hpp:410-425) applied on the fly: an entry touching a
// pinned slot is dropped, and every pinned slot s gets an I3 on its diagonal
// with emission index T1 + T2 + s (after every stream entry). The emission
// index of a kept entry is its index in the concatenated stream; the filter
// keeps order, so sorting by it is sorting in the filtered stream's order.
struct StreamSrc {
    const std::uint64_t* k1;
    const double* v1;
    std::int64_t T1;
    const std::uint64_t* k2;
    const double* v2;
    std::int64_t T2;
    const std::uint8_t* pinned;  // null: no filter
    std::int32_t n_pin;          // pinned slots (= n_block_rows when filtering)
    const std::uint32_t* vidx;   // optional: emission index of key i (sorted-stream callers), else i
    __device__ __forceinline__ std::int64_t total() const { return T1 + T2; }
    __device__ __forceinline__ std::uint64_t key(std::int64_t i) const { return i < T1 ? k1[i] : k2[i - T1]; }
    __device__ __forceinline__ bool kept(std::uint64_t k) const {
        return !pinned || !(pinned[static_cast<std::uint32_t>(k >> 32)] | pinned[static_cast<std::uint32_t>(k)]);
    }
    // address of the value of emission index q, or null for an appended I3
    __device__ __forceinline__ const double* value(std::uint32_t q) const {
        if (q < T1) return v1 + 9 * static_cast<std::int64_t>(q);
        if (q < T1 + T2) return v2 + 9 * (static_cast<std::int64_t>(q) - T1);
        return nullptr;
    }
};

// Warp-aggregated atomicAdd on a per-row counter: lanes with the same row
// share one atomic (FEM streams emit an element's blocks consecutively, so a
// warp's 32 entries touch few rows); returns this lane's slot among them.
__device__ __forceinline__ std::int32_t aggregated_add(std::int32_t* ctr, std::uint32_t row, bool valid) {
    const unsigned grp = __match_any_sync(0xffffffffu, valid ? row : 0xFFFFFFFFu);
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(grp) - 1;
    std::int32_t base = 0;
    if (valid && lane == leader) base = atomicAdd(ctr + row, __popc(grp));
    base = __shfl_sync(0xffffffffu, base, leader);
    return base + __popc(grp & ((1u << lane) - 1u));
}

// 1. row histogram of the kept entries (+ one I3 per pinned slot). Each
//    thread keeps kIlp independent keys in flight (coalesced: key i + k *
//    blockDim of its CTA's window).
constexpr int kIlp = 4;
__global__ void __launch_bounds__(256) k_row_hist(StreamSrc s, std::int32_t n, std::int32_t* __restrict__ row_cnt,
                                                  std::int32_t* __restrict__ err) {
    const std::int64_t T = s.total();
    const std::int64_t stride = static_cast<std::int64_t>(gridDim.x) * blockDim.x * kIlp;
    for (std::int64_t b = blockIdx.x * static_cast<std::int64_t>(blockDim.x) * kIlp; b < T; b += stride) {
        std::uint64_t k[kIlp];
#pragma unroll
        for (int u = 0; u < kIlp; ++u) {
            const std::int64_t i = b + threadIdx.x + u * blockDim.x;
            k[u] = i < T ? s.key(i) : ~0ull;
        }
#pragma unroll
        for (int u = 0; u < kIlp; ++u) {
            const std::uint32_t row = static_cast<std::uint32_t>(k[u] >> 32);
            bool valid = k[u] != ~0ull;
            if (valid && (row >= static_cast<std::uint32_t>(n) ||
                          (s.pinned && static_cast<std::uint32_t>(k[u]) >= static_cast<std::uint32_t>(s.n_pin)))) {
                atomicOr(err, 1);
                valid = false;
            }
            aggregated_add(row_cnt, row, valid && s.kept(k[u]));
        }
    }
    const std::int64_t tstride = static_cast<std::int64_t>(gridDim.x) * blockDim.x;
    if (s.pinned)
        for (std::int64_t q = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; q < s.n_pin; q += tstride)
            if (s.pinned[q]) atomicAdd(row_cnt + q, 1);
}

// 2. bucket scatter of (col << 32 | emission index) into the row's range
//    (slot order within a row is arbitrary here; fixed by the row sort)
__global__ void __launch_bounds__(256) k_row_scatter(StreamSrc s, std::int32_t n,
                                                     const std::int64_t* __restrict__ row_start,
                                                     std::int32_t* __restrict__ cursor,
                                                     std::uint64_t* __restrict__ out) {
    const std::int64_t T = s.total();
    const std::int64_t stride = static_cast<std::int64_t>(gridDim.x) * blockDim.x * kIlp;
    for (std::int64_t b = blockIdx.x * static_cast<std::int64_t>(blockDim.x) * kIlp; b < T; b += stride) {
        std::uint64_t k[kIlp];
        std::int64_t pos[kIlp];
#pragma unroll
        for (int u = 0; u < kIlp; ++u) {
            const std::int64_t i = b + threadIdx.x + u * blockDim.x;
            k[u] = i < T ? s.key(i) : ~0ull;
        }
#pragma unroll
        for (int u = 0; u < kIlp; ++u) {
            const std::uint32_t row = static_cast<std::uint32_t>(k[u] >> 32);
            const bool valid = k[u] != ~0ull && row < static_cast<std::uint32_t>(n) && s.kept(k[u]);
            const std::int32_t slot = aggregated_add(cursor, row, valid);
            pos[u] = valid ? row_start[row] + slot : -1;
        }
#pragma unroll
        for (int u = 0; u < kIlp; ++u) {
            const std::int64_t i = b + threadIdx.x + u * blockDim.x;
            if (pos[u] >= 0) out[pos[u]] = (k[u] << 32) | (s.vidx ? s.vidx[i] : static_cast<std::uint32_t>(i));
        }
    }
    const std::int64_t tstride = static_cast<std::int64_t>(gridDim.x) * blockDim.x;
    if (s.pinned)
        for (std::int64_t q = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; q < s.n_pin; q += tstride)
            if (s.pinned[q]) {
                const std::int64_t p = row_start[q] + atomicAdd(cursor + q, 1);
                out[p] = (static_cast<std::uint64_t>(q) << 32) | static_cast<std::uint32_t>(T + q);
            }
}

// Bitonic sort of s[0..N) (N power of two) by `nthr` cooperating threads.
template <bool kWarp>
__device__ __forceinline__ void bitonic(std::uint64_t* s, int N, int tid, int nthr) {
    for (int k = 2; k <= N; k <<= 1)
        for (int j = k >> 1; j > 0; j >>= 1) {
            // one compare-exchange per pair p: i = the pair's lower index
            // (bit j clear), its partner i + j — no idle half of the threads
            for (int p = tid; p < (N >> 1); p += nthr) {
                const int i = 2 * p - (p & (j - 1));
                const int ixj = i + j;
                const std::uint64_t a = s[i], b = s[ixj];
                const bool up = (i & k) == 0;
                if ((a > b) == up) {
                    s[i] = b;
                    s[ixj] = a;
                }
            }
            if (kWarp)
                __syncwarp();
            else
                __syncthreads();
        }
}

// Bitonic sort of 32 E 64-bit words held in registers, E per lane (element
// g = E lane + e): exchanges closer than E stay in a lane, the others are
// warp shuffles. No shared memory.
template <int E>
__device__ __forceinline__ void warp_bitonic(std::uint64_t (&v)[E], int lane) {
    constexpr int N = 32 * E;
#pragma unroll
    for (int k = 2; k <= N; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            if (j < E) {
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    const int p = e ^ j;
                    if (p > e) {
                        const bool up = ((lane * E + e) & k) == 0;
                        const std::uint64_t a = v[e], b = v[p];
                        if ((a > b) == up) {
                            v[e] = b;
                            v[p] = a;
                        }
                    }
                }
            } else {
                const int lj = j / E;
                const bool lower = (lane & lj) == 0;
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    const std::uint64_t o = __shfl_xor_sync(0xffffffffu, v[e], lj);
                    const bool up = ((lane * E + e) & k) == 0;
                    v[e] = (lower == up) ? (v[e] < o ? v[e] : o) : (v[e] < o ? o : v[e]);
                }
            }
        }
    }
}

template <int E>
__device__ __forceinline__ int warp_sort_row(std::uint64_t* seg, int len, int lane) {
    std::uint64_t v[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const int g = lane * E + e;
        v[e] = g < len ? seg[g] : ~0ull;
    }
    warp_bitonic<E>(v, lane);
    std::uint64_t prev = __shfl_up_sync(0xffffffffu, v[E - 1], 1);
    int uniq = 0;
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const int g = lane * E + e;
        if (g < len) {
            seg[g] = v[e];
            uniq += (g == 0 || (v[e] >> 32) != (prev >> 32)) ? 1 : 0;
        }
        prev = v[e];
    }
    for (int o = 16; o > 0; o >>= 1) uniq += __shfl_xor_sync(0xffffffffu, uniq, o);
    return uniq;
}

// 3. one warp per row: sort by (col, emission index) — the emission index as
//    the low word makes it the reference's STABLE order — and count unique
//    cols. Rows longer than kWarpSortMax are deferred to the CTA kernel.
__global__ void k_sort_rows_warp(std::uint64_t* __restrict__ sorted, const std::int64_t* __restrict__ row_start,
                                 std::int32_t n, std::int32_t* __restrict__ uniq_cnt,
                                 std::int32_t* __restrict__ big_rows, std::int32_t* __restrict__ n_big) {
    // n_big[0]: rows for k_sort_rows_cta (listed from big_rows[0] up);
    // n_big[1]: rows > kHugeRow (listed from big_rows[n - 1] down), n_big[2]: their longest
    const int lane = threadIdx.x & 31;
    const std::int32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const std::int32_t warps = (gridDim.x * blockDim.x) >> 5;
    for (std::int32_t r = warp; r < n; r += warps) {
        const std::int64_t b = row_start[r];
        const int len = static_cast<int>(row_start[r + 1] - b);
        std::uint64_t* seg = sorted + b;
        int uniq;
        if (len <= 1)
            uniq = len;
        else if (len <= 32)
            uniq = warp_sort_row<1>(seg, len, lane);
        else if (len <= 64)
            uniq = warp_sort_row<2>(seg, len, lane);
        else if (len <= kWarpSortMax)
            uniq = warp_sort_row<4>(seg, len, lane);
        else {
            if (lane == 0) {
                if (len > kHugeRow) {
                    big_rows[n - 1 - atomicAdd(n_big + 1, 1)] = r;
                    atomicMax(n_big + 2, len);
                } else {
                    big_rows[atomicAdd(n_big, 1)] = r;
                }
            }
            continue;
        }
        if (lane == 0) uniq_cnt[r] = uniq;
    }
}

// Merge two sorted runs a[0..na), b[0..nb) into out, cooperatively: each
// thread takes an equal slice of the output via a merge-path search.
__device__ void cta_merge(const std::uint64_t* a, int na, const std::uint64_t* b, int nb, std::uint64_t* out) {
    const int total = na + nb;
    const int per = (total + blockDim.x - 1) / blockDim.x;
    const int d0 = min(total, static_cast<int>(threadIdx.x) * per);
    const int d1 = min(total, d0 + per);
    if (d0 >= d1) return;
    auto split = [&](int d) {  // number of elements taken from a in the first d outputs
        int lo = max(0, d - nb), hi = min(d, na);
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (a[mid] <= b[d - mid - 1])  // a before b on ties (keys are unique anyway)
                lo = mid + 1;
            else
                hi = mid;
        }
        return lo;
    };
    int i = split(d0), j = d0 - i;
    for (int d = d0; d < d1; ++d) {
        if (j >= nb || (i < na && a[i] <= b[j]))
            out[d] = a[i++];
        else
            out[d] = b[j++];
    }
}

// One CTA per long row: shared-memory bitonic for rows <= kCtaSortMax,
// otherwise chunk sort + merge passes through `scratch` (rare: contact rows
// of affine bodies can collect very many tiles).
__global__ void k_sort_rows_cta(std::uint64_t* __restrict__ sorted, std::uint64_t* __restrict__ scratch,
                                const std::int64_t* __restrict__ row_start, const std::int32_t* __restrict__ big_rows,
                                const std::int32_t* __restrict__ n_big, std::int32_t* __restrict__ uniq_cnt) {
    extern __shared__ std::uint64_t s[];
    __shared__ int red[32];
    const int nb = *n_big;
    for (int bi = blockIdx.x; bi < nb; bi += gridDim.x) {
        const std::int32_t r = big_rows[bi];
        const std::int64_t b = row_start[r];
        const int len = static_cast<int>(row_start[r + 1] - b);
        std::uint64_t* seg = sorted + b;
        // sort chunks of kCtaSortMax in shared memory
        for (int c0 = 0; c0 < len; c0 += kCtaSortMax) {
            const int cl = min(kCtaSortMax, len - c0);
            int N = 2;
            while (N < cl) N <<= 1;
            for (int i = threadIdx.x; i < N; i += blockDim.x) s[i] = i < cl ? seg[c0 + i] : ~0ull;
            __syncthreads();
            bitonic<false>(s, N, threadIdx.x, blockDim.x);
            for (int i = threadIdx.x; i < cl; i += blockDim.x) seg[c0 + i] = s[i];
            __syncthreads();
        }
        // merge passes, ping-pong between seg and scratch
        std::uint64_t* src = seg;
        std::uint64_t* dst = scratch + b;
        for (int width = kCtaSortMax; width < len; width <<= 1) {
            for (int a0 = 0; a0 < len; a0 += 2 * width) {
                const int na = min(width, len - a0);
                const int nbb = min(width, max(0, len - a0 - width));
                cta_merge(src + a0, na, src + a0 + na, nbb, dst + a0);
            }
            __syncthreads();
            std::uint64_t* t = src;
            src = dst;
            dst = t;
        }
        if (src != seg) {
            for (int i = threadIdx.x; i < len; i += blockDim.x) seg[i] = src[i];
            __syncthreads();
        }
        int uniq = 0;
        for (int i = threadIdx.x; i < len; i += blockDim.x)
            uniq += (i == 0 || (seg[i] >> 32) != (seg[i - 1] >> 32)) ? 1 : 0;
        for (int o = 16; o > 0; o >>= 1) uniq += __shfl_xor_sync(0xffffffffu, uniq, o);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = uniq;
        __syncthreads();
        if (threadIdx.x == 0) {
            int t = 0;
            for (int i = 0; i < (blockDim.x >> 5); ++i) t += red[i];
            uniq_cnt[r] = t;
        }
        __syncthreads();
    }
}

// Rows longer than kHugeRow (contact rows of affine bodies: hundreds of
// thousands of entries) are sorted by the whole GPU instead of one CTA:
// every kCtaSortMax chunk of every such row by its own CTA (shared-memory
// bitonic), then log2 merge passes in which every kMergeTile-element tile
// of the output is one CTA (merge-path split of its pair of runs), ping-pong
// between `sorted` and `scratch`, and a final pass that moves odd-pass rows
// back and counts the unique columns. Rows are big_rows[n - 1 - y]; the
// host turns their lengths into exact (row, chunk / tile) work lists, so no
// CTA is launched past a row's end.
__device__ __forceinline__ int merge_split(const std::uint64_t* a, int na, const std::uint64_t* b, int nb, int d) {
    int lo = max(0, d - nb), hi = min(d, na);
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (a[mid] <= b[d - mid - 1])
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo;
}
__device__ __forceinline__ int huge_passes(int len) {
    int p = 0;
    for (int w = kCtaSortMax; w < len; w <<= 1) ++p;
    return p;
}
// (row, length) of the huge rows, for the host's work lists
__global__ void k_huge_info(const std::int32_t* __restrict__ huge_tail, const std::int64_t* __restrict__ row_start,
                            int nh, std::int32_t* __restrict__ info) {
    for (int y = blockIdx.x * blockDim.x + threadIdx.x; y < nh; y += gridDim.x * blockDim.x) {
        const std::int32_t r = huge_tail[-1 - y];
        info[2 * y] = r;
        info[2 * y + 1] = static_cast<std::int32_t>(row_start[r + 1] - row_start[r]);
    }
}
// work item k = (row r, chunk / tile x) at work[2 k], work[2 k + 1]
__global__ void __launch_bounds__(kCtaSortThreads) k_huge_chunks(std::uint64_t* __restrict__ sorted,
                                                                 const std::int64_t* __restrict__ row_start,
                                                                 const std::int32_t* __restrict__ work,
                                                                 std::int32_t* __restrict__ uniq_cnt) {
    extern __shared__ std::uint64_t s[];
    const std::int32_t r = work[2 * blockIdx.x];
    const std::int64_t b = row_start[r];
    const int len = static_cast<int>(row_start[r + 1] - b);
    const int c0 = work[2 * blockIdx.x + 1] * kCtaSortMax;
    if (c0 == 0 && threadIdx.x == 0) uniq_cnt[r] = 0;  // k_huge_finish adds the tiles' heads
    std::uint64_t* seg = sorted + b + c0;
    const int cl = min(kCtaSortMax, len - c0);
    int N = 2;
    while (N < cl) N <<= 1;
    for (int i = threadIdx.x; i < N; i += blockDim.x) s[i] = i < cl ? seg[i] : ~0ull;
    __syncthreads();
    bitonic<false>(s, N, threadIdx.x, blockDim.x);
    for (int i = threadIdx.x; i < cl; i += blockDim.x) seg[i] = s[i];
}
__global__ void __launch_bounds__(256) k_huge_merge(std::uint64_t* __restrict__ sorted,
                                                    std::uint64_t* __restrict__ scratch,
                                                    const std::int64_t* __restrict__ row_start,
                                                    const std::int32_t* __restrict__ work, int width, int pass) {
    __shared__ int split[2];
    const std::int32_t r = work[2 * blockIdx.x];
    const std::int64_t b = row_start[r];
    const int len = static_cast<int>(row_start[r + 1] - b);
    const int g0 = work[2 * blockIdx.x + 1] * kMergeTile;
    const std::uint64_t* src = ((pass & 1) ? scratch : sorted) + b;
    std::uint64_t* dst = ((pass & 1) ? sorted : scratch) + b;
    const int a0 = g0 / (2 * width) * (2 * width);  // kMergeTile divides 2 width
    const int na = min(width, len - a0);
    const int nb = min(width, max(0, len - a0 - width));
    const std::uint64_t* A = src + a0;
    const std::uint64_t* B = A + na;
    const int d0 = g0 - a0, d1 = min(d0 + kMergeTile, na + nb);
    if (threadIdx.x < 2) split[threadIdx.x] = merge_split(A, na, B, nb, threadIdx.x ? d1 : d0);
    __syncthreads();
    const int i0 = split[0], i1 = split[1];
    cta_merge(A + i0, i1 - i0, B + (d0 - i0), (d1 - i1) - (d0 - i0), dst + a0 + d0);
}
__global__ void __launch_bounds__(256) k_huge_finish(std::uint64_t* __restrict__ sorted,
                                                     const std::uint64_t* __restrict__ scratch,
                                                     const std::int64_t* __restrict__ row_start,
                                                     const std::int32_t* __restrict__ work,
                                                     std::int32_t* __restrict__ uniq_cnt) {
    __shared__ int red[8];
    const std::int32_t r = work[2 * blockIdx.x];
    const std::int64_t b = row_start[r];
    const int len = static_cast<int>(row_start[r + 1] - b);
    const int g0 = work[2 * blockIdx.x + 1] * kMergeTile;
    const int g1 = min(g0 + kMergeTile, len);
    const bool odd = huge_passes(len) & 1;
    const std::uint64_t* fin = (odd ? scratch : sorted) + b;
    int h = 0;
    for (int i = g0 + static_cast<int>(threadIdx.x); i < g1; i += blockDim.x) {
        const std::uint64_t v = fin[i];
        h += (i == 0 || (v >> 32) != (fin[i - 1] >> 32)) ? 1 : 0;
        if (odd) sorted[b + i] = v;
    }
    for (int o = 16; o > 0; o >>= 1) h += __shfl_xor_sync(0xffffffffu, h, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = h;
    __syncthreads();
    if (threadIdx.x == 0) {
        int t = 0;
        for (int i = 0; i < (blockDim.x >> 5); ++i) t += red[i];
        atomicAdd(&uniq_cnt[r], t);
    }
}

// 4. one warp per row, windows of 32 sorted entries. The warp first gathers
//    the window's 32 blocks into its shared tile cooperatively: load k of
//    lane L fetches double 32 k + L of the window's 288 (entry (32 k + L) / 9,
//    element (32 k + L) % 9), so each instruction reads ~4 whole 72-byte
//    records instead of one double of 32 scattered records. Then each run's
//    owner folds it SEQUENTIALLY in emission order (bitwise the reference's
//    deterministic left-to-right sum, reduction.hpp:39-53); a run crossing the
//    window boundary carries its partial sum (and output slot) to lane 0 of
//    the next window. Writes the unique blocks into the tiled block storage
//    (blk(), common.cuh).
constexpr int kReduceWarps = 8;

// window gather: load k of lane L fetches double 32 k + L of the window's 288
__device__ __forceinline__ void gather_window(const StreamSrc& s, std::uint32_t src, int nv, int lane, double (&g)[9]) {
#pragma unroll
    for (int k = 0; k < 9; ++k) {
        const int word = 32 * k + lane;
        const int j = word / 9, el = word - 9 * j;
        const std::uint32_t q = __shfl_sync(0xffffffffu, src, j);
        const double* sv = j < nv ? s.value(q) : nullptr;
        g[k] = sv ? __ldg(sv + el) : ((el & 3) == 0 ? 1.0 : 0.0);
    }
}

// One warp reduces the sorted entries [b, e) of row r — complete runs, the
// first entry a run head — into output slots from u on: windows of 32
// entries, every lane gathers its entry's block into the warp's shared tile,
// each run's owner sums it sequentially in emission order (a run crossing a
// window carries its partial sum to the next window).
__device__ __forceinline__ void reduce_range(const std::uint64_t* __restrict__ sorted, std::int32_t r, std::int64_t b,
                                             std::int64_t e, std::int64_t u, const StreamSrc& s,
                                             std::uint32_t* __restrict__ out_rows,
                                             std::uint32_t* __restrict__ out_cols, double* __restrict__ out_blocks,
                                             double (*Tl)[33], double* C, int lane) {
    bool carried = false;       // a run continues into this window (warp-uniform)
    std::int64_t carry_u = 0;   // its output slot
    // the carried partial sums, two slots by window parity: lane 0 reads the
    // incoming one while the owner of the window's last run may already
    // write the outgoing one (no lane order inside a window)
    int par = 0;
    for (std::int64_t base = b; base < e; base += 32, par ^= 1) {
        const double* Cin = C + 9 * par;
        double* Cout = C + 9 * (par ^ 1);
        const std::int64_t p = base + lane;
        const bool valid = p < e;
        const std::uint64_t v = valid ? sorted[p] : ~0ull;
        const std::uint32_t col = static_cast<std::uint32_t>(v >> 32);
        const std::uint32_t prev_col = __shfl_up_sync(0xffffffffu, col, 1);
        const bool head = valid && (lane == 0 ? (p == b || static_cast<std::uint32_t>(sorted[p - 1] >> 32) != col)
                                              : prev_col != col);
        const int nv = static_cast<int>(e - base < 32 ? e - base : 32);
        double g[9];
        gather_window(s, static_cast<std::uint32_t>(v), nv, lane, g);
#pragma unroll
        for (int k = 0; k < 9; ++k) {
            const int word = 32 * k + lane;
            const int j = word / 9, el = word - 9 * j;
            if (j < nv) Tl[el][j] = g[k];
        }
        // does the window's last run continue past it?
        const std::int64_t nxt = base + 32;
        const bool cont_out = __shfl_sync(0xffffffffu, nxt < e && lane == 31 &&
                                                           static_cast<std::uint32_t>(sorted[nxt] >> 32) == col,
                                          31);
        const unsigned hm = __ballot_sync(0xffffffffu, head);
        __syncwarp();
        const bool owner = head || (lane == 0 && carried);
        if (owner) {
            // run [lane, end): up to the next head of the window or its valid end
            const unsigned later = hm & ~((2u << lane) - 1u);
            const int end = later ? __ffs(later) - 1 : nv;
            double acc[9];
            if (head) {
#pragma unroll
                for (int k = 0; k < 9; ++k) acc[k] = Tl[k][lane];
            } else {  // continuing run: carried sum, then this window's entries
#pragma unroll
                for (int k = 0; k < 9; ++k) acc[k] = __dadd_rn(Cin[k], Tl[k][lane]);
            }
            for (int j = lane + 1; j < end; ++j)
#pragma unroll
                for (int k = 0; k < 9; ++k) acc[k] = __dadd_rn(acc[k], Tl[k][j]);
            const std::int64_t my_u = head ? u + __popc(hm & ((1u << lane) - 1u)) : carry_u;
            if (end == nv && cont_out) {  // hand over to the next window
#pragma unroll
                for (int k = 0; k < 9; ++k) Cout[k] = acc[k];
            } else {
                out_rows[my_u] = static_cast<std::uint32_t>(r);
                out_cols[my_u] = col;
#pragma unroll
                for (int k = 0; k < 9; ++k) out_blocks[blk(my_u, k)] = acc[k];
            }
        }
        // the continuing run's slot: the last head's, or the one already carried
        if (cont_out) carry_u = hm ? u + __popc(hm) - 1 : carry_u;
        carried = cont_out;
        u += __popc(hm);
        __syncwarp();
    }
}

__global__ void __launch_bounds__(32 * kReduceWarps, 3) k_reduce_rows(
    const std::uint64_t* __restrict__ sorted, const std::int64_t* __restrict__ row_start,
    const std::int64_t* __restrict__ uniq_start, std::int32_t n, StreamSrc s, std::uint32_t* __restrict__ out_rows,
    std::uint32_t* __restrict__ out_cols, double* __restrict__ out_blocks, std::int64_t max_len) {
    __shared__ double tile[kReduceWarps][9][33];
    __shared__ double carry[kReduceWarps][18];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int warps = gridDim.x * (blockDim.x >> 5);
    for (std::int32_t r = blockIdx.x * (blockDim.x >> 5) + w; r < n; r += warps)
        if (row_start[r + 1] - row_start[r] <= max_len)  // longer rows: k_reduce_segments
        reduce_range(sorted, r, row_start[r], row_start[r + 1], uniq_start[r], s, out_rows, out_cols, out_blocks,
                     tile[w], carry[w], lane);
}

// ---- long rows (contact scenes: affine-body rows with tens of thousands of
// entries): rows are cut into segments of about kSegLen entries at run
// heads, so one warp per SEGMENT reduces them; the runs stay whole and each
// is still summed left to right (bitwise the per-row path).
constexpr std::int64_t kSegLen = 1024;
// rows longer than this go through the segments; the others stay with
// k_reduce_rows (one warp per row) in the same assembly
constexpr std::int64_t kLongRow = 4 * kSegLen;

__global__ void k_seg_count(const std::int64_t* __restrict__ row_start, std::int32_t n, std::int32_t* __restrict__ cnt) {
    for (std::int64_t r = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; r < n;
         r += static_cast<std::int64_t>(gridDim.x) * blockDim.x)
    {
        const std::int64_t len = row_start[r + 1] - row_start[r];
        cnt[r] = len > kLongRow ? static_cast<std::int32_t>(ceil_div(len, kSegLen)) : 0;
    }
}
__global__ void k_seg_rows(const std::int64_t* __restrict__ item_ptr, std::int32_t n, std::int32_t* __restrict__ item_row) {
    for (std::int64_t r = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; r < n;
         r += static_cast<std::int64_t>(gridDim.x) * blockDim.x)
        for (std::int64_t i = item_ptr[r]; i < item_ptr[r + 1]; ++i) item_row[i] = static_cast<std::int32_t>(r);
}
// first run head at or after p in [b, e) (e if none); warp-cooperative
__device__ __forceinline__ std::int64_t next_head(const std::uint64_t* __restrict__ sorted, std::int64_t b,
                                                  std::int64_t e, std::int64_t p, int lane) {
    if (p <= b) return b;
    for (std::int64_t q0 = p; q0 < e; q0 += 32) {
        const std::int64_t q = q0 + lane;
        const bool h = q < e && static_cast<std::uint32_t>(sorted[q] >> 32) != static_cast<std::uint32_t>(sorted[q - 1] >> 32);
        const unsigned m = __ballot_sync(0xffffffffu, h);
        if (m) return q0 + __ffs(m) - 1;
    }
    return e;
}
// segment bounds and head counts, one warp per segment
__global__ void k_seg_heads(const std::uint64_t* __restrict__ sorted, const std::int64_t* __restrict__ row_start,
                            const std::int64_t* __restrict__ item_ptr, const std::int32_t* __restrict__ item_row,
                            std::int64_t m, std::int64_t* __restrict__ seg, std::int32_t* __restrict__ heads) {
    const int lane = threadIdx.x & 31;
    for (std::int64_t i = (blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x) >> 5; i < m;
         i += (static_cast<std::int64_t>(gridDim.x) * blockDim.x) >> 5) {
        const std::int32_t r = item_row[i];
        const std::int64_t b = row_start[r], e = row_start[r + 1], k = i - item_ptr[r];
        const std::int64_t s0 = next_head(sorted, b, e, b + k * kSegLen, lane);
        const std::int64_t s1 = next_head(sorted, b, e, std::min(e, b + (k + 1) * kSegLen), lane);
        int h = 0;
        for (std::int64_t q0 = s0; q0 < s1; q0 += 32) {
            const std::int64_t q = q0 + lane;
            const bool hd = q < s1 && (q == b || static_cast<std::uint32_t>(sorted[q] >> 32) !=
                                                     static_cast<std::uint32_t>(sorted[q - 1] >> 32));
            h += __popc(__ballot_sync(0xffffffffu, hd));
        }
        if (lane == 0) {
            seg[2 * i] = s0;
            seg[2 * i + 1] = s1;
            heads[i] = h;
        }
    }
}
// 8-byte asynchronous global -> shared copy (LDGSTS) and its group fences
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(static_cast<std::uint32_t>(__cvta_generic_to_shared(dst))),
                 "l"(src)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// reduce_range for long segments (affine-body rows: runs of tens of
// thousands of entries, one sequential chain each): the same windows and the
// same left-to-right run sums, but the window's keys are fetched kKeyAhead
// windows ahead and its 288 value words kValAhead windows ahead by
// asynchronous copies into per-warp shared rings, so a long run's chain no
// longer waits two dependent global round trips (key, then value) per window.
// Every iteration commits exactly one cp.async group: the keys of window
// w + kKeyAhead and the values of window w + kValAhead.
constexpr int kValAhead = 3, kKeyAhead = 6;
constexpr int kSegWarps = 4;
struct SegRing {
    double v[kValAhead][9][33];
    std::uint64_t k[kKeyAhead][32];
    double carry[2][9];  // by window parity (see reduce_range)
};
__device__ __forceinline__ void reduce_range_pipe(const std::uint64_t* __restrict__ sorted, std::int32_t r,
                                                  std::int64_t b, std::int64_t e, std::int64_t u, const StreamSrc& s,
                                                  std::uint32_t* __restrict__ out_rows,
                                                  std::uint32_t* __restrict__ out_cols,
                                                  double* __restrict__ out_blocks, SegRing& R, int lane) {
    const std::int64_t nwin = (e - b + 31) >> 5;
    auto issue_keys = [&](std::int64_t w) {
        if (w >= nwin) return;
        const std::int64_t p = b + 32 * w + lane;
        std::uint64_t* d = &R.k[w % kKeyAhead][lane];
        if (p < e)
            cp_async8(d, sorted + p);
        else
            *d = ~0ull;
    };
    auto issue_vals = [&](std::int64_t w) {  // keys of w have landed (and are visible to the warp)
        if (w >= nwin) return;
        const std::int64_t base = b + 32 * w;
        const int nv = static_cast<int>(e - base < 32 ? e - base : 32);
        double (*T)[33] = R.v[w % kValAhead];
        const std::uint64_t* kw = R.k[w % kKeyAhead];
#pragma unroll
        for (int k = 0; k < 9; ++k) {
            const int word = 32 * k + lane;
            const int j = word / 9, el = word - 9 * j;
            if (j < nv) {
                const double* sv = s.value(static_cast<std::uint32_t>(kw[j]));
                if (sv)
                    cp_async8(&T[el][j], sv + el);
                else
                    T[el][j] = (el & 3) == 0 ? 1.0 : 0.0;  // appended pinned-diagonal identity
            }
        }
    };
    // prologue: the keys of the first kKeyAhead windows (waited for), then
    // kValAhead groups P_j = {values of window j}. With the loop's groups
    // I_w = {values of w + kValAhead, keys of w + kKeyAhead}, the group
    // sequence P_0.., I_0.. has the values of window w at position w and the
    // keys of window w + kValAhead (kKeyAhead = 2 kValAhead) at position w
    // or in the prologue, so waiting for all but the newest kValAhead - 1
    // groups at the top of iteration w covers both.
    for (int w = 0; w < kKeyAhead; ++w) issue_keys(w);
    cp_async_commit();
    cp_async_wait<0>();
    __syncwarp();
    for (int j = 0; j < kValAhead; ++j) {
        issue_vals(j);
        cp_async_commit();
    }
    bool carried = false;
    std::int64_t carry_u = 0;
    std::uint32_t prev_last = 0;  // column of the previous window's last entry
    for (std::int64_t w = 0; w < nwin; ++w) {
        cp_async_wait<kValAhead - 1>();
        __syncwarp();
        const std::int64_t base = b + 32 * w;
        const int nv = static_cast<int>(e - base < 32 ? e - base : 32);
        double (*Tl)[33] = R.v[w % kValAhead];
        const std::uint64_t v = R.k[w % kKeyAhead][lane];
        const bool valid = lane < nv;
        const std::uint32_t col = static_cast<std::uint32_t>(v >> 32);
        const std::uint32_t prev_col = __shfl_up_sync(0xffffffffu, col, 1);
        const bool head = valid && (lane == 0 ? (w == 0 || prev_last != col) : prev_col != col);
        // does the window's last run continue past it?
        const bool cont_out = __shfl_sync(0xffffffffu,
                                          w + 1 < nwin && lane == 31 &&
                                              static_cast<std::uint32_t>(R.k[(w + 1) % kKeyAhead][0] >> 32) == col,
                                          31);
        prev_last = __shfl_sync(0xffffffffu, col, 31);
        const unsigned hm = __ballot_sync(0xffffffffu, head);
        if (hm <= 1u) {
            // one run fills the window (the body of a long run): lane k < 9
            // folds element k of the run's blocks, the nine chains in
            // parallel instead of interleaved in one owner thread (same
            // left-to-right order per element)
            const std::int64_t my_u = hm ? u : carry_u;
            if (lane < 9) {
                double acc = hm ? Tl[lane][0] : __dadd_rn(R.carry[w & 1][lane], Tl[lane][0]);
#pragma unroll 8
                for (int j = 1; j < nv; ++j) acc = __dadd_rn(acc, Tl[lane][j]);
                if (cont_out)
                    R.carry[(w & 1) ^ 1][lane] = acc;
                else
                    out_blocks[blk(my_u, lane)] = acc;
            }
            if (lane == 0 && !cont_out) {
                out_rows[my_u] = static_cast<std::uint32_t>(r);
                out_cols[my_u] = col;
            }
            if (cont_out) carry_u = my_u;
            carried = cont_out;
            u += __popc(hm);
            __syncwarp();
            issue_vals(w + kValAhead);
            issue_keys(w + kKeyAhead);
            cp_async_commit();
            continue;
        }
        const bool owner = head || (lane == 0 && carried);
        if (owner) {
            const unsigned later = hm & ~((2u << lane) - 1u);
            const int end = later ? __ffs(later) - 1 : nv;
            double acc[9];
            if (head) {
#pragma unroll
                for (int k = 0; k < 9; ++k) acc[k] = Tl[k][lane];
            } else {
#pragma unroll
                for (int k = 0; k < 9; ++k) acc[k] = __dadd_rn(R.carry[w & 1][k], Tl[k][lane]);
            }
            for (int j = lane + 1; j < end; ++j)
#pragma unroll
                for (int k = 0; k < 9; ++k) acc[k] = __dadd_rn(acc[k], Tl[k][j]);
            const std::int64_t my_u = head ? u + __popc(hm & ((1u << lane) - 1u)) : carry_u;
            if (end == nv && cont_out) {
#pragma unroll
                for (int k = 0; k < 9; ++k) R.carry[(w & 1) ^ 1][k] = acc[k];
            } else {
                out_rows[my_u] = static_cast<std::uint32_t>(r);
                out_cols[my_u] = col;
#pragma unroll
                for (int k = 0; k < 9; ++k) out_blocks[blk(my_u, k)] = acc[k];
            }
        }
        if (cont_out) carry_u = hm ? u + __popc(hm) - 1 : carry_u;
        carried = cont_out;
        u += __popc(hm);
        __syncwarp();  // slot w % kValAhead and key slot w % kKeyAhead are free again
        issue_vals(w + kValAhead);
        issue_keys(w + kKeyAhead);
        cp_async_commit();
    }
    cp_async_wait<0>();
    __syncwarp();
}

__global__ void __launch_bounds__(32 * kSegWarps) k_reduce_segments(
    const std::uint64_t* __restrict__ sorted, const std::int32_t* __restrict__ item_row,
    const std::int64_t* __restrict__ seg, const std::int64_t* __restrict__ item_u,
    const std::int64_t* __restrict__ item_ptr, const std::int64_t* __restrict__ uniq_start, std::int64_t m,
    StreamSrc s, std::uint32_t* __restrict__ out_rows, std::uint32_t* __restrict__ out_cols,
    double* __restrict__ out_blocks) {
    extern __shared__ __align__(16) unsigned char seg_smem[];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    SegRing& R = reinterpret_cast<SegRing*>(seg_smem)[w];
    const std::int64_t warps = static_cast<std::int64_t>(gridDim.x) * (blockDim.x >> 5);
    for (std::int64_t i = static_cast<std::int64_t>(blockIdx.x) * (blockDim.x >> 5) + w; i < m; i += warps)
    {
        // item_u: heads scanned over the long rows' segments only; the row's
        // output slots start at uniq_start[r]
        const std::int32_t r = item_row[i];
        const std::int64_t u = uniq_start[r] + item_u[i] - item_u[item_ptr[r]];
        reduce_range_pipe(sorted, r, seg[2 * i], seg[2 * i + 1], u, s, out_rows, out_cols, out_blocks, R, lane);
    }
}

__global__ void k_max_row(const std::uint64_t* __restrict__ keys, std::int64_t T, unsigned* __restrict__ out) {
    unsigned m = 0;
    for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < T;
         i += static_cast<std::int64_t>(gridDim.x) * blockDim.x)
        m = max(m, static_cast<unsigned>(keys[i] >> 32));
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

// sorted (col << 32 | index) per row -> sorted keys + gathered values
__global__ void k_gather_sorted(const std::uint64_t* __restrict__ sorted, const std::int64_t* __restrict__ row_start,
                                std::int32_t n, const double* __restrict__ vals, std::uint64_t* __restrict__ out_keys,
                                double* __restrict__ out_vals) {
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int warps = gridDim.x * (blockDim.x >> 5);
    for (std::int32_t r = blockIdx.x * (blockDim.x >> 5) + w; r < n; r += warps)
        for (std::int64_t p = row_start[r] + lane; p < row_start[r + 1]; p += 32) {
            const std::uint64_t v = sorted[p];
            out_keys[p] = (static_cast<std::uint64_t>(r) << 32) | (v >> 32);
            const double* src = vals + 9 * static_cast<std::int64_t>(static_cast<std::uint32_t>(v));
            for (int k = 0; k < 9; ++k) out_vals[9 * p + k] = src[k];
        }
}

// AoS (9 doubles per block, the reference's Mat3 storage) <-> tiled storage
__global__ void k_aos_to_soa(const double* __restrict__ aos, double* __restrict__ soa, std::int64_t U) {
    for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < 9 * U;
         i += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        const std::int64_t u = i / 9;
        soa[blk(u, static_cast<int>(i - 9 * u))] = aos[i];
    }
}
__global__ void k_soa_to_aos(const double* __restrict__ soa, double* __restrict__ aos, std::int64_t U) {
    for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < 9 * U;
         i += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        const std::int64_t u = i / 9;
        aos[i] = soa[blk(u, static_cast<int>(i - 9 * u))];
    }
}

__global__ void k_count_rows(const std::uint32_t* __restrict__ rows, std::int64_t U, std::int32_t n,
                             std::int32_t* __restrict__ cnt) {
    for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < U;
         i += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        const std::uint32_t r = rows[i];
        if (r < static_cast<std::uint32_t>(n)) atomicAdd(cnt + r, 1);
    }
}

// fast_segment_reduction (reduction.hpp:30-79): one thread per run head sums
// its run left to right (deterministic-mode order) and stores the segment.
__global__ void k_segment_reduce(const std::int32_t* __restrict__ O, std::int64_t n, const double* __restrict__ V,
                                 int width, std::int32_t n_seg, double* __restrict__ R) {
    for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        const std::int32_t seg = O[i];
        if (i > 0 && O[i - 1] == seg) continue;
        if (seg < 0 || seg >= n_seg) continue;
        double acc[9];
        for (int k = 0; k < width; ++k) acc[k] = V[i * width + k];
        for (std::int64_t j = i + 1; j < n && O[j] == seg; ++j)
            for (int k = 0; k < width; ++k) acc[k] = __dadd_rn(acc[k], V[j * width + k]);
        for (int k = 0; k < width; ++k) R[static_cast<std::int64_t>(seg) * width + k] = acc[k];
    }
}

// filter_pinned (incremental_potential.hpp:410-425), step 1: keep flags.
__global__ void k_pin_keep(const std::uint64_t* __restrict__ keys, std::int64_t T, const std::uint8_t* __restrict__ pinned,
                           std::int32_t* __restrict__ keep) {
    for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < T;
         i += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        const std::uint32_t r = static_cast<std::uint32_t>(keys[i] >> 32);
        const std::uint32_t c = static_cast<std::uint32_t>(keys[i]);
        keep[i] = (pinned[r] || pinned[c]) ? 0 : 1;
    }
}

__global__ void k_pin_compact(const std::uint64_t* __restrict__ keys, const double* __restrict__ vals, std::int64_t T,
                              const std::int32_t* __restrict__ keep, const std::int64_t* __restrict__ pos,
                              std::uint64_t* __restrict__ ok, double* __restrict__ ov) {
    for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < T;
         i += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        if (!keep[i]) continue;
        const std::int64_t p = pos[i];
        ok[p] = keys[i];
        for (int k = 0; k < 9; ++k) ov[9 * p + k] = vals[9 * i + k];
    }
}

__global__ void k_pin_identity(const std::uint8_t* __restrict__ pinned, std::int32_t n_slots,
                               const std::int64_t* __restrict__ pos, std::int64_t base, std::uint64_t* __restrict__ ok,
                               double* __restrict__ ov) {
    for (std::int64_t s = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; s < n_slots;
         s += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        if (!pinned[s]) continue;
        const std::int64_t p = base + pos[s];
        ok[p] = (static_cast<std::uint64_t>(s) << 32) | static_cast<std::uint64_t>(s);
        for (int k = 0; k < 9; ++k) ov[9 * p + k] = (k % 4 == 0) ? 1.0 : 0.0;
    }
}



__global__ void k_u8_to_i32(const std::uint8_t* __restrict__ a, std::int64_t n, std::int32_t* __restrict__ b) {
    for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<std::int64_t>(gridDim.x) * blockDim.x)
        b[i] = a[i] ? 1 : 0;
}

}  // namespace

// Steps 1-3: bucket by row, sort each row by (col, emission index), count
// unique cols. Leaves c.sorted / c.row_start / c.uniq_cnt filled. Throws
// kInvalidArgument if a key's row is >= n.
static void bucket_sort(Ctx& c, const StreamSrc& s, std::int32_t n) {
    cudaStream_t st = c.stream;
    const std::int64_t T = s.T1 + s.T2;
    const std::int64_t entries = T + (s.pinned ? s.n_pin : 0);
    if (entries >= (std::int64_t(1) << 32) - 1) throw StatusError(kInvalidArgument, "triplet stream longer than 2^32");
    c.row_cnt.reserve(static_cast<std::size_t>(n) + 1);
    c.row_cursor.reserve(static_cast<std::size_t>(n) + 1);
    c.uniq_cnt.reserve(static_cast<std::size_t>(n) + 1);
    c.big_rows.reserve(static_cast<std::size_t>(n) + 1);
    c.row_start.reserve(static_cast<std::size_t>(n) + 1);
    c.counters.reserve(4);
    c.sorted.reserve(static_cast<std::size_t>(std::max<std::int64_t>(entries, 1)));
    ADIPC_CUDA(cudaMemsetAsync(c.row_cnt.p, 0, sizeof(std::int32_t) * (n + 1), st));
    ADIPC_CUDA(cudaMemsetAsync(c.row_cursor.p, 0, sizeof(std::int32_t) * (n + 1), st));
    ADIPC_CUDA(cudaMemsetAsync(c.counters.p, 0, sizeof(std::int32_t) * 4, st));
    if (entries > 0) {
        k_row_hist<<<grid_for(ceil_div(entries, kIlp), 256, 16), 256, 0, st>>>(s, n, c.row_cnt.p, c.counters.p);
        ADIPC_LAUNCH_CHECK();
    }
    exclusive_scan(c.row_cnt.p, n, c.row_start.p, c.scan_scratch, st);
    if (entries > 0) {
        k_row_scatter<<<grid_for(ceil_div(entries, kIlp), 256, 16), 256, 0, st>>>(s, n, c.row_start.p, c.row_cursor.p,
                                                                                   c.sorted.p);
        ADIPC_LAUNCH_CHECK();
    }
    if (n > 0) {
        k_sort_rows_warp<<<grid_for(n, 8, 16), 256, 0, st>>>(c.sorted.p, c.row_start.p, n, c.uniq_cnt.p, c.big_rows.p,
                                                             c.counters.p + 1);
        ADIPC_LAUNCH_CHECK();
    }
    int h_counters[4] = {0, 0, 0, 0};
    ADIPC_CUDA(cudaMemcpyAsync(h_counters, c.counters.p, sizeof(h_counters), cudaMemcpyDeviceToHost, st));
    ADIPC_CUDA(cudaStreamSynchronize(st));
    if (h_counters[0])
        throw StatusError(kInvalidArgument, "block row index >= n_block_rows in triplet stream");
    c.sort_long_rows = h_counters[1] + h_counters[2];
    if (h_counters[2] > 0) {  // rows > kHugeRow: chunk sorts + merge passes over the whole GPU
        const int nh = h_counters[2], maxlen = h_counters[3];
        c.merge_scratch.reserve(static_cast<std::size_t>(entries));
        c.huge_info.reserve(2 * static_cast<std::size_t>(nh));
        k_huge_info<<<ceil_div(nh, 256), 256, 0, st>>>(c.big_rows.p + n, c.row_start.p, nh, c.huge_info.p);
        ADIPC_LAUNCH_CHECK();
        std::vector<std::int32_t> info(2 * static_cast<std::size_t>(nh));
        ADIPC_CUDA(cudaMemcpyAsync(info.data(), c.huge_info.p, info.size() * sizeof(std::int32_t),
                                   cudaMemcpyDeviceToHost, st));
        ADIPC_CUDA(cudaStreamSynchronize(st));
        // work lists: chunks, then each merge pass's tiles, then the finish tiles
        std::vector<std::int32_t> work;
        std::vector<std::size_t> start;  // offset (in items) of each list
        auto list = [&](int unit, int min_len) {
            start.push_back(work.size() / 2);
            for (int y = 0; y < nh; ++y)
                if (info[2 * y + 1] > min_len)
                    for (int x = 0; x < ceil_div(info[2 * y + 1], unit); ++x) {
                        work.push_back(info[2 * y]);
                        work.push_back(x);
                    }
        };
        list(kCtaSortMax, 0);
        int passes = 0;
        for (int width = kCtaSortMax; width < maxlen; width <<= 1, ++passes) list(kMergeTile, width);
        list(kMergeTile, 0);
        start.push_back(work.size() / 2);
        c.huge_work.reserve(work.size());
        ADIPC_CUDA(cudaMemcpyAsync(c.huge_work.p, work.data(), work.size() * sizeof(std::int32_t),
                                   cudaMemcpyHostToDevice, st));
        auto items = [&](int i) { return static_cast<unsigned>(start[i + 1] - start[i]); };
        auto at = [&](int i) { return c.huge_work.p + 2 * start[i]; };
        const int smem = kCtaSortMax * sizeof(std::uint64_t);
        ADIPC_CUDA(cudaFuncSetAttribute(k_huge_chunks, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        k_huge_chunks<<<items(0), kCtaSortThreads, smem, st>>>(c.sorted.p, c.row_start.p, at(0), c.uniq_cnt.p);
        ADIPC_LAUNCH_CHECK();
        for (int pass = 0, width = kCtaSortMax; pass < passes; ++pass, width <<= 1) {
            k_huge_merge<<<items(1 + pass), 256, 0, st>>>(c.sorted.p, c.merge_scratch.p, c.row_start.p, at(1 + pass),
                                                          width, pass);
            ADIPC_LAUNCH_CHECK();
        }
        k_huge_finish<<<items(1 + passes), 256, 0, st>>>(c.sorted.p, c.merge_scratch.p, c.row_start.p,
                                                         at(1 + passes), c.uniq_cnt.p);
        ADIPC_LAUNCH_CHECK();
        // the host vector must outlive the upload
        ADIPC_CUDA(cudaStreamSynchronize(st));
    }
    if (h_counters[1] > 0) {
        const int nb = h_counters[1];
        c.merge_scratch.reserve(static_cast<std::size_t>(entries));
        const int smem = kCtaSortMax * sizeof(std::uint64_t);
        ADIPC_CUDA(cudaFuncSetAttribute(k_sort_rows_cta, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        k_sort_rows_cta<<<std::min(nb, kSMs * 2), kCtaSortThreads, smem, st>>>(
            c.sorted.p, c.merge_scratch.p, c.row_start.p, c.big_rows.p, c.counters.p + 1, c.uniq_cnt.p);
        ADIPC_LAUNCH_CHECK();
    }
}

static StreamSrc plain_src(const std::uint64_t* k, const double* v, std::int64_t T) {
    return StreamSrc{k, v, T, nullptr, nullptr, 0, nullptr, 0, nullptr};
}

void bucket_sort(Ctx& c, const std::uint64_t* d_keys, std::int64_t T, std::int32_t n, const std::uint32_t* d_vidx) {
    StreamSrc s = plain_src(d_keys, nullptr, T);
    s.vidx = d_vidx;
    bucket_sort(c, s, n);
}

void blocks_aos_to_soa(Ctx& c, const double* aos, double* soa, std::int64_t U) {
    if (U == 0) return;
    k_aos_to_soa<<<grid_for(9 * U, 256, 16), 256, 0, c.stream>>>(aos, soa, U);
    ADIPC_LAUNCH_CHECK();
}
void blocks_soa_to_aos(Ctx& c, const double* soa, double* aos, std::int64_t U) {
    if (U == 0) return;
    k_soa_to_aos<<<grid_for(9 * U, 256, 16), 256, 0, c.stream>>>(soa, aos, U);
    ADIPC_LAUNCH_CHECK();
}

// Sort + reduce of a device-resident triplet stream into `out` (CSR row_ptr
// included). Shared by the global assembly, the solve-order matrix and the
// two-level ABD reduction.
static void sort_reduce(Ctx& c, const StreamSrc& s, std::int32_t n, DeviceMatrix& out, cudaEvent_t vals_ready) {
    cudaStream_t st = c.stream;
    bucket_sort(c, s, n);  // keys only: overlaps an upload of the values still in flight
    if (vals_ready) ADIPC_CUDA(cudaStreamWaitEvent(st, vals_ready, 0));
    out.n = n;
    out.row_ptr.reserve(static_cast<std::size_t>(n) + 1);
    exclusive_scan(c.uniq_cnt.p, n, out.row_ptr.p, c.scan_scratch, st);
    std::int64_t U = 0;
    ADIPC_CUDA(cudaMemcpyAsync(&U, out.row_ptr.p + n, sizeof(U), cudaMemcpyDeviceToHost, st));
    ADIPC_CUDA(cudaStreamSynchronize(st));
    out.U = U;
    // whole 32-block tiles (the SpMV reads rows/cols per tile)
    out.rows.reserve(static_cast<std::size_t>((U + 31) & ~std::int64_t(31)));
    out.cols.reserve(static_cast<std::size_t>((U + 31) & ~std::int64_t(31)));
    out.blocks.reserve(blk_doubles(U));
    if (n > 0 && U > 0) {
        k_reduce_rows<<<grid_for(n, 8, 16), 256, 0, st>>>(c.sorted.p, c.row_start.p, out.row_ptr.p, n, s, out.rows.p,
                                                          out.cols.p, out.blocks.p,
                                                          c.sort_long_rows ? kLongRow : INT64_MAX);
        ADIPC_LAUNCH_CHECK();
    }
    if (n > 0 && U > 0 && c.sort_long_rows) {  // rows > kLongRow: one warp per ~kSegLen-entry segment
        c.seg_cnt.reserve(static_cast<std::size_t>(n) + 1);
        c.seg_ptr.reserve(static_cast<std::size_t>(n) + 1);
        k_seg_count<<<grid_for(n, 256, 16), 256, 0, st>>>(c.row_start.p, n, c.seg_cnt.p);
        ADIPC_LAUNCH_CHECK();
        exclusive_scan(c.seg_cnt.p, n, c.seg_ptr.p, c.scan_scratch, st);
        std::int64_t m = 0;
        ADIPC_CUDA(cudaMemcpyAsync(&m, c.seg_ptr.p + n, sizeof(m), cudaMemcpyDeviceToHost, st));
        ADIPC_CUDA(cudaStreamSynchronize(st));
        if (m == 0) {  // no row beyond kLongRow: k_reduce_rows did them all
            ++out.version;
            return;
        }
        c.seg_row.reserve(static_cast<std::size_t>(std::max<std::int64_t>(m, 1)));
        c.seg_heads.reserve(static_cast<std::size_t>(std::max<std::int64_t>(m, 1)));
        c.seg_bounds.reserve(static_cast<std::size_t>(std::max<std::int64_t>(2 * m, 1)));
        c.seg_u.reserve(static_cast<std::size_t>(m) + 1);
        k_seg_rows<<<grid_for(n, 256, 16), 256, 0, st>>>(c.seg_ptr.p, n, c.seg_row.p);
        ADIPC_LAUNCH_CHECK();
        k_seg_heads<<<grid_for(m, 8, 16), 256, 0, st>>>(c.sorted.p, c.row_start.p, c.seg_ptr.p, c.seg_row.p, m,
                                                        c.seg_bounds.p, c.seg_heads.p);
        ADIPC_LAUNCH_CHECK();
        exclusive_scan(c.seg_heads.p, m, c.seg_u.p, c.scan_scratch, st);
        static_assert(kSegWarps * sizeof(SegRing) <= 48 * 1024, "k_reduce_segments ring exceeds the default smem");
        k_reduce_segments<<<grid_for(m, kSegWarps, 16), 32 * kSegWarps, kSegWarps * sizeof(SegRing), st>>>(
            c.sorted.p, c.seg_row.p, c.seg_bounds.p, c.seg_u.p, c.seg_ptr.p, out.row_ptr.p, m, s, out.rows.p,
            out.cols.p, out.blocks.p);
        ADIPC_LAUNCH_CHECK();
    }
    ++out.version;
}

void sort_reduce(Ctx& c, const std::uint64_t* d_keys, const double* d_vals, std::int64_t T, std::int32_t n,
                 DeviceMatrix& out, cudaEvent_t vals_ready) {
    sort_reduce(c, plain_src(d_keys, d_vals, T), n, out, vals_ready);
}

// sort_stream drop-in (block_coo.hpp:106-113): stable sort of the stream by
// key, values following. Rows must be < 2^30 (block coordinates).
void sort_stream(Ctx& c, const std::uint64_t* d_keys, const double* d_vals, std::int64_t T, std::uint64_t* d_out_keys,
                 double* d_out_vals) {
    cudaStream_t st = c.stream;
    if (T == 0) return;
    c.counters.reserve(4);
    ADIPC_CUDA(cudaMemsetAsync(c.counters.p, 0, sizeof(std::int32_t) * 4, st));
    k_max_row<<<grid_for(T, 256, 16), 256, 0, st>>>(d_keys, T, reinterpret_cast<unsigned*>(c.counters.p + 2));
    ADIPC_LAUNCH_CHECK();
    unsigned max_row = 0;
    ADIPC_CUDA(cudaMemcpyAsync(&max_row, c.counters.p + 2, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
    ADIPC_CUDA(cudaStreamSynchronize(st));
    if (max_row >= (1u << 30)) throw StatusError(kInvalidArgument, "sort_stream: block row index >= 2^30");
    const std::int32_t n = static_cast<std::int32_t>(max_row) + 1;
    bucket_sort(c, d_keys, T, n, nullptr);
    k_gather_sorted<<<grid_for(n, 8, 16), 256, 0, st>>>(c.sorted.p, c.row_start.p, n, d_vals, d_out_keys, d_out_vals);
    ADIPC_LAUNCH_CHECK();
}

void assemble(Ctx& c, const std::uint64_t* d_keys, const double* d_vals, std::int64_t T, std::int32_t n,
              int /*deterministic: the device path is always the bitwise-deterministic order*/, cudaEvent_t vals_ready) {
    sort_reduce(c, plain_src(d_keys, d_vals, T), n, c.A, vals_ready);
}

// filter_pinned + sort + reduce without moving a value: the pin filter runs
// inside the bucketing passes (dropped entries are never bucketed, the
// pinned-diagonal identities are bucketed with emission indices past the
// stream, incremental_potential.hpp:410-425), and the reduction reads each
// kept value from the ORIGINAL stream in the same emission order — bitwise
// the compacted-stream result. A second stream segment (the contact tiles
// two_level_abd_reduce appends, incremental_potential.hpp:392-394) may
// follow the first.
void assemble_filtered(Ctx& c, const std::uint64_t* d_keys, const double* d_vals, std::int64_t T, std::int32_t n,
                       const std::uint8_t* d_pinned, cudaEvent_t vals_ready, const std::uint64_t* d_keys2,
                       const double* d_vals2, std::int64_t T2) {
    const StreamSrc s{d_keys, d_vals, T, d_keys2, d_vals2, T2, d_pinned, n, nullptr};
    sort_reduce(c, s, n, c.A, vals_ready);
}

void upload_matrix(Ctx& c, std::int32_t n, std::int64_t U, const std::uint32_t* rows, const std::uint32_t* cols,
                   const double* blocks, bool host_ptrs) {
    DeviceMatrix& A = c.A;
    A.n = n;
    A.U = U;
    A.rows.reserve(static_cast<std::size_t>((U + 31) & ~std::int64_t(31)));
    A.cols.reserve(static_cast<std::size_t>((U + 31) & ~std::int64_t(31)));
    A.blocks.reserve(blk_doubles(U));
    A.row_ptr.reserve(static_cast<std::size_t>(n) + 1);
    const cudaMemcpyKind kind = host_ptrs ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
    if (U > 0) {
        ADIPC_CUDA(cudaMemcpyAsync(A.rows.p, rows, 4 * U, kind, c.stream));
        ADIPC_CUDA(cudaMemcpyAsync(A.cols.p, cols, 4 * U, kind, c.stream));
        c.vals.reserve(9 * U);  // AoS staging, then transposed into the tiled storage
        ADIPC_CUDA(cudaMemcpyAsync(c.vals.p, blocks, 72 * U, kind, c.stream));
        blocks_aos_to_soa(c, c.vals.p, A.blocks.p, U);
    }
    // row_ptr from the sorted rows: histogram + scan
    c.row_cnt.reserve(static_cast<std::size_t>(n) + 1);
    ADIPC_CUDA(cudaMemsetAsync(c.row_cnt.p, 0, 4 * (static_cast<std::size_t>(n) + 1), c.stream));
    if (U > 0) {
        k_count_rows<<<grid_for(U, 256, 16), 256, 0, c.stream>>>(A.rows.p, U, n, c.row_cnt.p);
        ADIPC_LAUNCH_CHECK();
    }
    exclusive_scan(c.row_cnt.p, n, A.row_ptr.p, c.scan_scratch, c.stream);
    ++A.version;
}

}  // namespace adipc_gpu

namespace adipc_gpu {

void segment_reduce(Ctx& c, const std::int32_t* d_O, std::int64_t n, const double* d_V, int width,
                    std::int32_t n_segments, double* d_R) {
    if (width != 1 && width != 3 && width != 9) throw StatusError(kInvalidArgument, "width must be 1, 3 or 9");
    if (n_segments > 0)
        ADIPC_CUDA(cudaMemsetAsync(d_R, 0, sizeof(double) * width * static_cast<std::size_t>(n_segments), c.stream));
    if (n > 0) {
        k_segment_reduce<<<grid_for(n, 256, 16), 256, 0, c.stream>>>(d_O, n, d_V, width, n_segments, d_R);
        ADIPC_LAUNCH_CHECK();
    }
}

std::int64_t filter_pinned(Ctx& c, const std::uint64_t* d_keys, const double* d_vals, std::int64_t T,
                           const std::uint8_t* d_pinned, std::int32_t n_slots, std::uint64_t* d_out_keys,
                           double* d_out_vals) {
    cudaStream_t st = c.stream;
    DBuf<std::int32_t>& keep = c.pin_keep;
    DBuf<std::int64_t>& pos = c.pin_pos;
    DBuf<std::int64_t>& spos = c.pin_spos;
    keep.reserve(static_cast<std::size_t>(std::max<std::int64_t>(T, n_slots)) + 1);
    pos.reserve(static_cast<std::size_t>(T) + 1);
    spos.reserve(static_cast<std::size_t>(n_slots) + 1);
    std::int64_t kept = 0, npin = 0;
    if (T > 0) {
        k_pin_keep<<<grid_for(T, 256, 16), 256, 0, st>>>(d_keys, T, d_pinned, keep.p);
        ADIPC_LAUNCH_CHECK();
    }
    exclusive_scan(keep.p, T, pos.p, c.scan_scratch, st);
    if (T > 0) {
        k_pin_compact<<<grid_for(T, 256, 16), 256, 0, st>>>(d_keys, d_vals, T, keep.p, pos.p, d_out_keys, d_out_vals);
        ADIPC_LAUNCH_CHECK();
    }
    ADIPC_CUDA(cudaMemcpyAsync(&kept, pos.p + T, sizeof(kept), cudaMemcpyDeviceToHost, st));
    ADIPC_CUDA(cudaStreamSynchronize(st));
    if (n_slots > 0) {
        k_u8_to_i32<<<grid_for(n_slots, 256, 16), 256, 0, st>>>(d_pinned, n_slots, keep.p);
        ADIPC_LAUNCH_CHECK();
    }
    exclusive_scan(keep.p, n_slots, spos.p, c.scan_scratch, st);
    if (n_slots > 0) {
        k_pin_identity<<<grid_for(n_slots, 256, 16), 256, 0, st>>>(d_pinned, n_slots, spos.p, kept, d_out_keys,
                                                                 d_out_vals);
        ADIPC_LAUNCH_CHECK();
    }
    ADIPC_CUDA(cudaMemcpyAsync(&npin, spos.p + n_slots, sizeof(npin), cudaMemcpyDeviceToHost, st));
    ADIPC_CUDA(cudaStreamSynchronize(st));
    return kept + npin;
}

}  // namespace adipc_gpu
