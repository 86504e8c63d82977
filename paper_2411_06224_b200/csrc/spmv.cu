// Symmetric reduce-by-key block SpMV (SRBK, paper Alg. 4; reference
// sparse/srbk_spmv.hpp:13-49): y = A x with A stored as its sorted upper block
// triangle. Each warp owns 32 consecutive blocks (the reference's lane group
// of width 32): lane e computes H_e x[col] and, off the diagonal, H_e^T x[row]
// (scattered with fp64 RED atomics to y[col]); the row contributions are
// summed with a head-segmented shuffle reduction over the warp's sorted rows
// and the run heads add them to y[row] atomically.
//
// Optional fusion for PCG: the same pass accumulates p.(A p) directly from the
// blocks, p_r.(H p_c) * (r != c ? 2 : 1), so the dot needs no second sweep
// over Ap; the grid total is finished by the last CTA (deterministic order).
#include <algorithm>

#include "mas_kernels.cuh"

namespace adipc_gpu {

namespace {

constexpr int kSpmvThreads = 256;
#ifndef ADIPC_SPMV_MIN_BLOCKS
#define ADIPC_SPMV_MIN_BLOCKS 3
#endif
constexpr int kSpmvMinBlocks = ADIPC_SPMV_MIN_BLOCKS;  // 3 x 256 threads (<= 85 registers, 24 warps/SM); 4 spills: 85 vs 61 us

template <bool kDot, bool kPad = false, bool kCoalesce = false>
__global__ void __launch_bounds__(kSpmvThreads, kSpmvMinBlocks) k_spmv(const std::uint32_t* __restrict__ rows,
                                                     const std::uint32_t* __restrict__ cols,
                                                     const double* __restrict__ blocks, std::int64_t U,
                                                     const double* __restrict__ x, double* __restrict__ y,
                                                     double* __restrict__ partials, unsigned* __restrict__ ticket,
                                                     double* __restrict__ dot_out, const int* __restrict__ flags,
                                                     int dbg = 0, int persist_1024 = 0) {
    const int lane = threadIdx.x & 31;
    // L2 residency control: the first persist_1024/1024 of A's tiles are
    // loaded evict-last so they survive in the 126 MB L2 from one SpMV to the
    // next (the MAS inverses stream evict-first in between); the rest
    // evict-first.
    const std::uint64_t pol_keep = policy_evict_last(), pol_stream = policy_evict_first();
    const std::int64_t warp0 = (static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const std::int64_t nwarps = (static_cast<std::int64_t>(gridDim.x) * blockDim.x) >> 5;
    // each warp owns a contiguous run of 32-block chunks (row locality for the
    // x gathers and y atomics); software-pipelined: the next chunk's indices
    // and block planes are in flight while the current chunk is processed
    const std::int64_t n_chunks = (U + 31) >> 5;
    const std::int64_t ch0 = warp0 * n_chunks / nwarps, ch1 = (warp0 + 1) * n_chunks / nwarps;
    double dsum = 0;
    std::uint32_t nr = 0xFFFFFFFFu, nc = 0;
    double nh[9];
    auto load = [&](std::int64_t ch) {
        const std::int64_t e = (ch << 5) + lane;
        nr = 0xFFFFFFFFu;
        nc = 0;
        if (ch < ch1 && e < U) {
            const std::uint64_t pol = (ch * 1024 < static_cast<std::int64_t>(persist_1024) * n_chunks) ? pol_keep
                                                                                                      : pol_stream;
            nr = ld_nc_policy(rows + e, pol);
            nc = ld_nc_policy(cols + e, pol);
#pragma unroll
            for (int k = 0; k < 9; ++k) nh[k] = ld_nc_policy(blocks + blk(e, k), pol);  // one contiguous tile
        }
    };
    load(ch0);  // the matrix does not change during the solve: prefetched before the dependency wait
    pdl_wait();
    if (flags && flags[0]) return;  // PCG already finished (F_DONE)
    pdl_launch();
    for (std::int64_t ch = ch0; ch < ch1; ++ch) {
        const std::uint32_t r = nr, c = nc;
        double h[9];
#pragma unroll
        for (int k = 0; k < 9; ++k) h[k] = nh[k];
        load(ch + 1);
        const bool valid = r != 0xFFFFFFFFu;
        double yr0 = 0, yr1 = 0, yr2 = 0;
        double tc0 = 0, tc1 = 0, tc2 = 0;  // H^T x[row], towards y[col]
        bool tr = false;
        if (valid) {
            const std::uint32_t cx = dbg == 3 ? r : c;  // dbg 3: no column gather
            double xc0, xc1, xc2, xr0, xr1, xr2;
            if (kPad) {  // x padded to 4 doubles per slot: one 256-bit gather each
                double u0, u1;
                ldg_v4(x + 4 * static_cast<std::int64_t>(cx), xc0, xc1, xc2, u0);
                ldg_v4(x + 4 * static_cast<std::int64_t>(r), xr0, xr1, xr2, u1);
            } else {
                xc0 = ldg_issue(x + 3 * cx);
                xc1 = ldg_issue(x + 3 * cx + 1);
                xc2 = ldg_issue(x + 3 * cx + 2);
                xr0 = ldg_issue(x + 3 * r);
                xr1 = ldg_issue(x + 3 * r + 1);
                xr2 = ldg_issue(x + 3 * r + 2);
            }
            // column-major H(i,j) = h[3j+i]
            yr0 = h[0] * xc0 + h[3] * xc1 + h[6] * xc2;
            yr1 = h[1] * xc0 + h[4] * xc1 + h[7] * xc2;
            yr2 = h[2] * xc0 + h[5] * xc1 + h[8] * xc2;
            if (r != c && dbg != 1 && dbg != 2) {
                tc0 = h[0] * xr0 + h[1] * xr1 + h[2] * xr2;
                tc1 = h[3] * xr0 + h[4] * xr1 + h[5] * xr2;
                tc2 = h[6] * xr0 + h[7] * xr1 + h[8] * xr2;
                tr = true;
                if (!kCoalesce) {
                    red_add(y + 3 * c, tc0);
                    red_add(y + 3 * c + 1, tc1);
                    red_add(y + 3 * c + 2, tc2);
                }
            }
            if (kDot) dsum += (r != c ? 2.0 : 1.0) * (xr0 * yr0 + xr1 * yr1 + xr2 * yr2);
        }
        if (kCoalesce) {
            // the 96 scatter values of the chunk (block b, component k) go out in
            // three RED instructions, lane L of round I taking value 32 I + L:
            // each instruction hits ~11 blocks' contiguous 24-byte targets
            // instead of 32 scattered doubles
#pragma unroll
            for (int round = 0; round < 3; ++round) {
                const int v = 32 * round + lane;
                const int bsrc = v / 3, k = v - 3 * bsrc;
                const double a0 = __shfl_sync(0xffffffffu, tc0, bsrc);
                const double a1 = __shfl_sync(0xffffffffu, tc1, bsrc);
                const double a2 = __shfl_sync(0xffffffffu, tc2, bsrc);
                const std::uint32_t cb = __shfl_sync(0xffffffffu, c, bsrc);
                const bool tb = __shfl_sync(0xffffffffu, tr ? 1 : 0, bsrc) != 0;
                if (tb) red_add(y + 3 * static_cast<std::int64_t>(cb) + k, k == 0 ? a0 : (k == 1 ? a1 : a2));
            }
        }
        // head-segmented sum of the row contributions (rows sorted within the warp)
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const double a0 = __shfl_down_sync(0xffffffffu, yr0, off);
            const double a1 = __shfl_down_sync(0xffffffffu, yr1, off);
            const double a2 = __shfl_down_sync(0xffffffffu, yr2, off);
            const std::uint32_t ro = __shfl_down_sync(0xffffffffu, r, off);
            if (lane + off < 32 && ro == r) {
                yr0 += a0;
                yr1 += a1;
                yr2 += a2;
            }
        }
        const std::uint32_t rprev = __shfl_up_sync(0xffffffffu, r, 1);
        if (valid && (lane == 0 || rprev != r) && dbg != 2) {
            red_add(y + 3 * r, yr0);
            red_add(y + 3 * r + 1, yr1);
            red_add(y + 3 * r + 2, yr2);
        }
    }
    // the PCG's p.Ap SpMV opens an iteration: its last CTA advances F_K
    if (kDot) grid_sum_last_block(dsum, partials, ticket, dot_out, flags ? const_cast<int*>(flags) + F_K : nullptr);
}

// TMA-staged variant. On B200 the L1 data pipe moves one 32-byte sector per
// wavefront for LDG traffic, so streaming the matrix tiles through LDG costs
// as many L1 cycles as the scattered x gathers and y atomics together (ncu:
// ~146 sectors per 32-block chunk, 61 % of the L1 wavefront peak at 82 us).
// Here the tiles (2,304 B of blocks + 128 B rows + 128 B cols, one contiguous
// chunk each) arrive by cp.async.bulk into a per-warp ring of kStages shared
// buffers, bypassing the LSU; the warp reads them back with conflict-free
// 128-byte-per-wavefront LDS, and the LDG path carries only the x gathers.
struct __align__(16) ChunkStage {
    double blk[288];
    std::uint32_t rows[32];
    std::uint32_t cols[32];
};
constexpr int kTmaWarps = 8;
constexpr std::uint32_t kChunkBytes = sizeof(ChunkStage);

template <bool kDot, int kStages>
__global__ void __launch_bounds__(32 * kTmaWarps) k_spmv_tma(const std::uint32_t* __restrict__ rows,
                                                             const std::uint32_t* __restrict__ cols,
                                                             const double* __restrict__ blocks, std::int64_t U,
                                                             const double* __restrict__ x, double* __restrict__ y,
                                                             double* __restrict__ partials,
                                                             unsigned* __restrict__ ticket, double* __restrict__ dot_out,
                                                             const int* __restrict__ flags, int dbg = 0) {
    if (flags && flags[0]) return;  // PCG already finished (F_DONE)
    extern __shared__ __align__(128) unsigned char smem[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    ChunkStage* stage = reinterpret_cast<ChunkStage*>(smem) + w * kStages;
    std::uint64_t* bar = reinterpret_cast<std::uint64_t*>(smem + sizeof(ChunkStage) * kStages * kTmaWarps) + w * kStages;
    const std::int64_t warp0 = static_cast<std::int64_t>(blockIdx.x) * kTmaWarps + w;
    const std::int64_t nwarps = static_cast<std::int64_t>(gridDim.x) * kTmaWarps;
    const std::int64_t n_chunks = (U + 31) >> 5;
    const std::int64_t ch0 = warp0 * n_chunks / nwarps, ch1 = (warp0 + 1) * n_chunks / nwarps;
    auto issue = [&](std::int64_t ch, int s) {  // lane 0 only
        mbar_arrive_expect_tx(&bar[s], kChunkBytes);
        bulk_g2s_evict_first(stage[s].blk, blocks + ch * 288, 288 * 8, &bar[s]);
        bulk_g2s_evict_first(stage[s].rows, rows + ch * 32, 128, &bar[s]);
        bulk_g2s_evict_first(stage[s].cols, cols + ch * 32, 128, &bar[s]);
    };
    if (lane == 0) {
        for (int s = 0; s < kStages; ++s) mbar_init(&bar[s], 1);
        fence_mbar_init();
        for (int s = 0; s < kStages && ch0 + s < ch1; ++s) issue(ch0 + s, s);
    }
    __syncwarp();
    // Gathers run one chunk ahead: while chunk ch is multiplied, the x[col]
    // and x[row] loads of chunk ch+1 (whose indices are already staged) are in
    // flight, so the L2 round trip of the gathers is off the critical path.
    std::uint32_t r = 0xFFFFFFFFu, c = 0;
    double g[6];
    auto gather = [&](std::int64_t ch, int s, std::uint32_t par, std::uint32_t& rr, std::uint32_t& cc, double* gg) {
        mbar_wait(&bar[s], par);
        const bool valid = (ch << 5) + lane < U;
        rr = valid ? stage[s].rows[lane] : 0xFFFFFFFFu;
        cc = valid ? stage[s].cols[lane] : 0u;
        const std::uint32_t rx = valid ? rr : 0u;
        gg[0] = ldg_issue(x + 3 * cc);
        gg[1] = ldg_issue(x + 3 * cc + 1);
        gg[2] = ldg_issue(x + 3 * cc + 2);
        gg[3] = ldg_issue(x + 3 * rx);
        gg[4] = ldg_issue(x + 3 * rx + 1);
        gg[5] = ldg_issue(x + 3 * rx + 2);
    };
    if (ch0 < ch1) gather(ch0, 0, 0u, r, c, g);
    double dsum = 0;
    int s = 0;
    std::uint32_t par = 0;
    for (std::int64_t ch = ch0; ch < ch1; ++ch) {
        double h[9];
#pragma unroll
        for (int k = 0; k < 9; ++k) h[k] = stage[s].blk[32 * k + lane];
        int sn = s + 1;
        std::uint32_t pn = par;
        if (sn == kStages) {
            sn = 0;
            pn ^= 1u;
        }
        std::uint32_t rn = 0xFFFFFFFFu, cn = 0;
        double gn[6];
        if (ch + 1 < ch1) gather(ch + 1, sn, pn, rn, cn, gn);
        __syncwarp();
        if (lane == 0 && ch + kStages < ch1) {  // refill this stage kStages chunks ahead
            fence_proxy_async();
            issue(ch + kStages, s);
        }
        s = sn;
        par = pn;
        const bool valid = r != 0xFFFFFFFFu;
        double yr0 = 0, yr1 = 0, yr2 = 0;
        if (valid) {
            const double xc0 = g[0], xc1 = g[1], xc2 = g[2], xr0 = g[3], xr1 = g[4], xr2 = g[5];
            // column-major H(i,j) = h[3j+i]
            yr0 = h[0] * xc0 + h[3] * xc1 + h[6] * xc2;
            yr1 = h[1] * xc0 + h[4] * xc1 + h[7] * xc2;
            yr2 = h[2] * xc0 + h[5] * xc1 + h[8] * xc2;
            if (r != c && dbg != 2) {
                red_add(y + 3 * c, h[0] * xr0 + h[1] * xr1 + h[2] * xr2);
                red_add(y + 3 * c + 1, h[3] * xr0 + h[4] * xr1 + h[5] * xr2);
                red_add(y + 3 * c + 2, h[6] * xr0 + h[7] * xr1 + h[8] * xr2);
            }
            if (kDot) dsum += (r != c ? 2.0 : 1.0) * (xr0 * yr0 + xr1 * yr1 + xr2 * yr2);
        }
        // head-segmented sum of the row contributions (rows sorted within the chunk)
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const double a0 = __shfl_down_sync(0xffffffffu, yr0, off);
            const double a1 = __shfl_down_sync(0xffffffffu, yr1, off);
            const double a2 = __shfl_down_sync(0xffffffffu, yr2, off);
            const std::uint32_t ro = __shfl_down_sync(0xffffffffu, r, off);
            if (lane + off < 32 && ro == r) {
                yr0 += a0;
                yr1 += a1;
                yr2 += a2;
            }
        }
        const std::uint32_t rprev = __shfl_up_sync(0xffffffffu, r, 1);
        if (valid && (lane == 0 || rprev != r) && dbg != 2) {
            red_add(y + 3 * r, yr0);
            red_add(y + 3 * r + 1, yr1);
            red_add(y + 3 * r + 2, yr2);
        }
        r = rn;
        c = cn;
#pragma unroll
        for (int k = 0; k < 6; ++k) g[k] = gn[k];
    }
    // the PCG's p.Ap SpMV opens an iteration: its last CTA advances F_K
    if (kDot) grid_sum_last_block(dsum, partials, ticket, dot_out, flags ? const_cast<int*>(flags) + F_K : nullptr);
}

// Two blocks per lane: a warp step covers a pair of 32-block tiles (one
// 5,120-byte TMA stage); lane l owns blocks 2l and 2l+1 of the pair (its two
// values of each of the 9 planes are one 128-bit shared load). Rows are
// sorted, so a lane holds at most two rows: its last row r1 with the partial
// y1 (+ y0 when r0 == r1) enters an inclusive segmented scan over the lanes
// (shfl_up, keyed by r1); a first row r0 != r1 closes there, completed by the
// scanned total of the previous lane when that lane's key is r0. Half the
// shared-load instructions, ~40 % fewer shuffles per block than k_spmv_tma.
struct __align__(16) PairStage {
    double blk[576];
    std::uint32_t rows[64];
    std::uint32_t cols[64];
};

template <bool kDot, int kStages>
__global__ void __launch_bounds__(32 * kTmaWarps) k_spmv_tma2(const std::uint32_t* __restrict__ rows,
                                                              const std::uint32_t* __restrict__ cols,
                                                              const double* __restrict__ blocks, std::int64_t U,
                                                              const double* __restrict__ x, double* __restrict__ y,
                                                              double* __restrict__ partials,
                                                              unsigned* __restrict__ ticket,
                                                              double* __restrict__ dot_out,
                                                              const int* __restrict__ flags, int dbg = 0) {
    if (flags && flags[0]) return;  // PCG already finished (F_DONE)
    extern __shared__ __align__(128) unsigned char smem[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    PairStage* stage = reinterpret_cast<PairStage*>(smem) + w * kStages;
    std::uint64_t* bar = reinterpret_cast<std::uint64_t*>(smem + sizeof(PairStage) * kStages * kTmaWarps) + w * kStages;
    const std::int64_t warp0 = static_cast<std::int64_t>(blockIdx.x) * kTmaWarps + w;
    const std::int64_t nwarps = static_cast<std::int64_t>(gridDim.x) * kTmaWarps;
    const std::int64_t n_chunks = (U + 31) >> 5;      // 32-block tiles (rows/cols padded to whole tiles)
    const std::int64_t n_pairs = (n_chunks + 1) >> 1;  // tile pairs
    const std::int64_t q0 = warp0 * n_pairs / nwarps, q1 = (warp0 + 1) * n_pairs / nwarps;
    auto issue = [&](std::int64_t q, int s) {  // lane 0 only
        const std::int64_t t0 = 2 * q;
        const int nt = t0 + 1 < n_chunks ? 2 : 1;
        mbar_arrive_expect_tx(&bar[s], static_cast<std::uint32_t>(nt * (288 * 8 + 256)));
        bulk_g2s_evict_first(stage[s].blk, blocks + t0 * 288, nt * 288 * 8, &bar[s]);
        bulk_g2s_evict_first(stage[s].rows, rows + t0 * 32, nt * 128, &bar[s]);
        bulk_g2s_evict_first(stage[s].cols, cols + t0 * 32, nt * 128, &bar[s]);
    };
    if (lane == 0) {
        for (int s = 0; s < kStages; ++s) mbar_init(&bar[s], 1);
        fence_mbar_init();
        for (int s = 0; s < kStages && q0 + s < q1; ++s) issue(q0 + s, s);
    }
    __syncwarp();
    const int tile = lane >> 4;
    const int wi = tile * 288 + 2 * (lane & 15);  // double offset of block 2l inside plane 0 of the stage
    constexpr std::uint32_t kNone = 0xFFFFFFFFu;
    // indices + gathers of a pair (issued one pair ahead)
    std::uint32_t r0 = kNone, r1 = kNone, c0 = 0, c1 = 0;
    double g[12];
    auto gather = [&](std::int64_t q, int s, std::uint32_t par, std::uint32_t& a0, std::uint32_t& a1,
                      std::uint32_t& b0, std::uint32_t& b1, double* gg) {
        mbar_wait(&bar[s], par);
        const std::int64_t e = 64 * q + 2 * lane;
        const uint2 rr = *reinterpret_cast<const uint2*>(&stage[s].rows[2 * lane]);
        const uint2 cc = *reinterpret_cast<const uint2*>(&stage[s].cols[2 * lane]);
        a0 = e < U ? rr.x : kNone;
        a1 = e + 1 < U ? rr.y : kNone;
        b0 = e < U ? cc.x : 0u;
        b1 = e + 1 < U ? cc.y : 0u;
        const std::uint32_t x0 = a0 != kNone ? a0 : 0u, x1 = a1 != kNone ? a1 : x0;
        gg[0] = ldg_issue(x + 3 * b0);
        gg[1] = ldg_issue(x + 3 * b0 + 1);
        gg[2] = ldg_issue(x + 3 * b0 + 2);
        gg[3] = ldg_issue(x + 3 * b1);
        gg[4] = ldg_issue(x + 3 * b1 + 1);
        gg[5] = ldg_issue(x + 3 * b1 + 2);
        gg[6] = ldg_issue(x + 3 * x0);
        gg[7] = ldg_issue(x + 3 * x0 + 1);
        gg[8] = ldg_issue(x + 3 * x0 + 2);
        if (x1 != x0) {
            gg[9] = ldg_issue(x + 3 * x1);
            gg[10] = ldg_issue(x + 3 * x1 + 1);
            gg[11] = ldg_issue(x + 3 * x1 + 2);
        } else {
            gg[9] = gg[6];
            gg[10] = gg[7];
            gg[11] = gg[8];
        }
    };
    if (q0 < q1) gather(q0, 0, 0u, r0, r1, c0, c1, g);
    double dsum = 0;
    int s = 0;
    std::uint32_t par = 0;
    for (std::int64_t q = q0; q < q1; ++q) {
        double h0[9], h1[9];
#pragma unroll
        for (int k = 0; k < 9; ++k) {
            const double2 v = *reinterpret_cast<const double2*>(&stage[s].blk[wi + 32 * k]);
            h0[k] = v.x;
            h1[k] = v.y;
        }
        int sn = s + 1;
        std::uint32_t pn = par;
        if (sn == kStages) {
            sn = 0;
            pn ^= 1u;
        }
        std::uint32_t rn0 = kNone, rn1 = kNone, cn0 = 0, cn1 = 0;
        double gn[12];
        if (q + 1 < q1) gather(q + 1, sn, pn, rn0, rn1, cn0, cn1, gn);
        __syncwarp();
        if (lane == 0 && q + kStages < q1) {
            fence_proxy_async();
            issue(q + kStages, s);
        }
        s = sn;
        par = pn;
        // the two blocks: H x[col] towards the row, H^T x[row] scattered to col
        double y0[3] = {0, 0, 0}, y1[3] = {0, 0, 0};
        if (r0 != kNone) {
            y0[0] = h0[0] * g[0] + h0[3] * g[1] + h0[6] * g[2];
            y0[1] = h0[1] * g[0] + h0[4] * g[1] + h0[7] * g[2];
            y0[2] = h0[2] * g[0] + h0[5] * g[1] + h0[8] * g[2];
            if (r0 != c0 && dbg != 2) {
                red_add(y + 3 * c0, h0[0] * g[6] + h0[1] * g[7] + h0[2] * g[8]);
                red_add(y + 3 * c0 + 1, h0[3] * g[6] + h0[4] * g[7] + h0[5] * g[8]);
                red_add(y + 3 * c0 + 2, h0[6] * g[6] + h0[7] * g[7] + h0[8] * g[8]);
            }
            if (kDot) dsum += (r0 != c0 ? 2.0 : 1.0) * (g[6] * y0[0] + g[7] * y0[1] + g[8] * y0[2]);
        }
        if (r1 != kNone) {
            y1[0] = h1[0] * g[3] + h1[3] * g[4] + h1[6] * g[5];
            y1[1] = h1[1] * g[3] + h1[4] * g[4] + h1[7] * g[5];
            y1[2] = h1[2] * g[3] + h1[5] * g[4] + h1[8] * g[5];
            if (r1 != c1 && dbg != 2) {
                red_add(y + 3 * c1, h1[0] * g[9] + h1[1] * g[10] + h1[2] * g[11]);
                red_add(y + 3 * c1 + 1, h1[3] * g[9] + h1[4] * g[10] + h1[5] * g[11]);
                red_add(y + 3 * c1 + 2, h1[6] * g[9] + h1[7] * g[10] + h1[8] * g[11]);
            }
            if (kDot) dsum += (r1 != c1 ? 2.0 : 1.0) * (g[9] * y1[0] + g[10] * y1[1] + g[11] * y1[2]);
        }
        // lane key = last row; a first row that differs closes in this lane
        const bool two = r0 != r1 && r1 != kNone;
        const std::uint32_t key = r1 != kNone ? r1 : r0;
        double v0 = two ? y1[0] : y0[0] + y1[0];
        double v1 = two ? y1[1] : y0[1] + y1[1];
        double v2 = two ? y1[2] : y0[2] + y1[2];
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {  // inclusive segmented scan over lanes
            const double a0 = __shfl_up_sync(0xffffffffu, v0, off);
            const double a1 = __shfl_up_sync(0xffffffffu, v1, off);
            const double a2 = __shfl_up_sync(0xffffffffu, v2, off);
            const std::uint32_t ko = __shfl_up_sync(0xffffffffu, key, off);
            if (lane >= off && ko == key) {
                v0 += a0;
                v1 += a1;
                v2 += a2;
            }
        }
        const std::uint32_t kprev = __shfl_up_sync(0xffffffffu, key, 1);
        const double p0 = __shfl_up_sync(0xffffffffu, v0, 1);
        const double p1 = __shfl_up_sync(0xffffffffu, v1, 1);
        const double p2 = __shfl_up_sync(0xffffffffu, v2, 1);
        const std::uint32_t knext_first = __shfl_down_sync(0xffffffffu, r0, 1);
        if (two && dbg != 2) {  // row r0 ends here
            const bool cont = lane > 0 && kprev == r0;
            red_add(y + 3 * r0, y0[0] + (cont ? p0 : 0.0));
            red_add(y + 3 * r0 + 1, y0[1] + (cont ? p1 : 0.0));
            red_add(y + 3 * r0 + 2, y0[2] + (cont ? p2 : 0.0));
        }
        // the key's total leaves from its last lane, unless the next lane
        // closes the same row as its first row
        if (key != kNone && dbg != 2 && (lane == 31 || knext_first != key)) {
            red_add(y + 3 * key, v0);
            red_add(y + 3 * key + 1, v1);
            red_add(y + 3 * key + 2, v2);
        }
        r0 = rn0;
        r1 = rn1;
        c0 = cn0;
        c1 = cn1;
#pragma unroll
        for (int k = 0; k < 12; ++k) g[k] = gn[k];
    }
    if (kDot) grid_sum_last_block(dsum, partials, ticket, dot_out, flags ? const_cast<int*>(flags) + F_K : nullptr);
}

template <int kStages>
constexpr std::size_t tma2_smem() {
    return (sizeof(PairStage) + sizeof(std::uint64_t)) * kStages * kTmaWarps;
}

template <int kStages>
constexpr std::size_t tma_smem() {
    return (sizeof(ChunkStage) + sizeof(std::uint64_t)) * kStages * kTmaWarps;
}

}  // namespace

// Launch of one SpMV variant (0: LDG-streamed k_spmv; 2/3/4: k_spmv_tma with
// that many stages per warp). One wave: SMs x resident CTAs per SM, each warp
// then streams one contiguous run of chunks.
namespace {
struct SpmvLaunch {
    int grid = 1, block = 256;
    std::size_t smem = 0;
};

template <class K>
SpmvLaunch spmv_config(K kernel, int block, std::size_t smem, const Ctx& c, std::int64_t U) {
    static_assert(sizeof(K) > 0, "");
    int occ = 0;
    if (smem > 0) ADIPC_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    ADIPC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, block, smem));
    if (occ < 1) occ = 1;
    int sms = kSMs;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c.device);
    const std::int64_t need = ceil_div(ceil_div(U, 32), block / 32);
    SpmvLaunch l;
    l.grid = static_cast<int>(std::max<std::int64_t>(1, std::min<std::int64_t>(need, static_cast<std::int64_t>(sms) * occ)));
    l.block = block;
    l.smem = smem;
    return l;
}

template <bool kDot>
void launch_variant(Ctx& c, const DeviceMatrix& M, int variant, const double* d_x, double* d_y, double* partials,
                    unsigned* ticket, double* dot_out, const int* flags, int dbg, bool pad = false) {
    cudaStream_t st = c.stream;
#define ADIPC_TMA(S)                                                                                              \
    do {                                                                                                          \
        static SpmvLaunch cfg;                                                                                    \
        static std::int64_t cfg_u = -1;                                                                           \
        if (cfg_u != M.U) {                                                                                       \
            cfg = spmv_config(k_spmv_tma<kDot, S>, 32 * kTmaWarps, tma_smem<S>(), c, M.U);                         \
            cfg_u = M.U;                                                                                          \
        }                                                                                                         \
        k_spmv_tma<kDot, S><<<cfg.grid, cfg.block, cfg.smem, st>>>(M.rows.p, M.cols.p, M.blocks.p, M.U, d_x, d_y, \
                                                                   partials, ticket, dot_out, flags, dbg);        \
    } while (0)
#define ADIPC_TMA2(S)                                                                                         \
    do {                                                                                                          \
        static SpmvLaunch cfg;                                                                                    \
        static std::int64_t cfg_u = -1;                                                                           \
        if (cfg_u != M.U) {                                                                                       \
            cfg = spmv_config(k_spmv_tma2<kDot, S>, 32 * kTmaWarps, tma2_smem<S>(), c, M.U);                       \
            cfg_u = M.U;                                                                                          \
        }                                                                                                         \
        k_spmv_tma2<kDot, S><<<cfg.grid, cfg.block, cfg.smem, st>>>(M.rows.p, M.cols.p, M.blocks.p, M.U, d_x, d_y, \
                                                                    partials, ticket, dot_out, flags, dbg);       \
    } while (0)
    if (variant == 5)
        ADIPC_TMA2(2);
    else if (variant == 6)
        ADIPC_TMA2(3);
    else if (variant == 2)
        ADIPC_TMA(2);
    else if (variant == 3)
        ADIPC_TMA(3);
    else if (variant == 4)
        ADIPC_TMA(4);
    else {
        static SpmvLaunch cfg;
        static std::int64_t cfg_u = -1;
        if (cfg_u != M.U) {
            cfg = spmv_config(k_spmv<kDot>, kSpmvThreads, 0, c, M.U);
            cfg_u = M.U;
        }
        if (pad)
            k_spmv<kDot, true><<<cfg.grid, cfg.block, 0, st>>>(M.rows.p, M.cols.p, M.blocks.p, M.U, d_x, d_y, partials,
                                                               ticket, dot_out, flags, dbg, c.l2_persist_1024);
        else if (variant == 7)
            k_spmv<kDot, false, true><<<cfg.grid, cfg.block, 0, st>>>(M.rows.p, M.cols.p, M.blocks.p, M.U, d_x, d_y,
                                                                      partials, ticket, dot_out, flags, dbg,
                                                                      c.l2_persist_1024);
        else
            ADIPC_CUDA(launch_pdl(k_spmv<kDot, false, false>, dim3(cfg.grid), dim3(cfg.block), 0, st, c.pdl, M.rows.p,
                                  M.cols.p, M.blocks.p, M.U, d_x, d_y, partials, ticket, dot_out, flags, dbg,
                                  c.l2_persist_1024));
    }
#undef ADIPC_TMA
#undef ADIPC_TMA2
    ADIPC_LAUNCH_CHECK();
}
}  // namespace

// upper bound of the grid of any variant (sizes the per-CTA partials)
int spmv_grid(const Ctx& c, const DeviceMatrix& M) {
    int sms = kSMs;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c.device);
    return sms * 8;
}

// y (+)= A x. zero_y: clear y first (otherwise the caller guarantees y == 0).
// With `dot_out`: x.(A x) -> *dot_out (device), using `partials`
// (>= spmv_grid doubles) and `ticket` (one zeroed unsigned). `flags`: skip
// when the PCG solve is done.
void spmv_launch(Ctx& c, const DeviceMatrix& M, const double* d_x, double* d_y, bool zero_y, const int* flags,
                 double* partials, unsigned* ticket, double* dot_out, bool pad) {
    const std::int64_t nx3 = 3 * static_cast<std::int64_t>(M.n);
    if (zero_y) ADIPC_CUDA(cudaMemsetAsync(d_y, 0, sizeof(double) * nx3, c.stream));
    if (M.U == 0) {
        if (dot_out) ADIPC_CUDA(cudaMemsetAsync(dot_out, 0, sizeof(double), c.stream));
        return;
    }
    if (c.spmv_variant == 8 && &M == &c.S() && sell_current(c)) {  // sliced-ELL copy (sell.cu)
        sell_spmv_launch(c, d_x, d_y, flags, partials, ticket, dot_out);
        return;
    }
    if (dot_out)
        launch_variant<true>(c, M, pad ? 0 : c.spmv_variant, d_x, d_y, partials, ticket, dot_out, flags, 0, pad);
    else
        launch_variant<false>(c, M, pad ? 0 : c.spmv_variant, d_x, d_y, nullptr, nullptr, nullptr, flags, 0, pad);
}

// Debug timing of the SpMV variants: mode & 7 = 0 normal, 1 no transposed
// scatter, 2 no atomics, 3 no column gather (LDG kernel only); +8: evict L2
// (256 MB write) before every launch, as inside PCG; mode >> 4 = variant
// (0 LDG-streamed, 2/3/4 TMA stages). ms per launch over `iters` launches.
// +256: the solve-order matrix with the last PCG's p as x (in-situ inputs).
float spmv_debug_time(Ctx& c, const double* d_x, double* d_y, int mode, int iters) {
    const int mode_all = mode;
    const bool cold = (mode & 8) != 0;
    const bool insitu = (mode & 256) != 0;
    const int variant = (mode >> 4) & 15;
    mode &= 7;
    const DeviceMatrix& M = insitu ? c.S() : c.A;
    if (insitu) {
        d_x = c.w.p.p;
        c.w.tmp.reserve(3 * static_cast<std::size_t>(M.n));
        d_y = c.w.tmp.p;
    }
    cudaEvent_t e0, e1;
    ADIPC_CUDA(cudaEventCreate(&e0));
    ADIPC_CUDA(cudaEventCreate(&e1));
    DBuf<char> flush;
    if (cold) flush.reserve(256u << 20);
    // +512: the p.Ap-fused kernel (own partials / ticket / result)
    const bool dot = (mode_all & 512) != 0;
    DBuf<double> dpart;
    DBuf<unsigned> dtick;
    if (dot) {
        dpart.reserve(static_cast<std::size_t>(spmv_grid(c, M)) + 1);
        dtick.reserve(1);
        ADIPC_CUDA(cudaMemsetAsync(dtick.p, 0, sizeof(unsigned), c.stream));
    }
    float total = 0;
    for (int i = -2; i < iters; ++i) {
        if (cold) ADIPC_CUDA(cudaMemsetAsync(flush.p, i & 0xff, 256u << 20, c.stream));
        ADIPC_CUDA(cudaEventRecord(e0, c.stream));
        if (variant == 8)  // the sliced-ELL copy as built (c.sell)
            sell_spmv_launch(c, d_x, d_y, nullptr, dot ? dpart.p : nullptr, dot ? dtick.p : nullptr,
                             dot ? dpart.p + spmv_grid(c, M) : nullptr);
        else if (dot)
            launch_variant<true>(c, M, variant, d_x, d_y, dpart.p, dtick.p, dpart.p + spmv_grid(c, M), nullptr, mode);
        else
            launch_variant<false>(c, M, variant, d_x, d_y, nullptr, nullptr, nullptr, nullptr, mode);
        ADIPC_CUDA(cudaEventRecord(e1, c.stream));
        ADIPC_CUDA(cudaEventSynchronize(e1));
        float ms = 0;
        ADIPC_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        if (i >= 0) total += ms;
    }
    flush.free();
    dpart.free();
    dtick.free();
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return total / iters;
}

void spmv(Ctx& c, const double* d_x, double* d_y, double*, int) {
    spmv_launch(c, c.A, d_x, d_y, true, nullptr, nullptr, nullptr, nullptr);
}

}  // namespace adipc_gpu
