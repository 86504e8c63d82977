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
constexpr int kSpmvMinBlocks = 3;  // 3 x 256 threads (<= 85 registers, 24 warps/SM); 4 spills: 85 vs 61 us

template <bool kDot>
__global__ void __launch_bounds__(kSpmvThreads, kSpmvMinBlocks) k_spmv(const std::uint32_t* __restrict__ rows,
                                                     const std::uint32_t* __restrict__ cols,
                                                     const double* __restrict__ blocks, std::int64_t U,
                                                     const double* __restrict__ x, double* __restrict__ y,
                                                     double* __restrict__ partials, unsigned* __restrict__ ticket,
                                                     double* __restrict__ dot_out, const int* __restrict__ flags) {
    const int lane = threadIdx.x & 31;
    // A streams through L2 once per SpMV (evict-first): it is 200 MB at cfg5,
    // larger than the 126 MB L2, and the vectors the gathers hit should stay
    const std::uint64_t pol = policy_evict_first();
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
        if (valid) {
            const double xc0 = ldg_issue(x + 3 * c);
            const double xc1 = ldg_issue(x + 3 * c + 1);
            const double xc2 = ldg_issue(x + 3 * c + 2);
            const double xr0 = ldg_issue(x + 3 * r);
            const double xr1 = ldg_issue(x + 3 * r + 1);
            const double xr2 = ldg_issue(x + 3 * r + 2);
            // column-major H(i,j) = h[3j+i]
            yr0 = h[0] * xc0 + h[3] * xc1 + h[6] * xc2;
            yr1 = h[1] * xc0 + h[4] * xc1 + h[7] * xc2;
            yr2 = h[2] * xc0 + h[5] * xc1 + h[8] * xc2;
            if (r != c) {  // H^T x[row] towards y[col]
                red_add(y + 3 * c, h[0] * xr0 + h[1] * xr1 + h[2] * xr2);
                red_add(y + 3 * c + 1, h[3] * xr0 + h[4] * xr1 + h[5] * xr2);
                red_add(y + 3 * c + 2, h[6] * xr0 + h[7] * xr1 + h[8] * xr2);
            }
            if (kDot) dsum += (r != c ? 2.0 : 1.0) * (xr0 * yr0 + xr1 * yr1 + xr2 * yr2);
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
        if (valid && (lane == 0 || rprev != r)) {
            red_add(y + 3 * r, yr0);
            red_add(y + 3 * r + 1, yr1);
            red_add(y + 3 * r + 2, yr2);
        }
    }
    // the PCG's p.Ap SpMV opens an iteration: its last CTA advances F_K
    if (kDot) grid_sum_last_block(dsum, partials, ticket, dot_out, flags ? const_cast<int*>(flags) + F_K : nullptr);
}

}  // namespace

// One wave: SMs x resident CTAs per SM, each warp then streams one contiguous
// run of chunks.
int spmv_grid(const Ctx& c, const DeviceMatrix& M) {
    int sms = kSMs;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c.device);
    return sms * kSpmvMinBlocks;
}

// y (+)= A x. zero_y: clear y first (otherwise the caller guarantees y == 0).
// With `dot_out`: x.(A x) -> *dot_out (device), using `partials`
// (>= spmv_grid doubles) and `ticket` (one zeroed unsigned). `flags`: skip
// when the PCG solve is done.
void spmv_launch(Ctx& c, const DeviceMatrix& M, const double* d_x, double* d_y, bool zero_y, const int* flags,
                 double* partials, unsigned* ticket, double* dot_out) {
    const std::int64_t nx3 = 3 * static_cast<std::int64_t>(M.n);
    if (zero_y) ADIPC_CUDA(cudaMemsetAsync(d_y, 0, sizeof(double) * nx3, c.stream));
    if (M.U == 0) {
        if (dot_out) ADIPC_CUDA(cudaMemsetAsync(dot_out, 0, sizeof(double), c.stream));
        return;
    }
    const std::int64_t need = ceil_div(ceil_div(M.U, 32), kSpmvThreads / 32);
    const int grid = static_cast<int>(std::max<std::int64_t>(1, std::min<std::int64_t>(need, spmv_grid(c, M))));
    if (dot_out)
        ADIPC_CUDA(launch_pdl(k_spmv<true>, dim3(grid), dim3(kSpmvThreads), 0, c.stream, true, M.rows.p, M.cols.p,
                              M.blocks.p, M.U, d_x, d_y, partials, ticket, dot_out, flags));
    else
        ADIPC_CUDA(launch_pdl(k_spmv<false>, dim3(grid), dim3(kSpmvThreads), 0, c.stream, true, M.rows.p, M.cols.p,
                              M.blocks.p, M.U, d_x, d_y, static_cast<double*>(nullptr),
                              static_cast<unsigned*>(nullptr), static_cast<double*>(nullptr), flags));
    ADIPC_LAUNCH_CHECK();
}

void spmv(Ctx& c, const double* d_x, double* d_y) {
    spmv_launch(c, c.A, d_x, d_y, true, nullptr, nullptr, nullptr, nullptr);
}

}  // namespace adipc_gpu
