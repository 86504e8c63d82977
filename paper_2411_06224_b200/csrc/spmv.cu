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
constexpr int kSpmvMinBlocks = 2;  // 2 x 256 threads: the two-stage pipeline's 114 registers without spills

// Each warp owns a contiguous run of 32-block chunks (row locality for the x
// gathers and y atomics), software-pipelined two deep: chunk ch is computed
// while the x gathers of chunk ch + 1 and the indices / blocks of chunk ch + 2
// are in flight (114 registers, 2 CTAs of 256 per SM; one stage deep at 3
// CTAs / SM measured 63.2 vs 62.0 us per cfg5 SpMV, 136.8 vs 134.8 us per PCG
// iteration). A streams through L2 once per SpMV (evict-first): it is 200 MB
// at cfg5, larger than the 126 MB L2, and the vectors the gathers hit stay.
template <bool kDot>
__global__ void __launch_bounds__(kSpmvThreads, kSpmvMinBlocks) k_spmv(const std::uint32_t* __restrict__ rows,
                                                     const std::uint32_t* __restrict__ cols,
                                                     const double* __restrict__ blocks, std::int64_t U,
                                                     const double* __restrict__ x, double* __restrict__ y,
                                                     double* __restrict__ partials, unsigned* __restrict__ ticket,
                                                     double* __restrict__ dot_out, const int* __restrict__ flags) {
    const int lane = threadIdx.x & 31;
    const std::uint64_t pol = policy_evict_first();
    const std::int64_t warp0 = (static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const std::int64_t nwarps = (static_cast<std::int64_t>(gridDim.x) * blockDim.x) >> 5;
    const std::int64_t n_chunks = (U + 31) >> 5;
    const std::int64_t ch0 = warp0 * n_chunks / nwarps, ch1 = (warp0 + 1) * n_chunks / nwarps;
    double dsum = 0;
    std::uint32_t ar = 0xFFFFFFFFu, ac = 0;  // stage A: indices + blocks in flight
    double ah[9];
    auto load = [&](std::int64_t ch) {
        const std::int64_t e = (ch << 5) + lane;
        ar = 0xFFFFFFFFu;
        ac = 0;
        if (ch < ch1 && e < U) {
            ar = ld_nc_policy(rows + e, pol);
            ac = ld_nc_policy(cols + e, pol);
#pragma unroll
            for (int k = 0; k < 9; ++k) ah[k] = ld_nc_policy(blocks + blk(e, k), pol);
        }
    };
    std::uint32_t br = 0xFFFFFFFFu, bc = 0;  // stage B: x gathers in flight
    double bh[9], bx[6];
    auto advance = [&] {  // A -> B, issue B's gathers
        br = ar;
        bc = ac;
#pragma unroll
        for (int k = 0; k < 9; ++k) bh[k] = ah[k];
        if (br != 0xFFFFFFFFu) {
            bx[0] = ldg_issue(x + 3 * bc);
            bx[1] = ldg_issue(x + 3 * bc + 1);
            bx[2] = ldg_issue(x + 3 * bc + 2);
            bx[3] = ldg_issue(x + 3 * br);
            bx[4] = ldg_issue(x + 3 * br + 1);
            bx[5] = ldg_issue(x + 3 * br + 2);
        }
    };
    load(ch0);
    pdl_wait();
    if (flags && flags[0]) return;
    pdl_launch();
    advance();
    load(ch0 + 1);
    for (std::int64_t ch = ch0; ch < ch1; ++ch) {
        const std::uint32_t r = br, c = bc;
        double h[9], xv[6];
#pragma unroll
        for (int k = 0; k < 9; ++k) h[k] = bh[k];
#pragma unroll
        for (int k = 0; k < 6; ++k) xv[k] = bx[k];
        advance();
        load(ch + 2);
        const bool valid = r != 0xFFFFFFFFu;
        double yr0 = 0, yr1 = 0, yr2 = 0;
        if (valid) {
            yr0 = h[0] * xv[0] + h[3] * xv[1] + h[6] * xv[2];
            yr1 = h[1] * xv[0] + h[4] * xv[1] + h[7] * xv[2];
            yr2 = h[2] * xv[0] + h[5] * xv[1] + h[8] * xv[2];
            if (kDot) dsum += (r != c ? 2.0 : 1.0) * (xv[3] * yr0 + xv[4] * yr1 + xv[5] * yr2);
        }
        // H^T x[row] towards y[col]: lanes of the chunk with the same column
        // (~30 % at cfg5: a node shared by the chunk's ~5 rows) are summed
        // into their lowest lane first, which alone issues the REDs
        {
            const bool tr = valid && r != c;
            double t0 = tr ? h[0] * xv[3] + h[1] * xv[4] + h[2] * xv[5] : 0.0;
            double t1 = tr ? h[3] * xv[3] + h[4] * xv[4] + h[5] * xv[5] : 0.0;
            double t2 = tr ? h[6] * xv[3] + h[7] * xv[4] + h[8] * xv[5] : 0.0;
            const std::uint32_t key = tr ? c : 0xFFFFFFFFu;
            const unsigned grp = __match_any_sync(0xffffffffu, key);
            const int gsize = __popc(grp);
            const int rounds = __reduce_max_sync(0xffffffffu, tr ? gsize : 1) - 1;
            const bool lead = tr && (__ffs(grp) - 1) == lane;
            unsigned rest = grp & (grp - 1u);  // members after the leader
            for (int k = 0; k < rounds; ++k) {
                const int src = rest ? __ffs(rest) - 1 : lane;
                const double a0 = __shfl_sync(0xffffffffu, t0, src);
                const double a1 = __shfl_sync(0xffffffffu, t1, src);
                const double a2 = __shfl_sync(0xffffffffu, t2, src);
                if (lead && rest) {
                    t0 += a0;
                    t1 += a1;
                    t2 += a2;
                }
                rest &= rest - 1u;
            }
            if (lead) {
                red_add(y + 3 * c, t0);
                red_add(y + 3 * c + 1, t1);
                red_add(y + 3 * c + 2, t2);
            }
        }
        // head-segmented sum of the row contributions (rows sorted within the
        // chunk): run heads from one ballot, and in each shuffle round a lane
        // adds its partner's value when no run starts between them
        const std::uint32_t rprev = __shfl_up_sync(0xffffffffu, r, 1);
        const bool head = lane == 0 || rprev != r;
        const std::uint64_t heads = __ballot_sync(0xffffffffu, head);
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const double a0 = __shfl_down_sync(0xffffffffu, yr0, off);
            const double a1 = __shfl_down_sync(0xffffffffu, yr1, off);
            const double a2 = __shfl_down_sync(0xffffffffu, yr2, off);
            const bool same = lane + off < 32 && ((heads >> (lane + 1)) & ((1ull << off) - 1ull)) == 0;
            if (same) {
                yr0 += a0;
                yr1 += a1;
                yr2 += a2;
            }
        }
        if (valid && head) {
            red_add(y + 3 * r, yr0);
            red_add(y + 3 * r + 1, yr1);
            red_add(y + 3 * r + 2, yr2);
        }
    }
    if (kDot) grid_sum_last_block(dsum, partials, ticket, dot_out, flags ? const_cast<int*>(flags) + F_K : nullptr);
}

// Deterministic SpMV (srbk_spmv.hpp:20-27, the serial path the reference
// takes under ExecPolicy::deterministic): one warp per row i, no atomics.
// y[i] receives, in the reference's serial order, first the transposed
// contributions H_e^T x[r] of the entries e = (r, i), r < i (ascending r —
// the column index built by build_transpose_index), then H_e x[c] of row i's
// own entries (ascending c, diagonal first). Lanes compute the 3x3 products in
// parallel (explicitly rounded mul/add in Eigen's ((h0 x0 + h1 x1) + h2 x2)
// order), lane 0 folds them sequentially: bitwise the reference's serial y,
// and identical from run to run. With kDot: p.Ap = sum_i x_i . y_i (fixed
// order, finished by the last CTA).
template <bool kDot>
__global__ void __launch_bounds__(256) k_spmv_det(std::int32_t n, const std::uint32_t* __restrict__ rows,
                                                  const std::uint32_t* __restrict__ cols,
                                                  const double* __restrict__ blocks,
                                                  const std::int64_t* __restrict__ row_ptr,
                                                  const std::int64_t* __restrict__ tptr,
                                                  const std::uint32_t* __restrict__ tidx, const double* __restrict__ x,
                                                  double* __restrict__ y, double* __restrict__ partials,
                                                  unsigned* __restrict__ ticket, double* __restrict__ dot_out,
                                                  const int* __restrict__ flags) {
    pdl_wait();
    if (flags && flags[0]) return;
    pdl_launch();
    const int lane = threadIdx.x & 31;
    const std::int32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const std::int32_t warps = (gridDim.x * blockDim.x) >> 5;
    double dsum = 0;
    for (std::int32_t i = warp; i < n; i += warps) {
        const std::int64_t t0 = tptr[i], nt = tptr[i + 1] - t0;
        const std::int64_t r0 = row_ptr[i], m = nt + (row_ptr[i + 1] - r0);
        double a0 = 0, a1 = 0, a2 = 0;  // lane 0: y[i]
        for (std::int64_t base = 0; base < m; base += 32) {
            const std::int64_t j = base + lane;
            double v0 = 0, v1 = 0, v2 = 0;
            if (j < m) {
                const bool tr = j < nt;
                const std::int64_t e = tr ? static_cast<std::int64_t>(tidx[t0 + j]) : r0 + (j - nt);
                const std::uint32_t o = tr ? rows[e] : cols[e];
                double h[9];
#pragma unroll
                for (int k = 0; k < 9; ++k) h[k] = blocks[blk(e, k)];
                const double x0 = x[3 * static_cast<std::int64_t>(o)], x1 = x[3 * static_cast<std::int64_t>(o) + 1],
                             x2 = x[3 * static_cast<std::int64_t>(o) + 2];
                // H(i,j) = h[3j+i]; tr: H^T x, else H x
                auto dot3 = [](double p0, double q0, double p1, double q1, double p2, double q2) {
                    return __dadd_rn(__dadd_rn(__dmul_rn(p0, q0), __dmul_rn(p1, q1)), __dmul_rn(p2, q2));
                };
                if (tr) {
                    v0 = dot3(h[0], x0, h[1], x1, h[2], x2);
                    v1 = dot3(h[3], x0, h[4], x1, h[5], x2);
                    v2 = dot3(h[6], x0, h[7], x1, h[8], x2);
                } else {
                    v0 = dot3(h[0], x0, h[3], x1, h[6], x2);
                    v1 = dot3(h[1], x0, h[4], x1, h[7], x2);
                    v2 = dot3(h[2], x0, h[5], x1, h[8], x2);
                }
            }
            const int nv = static_cast<int>(m - base < 32 ? m - base : 32);
            for (int q = 0; q < nv; ++q) {
                const double b0 = __shfl_sync(0xffffffffu, v0, q);
                const double b1 = __shfl_sync(0xffffffffu, v1, q);
                const double b2 = __shfl_sync(0xffffffffu, v2, q);
                a0 = __dadd_rn(a0, b0);
                a1 = __dadd_rn(a1, b1);
                a2 = __dadd_rn(a2, b2);
            }
        }
        if (lane == 0) {
            y[3 * static_cast<std::int64_t>(i)] = a0;
            y[3 * static_cast<std::int64_t>(i) + 1] = a1;
            y[3 * static_cast<std::int64_t>(i) + 2] = a2;
            if (kDot)
                dsum += x[3 * static_cast<std::int64_t>(i)] * a0 + x[3 * static_cast<std::int64_t>(i) + 1] * a1 +
                        x[3 * static_cast<std::int64_t>(i) + 2] * a2;
        }
    }
    if (kDot) grid_sum_last_block(dsum, partials, ticket, dot_out, flags ? const_cast<int*>(flags) + F_K : nullptr);
}

// keys of the transpose index: off-diagonal entry e = (r, c) -> bucket c,
// sorted by r (then e); diagonal entries go to the spare bucket n
__global__ void k_transpose_keys(const std::uint32_t* __restrict__ rows, const std::uint32_t* __restrict__ cols,
                                 std::int64_t U, std::uint32_t n, std::uint64_t* __restrict__ keys) {
    for (std::int64_t e = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; e < U;
         e += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        const std::uint32_t r = rows[e], c = cols[e];
        keys[e] = r == c ? (static_cast<std::uint64_t>(n) << 32) : ((static_cast<std::uint64_t>(c) << 32) | r);
    }
}

__global__ void k_low_words(const std::uint64_t* __restrict__ in, std::int64_t n, std::uint32_t* __restrict__ out) {
    for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<std::int64_t>(gridDim.x) * blockDim.x)
        out[i] = static_cast<std::uint32_t>(in[i]);
}

}  // namespace

// Column index of the upper-stored matrix M for the deterministic SpMV:
// tptr[c] .. tptr[c+1] lists the off-diagonal entries (r, c), r < c, in
// ascending r (= entry order). Cached per matrix version.
static void build_transpose_index(Ctx& c, const DeviceMatrix& M) {
    if (c.det_version == M.version && c.det_matrix == &M) return;
    const std::int32_t n = M.n;
    c.perm_keys.reserve(static_cast<std::size_t>(std::max<std::int64_t>(M.U, 1)));
    if (M.U > 0) {
        k_transpose_keys<<<grid_for(M.U, 256, 16), 256, 0, c.stream>>>(M.rows.p, M.cols.p, M.U,
                                                                       static_cast<std::uint32_t>(n),
                                                                       c.perm_keys.p);
        ADIPC_LAUNCH_CHECK();
    }
    bucket_sort(c, c.perm_keys.p, M.U, n + 1, nullptr);  // sorted word: (r << 32) | e
    c.det_tptr.reserve(static_cast<std::size_t>(n) + 2);
    c.det_tidx.reserve(static_cast<std::size_t>(std::max<std::int64_t>(M.U, 1)));
    ADIPC_CUDA(cudaMemcpyAsync(c.det_tptr.p, c.row_start.p, sizeof(std::int64_t) * (n + 1), cudaMemcpyDeviceToDevice,
                               c.stream));
    if (M.U > 0) {
        k_low_words<<<grid_for(M.U, 256, 16), 256, 0, c.stream>>>(c.sorted.p, M.U, c.det_tidx.p);
        ADIPC_LAUNCH_CHECK();
    }
    c.det_version = M.version;
    c.det_matrix = &M;
}

// before capturing a deterministic PCG: the transpose index of the solve matrix
void prepare_spmv(Ctx& c, const DeviceMatrix& M) {
    if (c.deterministic && M.U > 0) build_transpose_index(c, M);
}

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
    if (c.deterministic) {
        build_transpose_index(c, M);
        const int grid = grid_for(M.n, 8, 8);
        if (dot_out)
            ADIPC_CUDA(launch_pdl(k_spmv_det<true>, dim3(grid), dim3(256), 0, c.stream, true, M.n, M.rows.p, M.cols.p,
                                  M.blocks.p, M.row_ptr.p, c.det_tptr.p, c.det_tidx.p, d_x, d_y, partials, ticket,
                                  dot_out, flags));
        else
            ADIPC_CUDA(launch_pdl(k_spmv_det<false>, dim3(grid), dim3(256), 0, c.stream, true, M.n, M.rows.p,
                                  M.cols.p, M.blocks.p, M.row_ptr.p, c.det_tptr.p, c.det_tidx.p, d_x, d_y,
                                  static_cast<double*>(nullptr), static_cast<unsigned*>(nullptr),
                                  static_cast<double*>(nullptr), flags));
        ADIPC_LAUNCH_CHECK();
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
