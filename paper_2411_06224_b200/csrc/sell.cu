// Sliced-ELL copy of the assembled matrix for the PCG's SpMV (SRBK semantics,
// sparse/srbk_spmv.hpp:13-49: every stored block H = A(r,c) contributes
// H x[c] to y[r] and, off the diagonal, H^T x[r] to y[c]).
//
// Why: the tile-per-warp SRBK kernel (spmv.cu) spends most of its issue slots
// in the head-segmented shuffle reduction of the row sums (~320 instructions
// per 32-block chunk at IPC ~1.3; neither its gathers, its REDs nor its
// streaming method bound it). Here one LANE owns one ROW: slices of 32
// consecutive rows of the reference-numbered matrix (whose rows are almost
// uniformly 8 upper blocks long: 97.7 % slot efficiency at cfg5, versus 67 %
// in solve order), slot s of a slice holding block s of each lane's row in
// the same 32-block SoA tile format as A (coalesced 256-byte loads per value
// plane). Row and column ids are stored already translated to the solve
// order, so the kernel works on the solve-order vectors directly; SRBK only
// needs each unordered block pair once, whichever numbering made it "upper".
// The row sum stays in registers (one RED per row component), no shuffles.
#include <algorithm>
#include <cstdlib>

#include "mas_kernels.cuh"
#include "scan.cuh"

namespace adipc_gpu {

namespace {

constexpr std::uint32_t kPad = 0xFFFFFFFFu;

__global__ void k_sell_len(std::int32_t n, const std::int64_t* __restrict__ row_ptr, std::int32_t n_slices,
                           std::int64_t* __restrict__ slice_len) {
    const std::int64_t w = (blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= n_slices) return;
    const std::int64_t r = 32 * w + lane;
    std::int64_t len = r < n ? row_ptr[r + 1] - row_ptr[r] : 0;
    for (int o = 16; o > 0; o >>= 1) len = max(len, __shfl_xor_sync(0xffffffffu, len, o));
    if (lane == 0) slice_len[w] = len;
}

// one thread per stored block: copy it into its (slice, slot, lane) position
__global__ void k_sell_fill(std::int32_t n, std::int64_t U, const std::uint32_t* __restrict__ rows,
                            const std::uint32_t* __restrict__ cols, const double* __restrict__ blocks,
                            const std::int64_t* __restrict__ row_ptr, const std::int64_t* __restrict__ slice_off,
                            const std::int32_t* __restrict__ perm, std::uint32_t* __restrict__ scol,
                            double* __restrict__ svals) {
    for (std::int64_t e = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; e < U;
         e += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        const std::uint32_t r = rows[e];
        const std::int64_t s = e - row_ptr[r];
        const std::int64_t slot = slice_off[r >> 5] + s;
        const int lane = r & 31;
        const std::uint32_t c = cols[e];
        scol[slot * 32 + lane] = perm ? static_cast<std::uint32_t>(perm[c]) : c;
#pragma unroll
        for (int k = 0; k < 9; ++k) svals[slot * 288 + 32 * k + lane] = blocks[blk(e, k)];
    }
}

__global__ void k_sell_rows(std::int32_t n, std::int32_t n_slices, const std::int32_t* __restrict__ perm,
                            std::int32_t* __restrict__ row_id) {
    for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x;
         i < 32 * static_cast<std::int64_t>(n_slices); i += static_cast<std::int64_t>(gridDim.x) * blockDim.x)
        row_id[i] = i < n ? (perm ? perm[i] : static_cast<std::int32_t>(i)) : -1;
}

// y (+)= A x; warp w owns a contiguous run of slices, lane = row.
template <bool kDot>
__global__ void __launch_bounds__(256) k_spmv_sell(std::int32_t n_slices, const std::int64_t* __restrict__ slice_off,
                                                  const std::int32_t* __restrict__ row_id,
                                                  const std::uint32_t* __restrict__ scol,
                                                  const double* __restrict__ svals, const double* __restrict__ x,
                                                  double* __restrict__ y, double* __restrict__ partials,
                                                  unsigned* __restrict__ ticket, double* __restrict__ dot_out,
                                                  const int* __restrict__ flags) {
    if (flags && flags[F_DONE]) return;
    const int lane = threadIdx.x & 31;
    const std::int64_t w = (static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const std::int64_t nw = (static_cast<std::int64_t>(gridDim.x) * blockDim.x) >> 5;
    const std::int64_t s0 = w * n_slices / nw, s1 = (w + 1) * n_slices / nw;
    double dsum = 0;
    for (std::int64_t S = s0; S < s1; ++S) {
        const std::int32_t r = row_id[32 * S + lane];
        const std::int64_t o0 = slice_off[S], o1 = slice_off[S + 1];
        double xr0 = 0, xr1 = 0, xr2 = 0;
        if (r >= 0) {
            xr0 = ldg_issue(x + 3 * static_cast<std::int64_t>(r));
            xr1 = ldg_issue(x + 3 * static_cast<std::int64_t>(r) + 1);
            xr2 = ldg_issue(x + 3 * static_cast<std::int64_t>(r) + 2);
        }
        double a0 = 0, a1 = 0, a2 = 0;
#pragma unroll 2
        for (std::int64_t slot = o0; slot < o1; ++slot) {
            const std::uint32_t c = __ldg(scol + slot * 32 + lane);
            if (c == kPad) continue;
            double h[9];
#pragma unroll
            for (int k = 0; k < 9; ++k) h[k] = __ldg(svals + slot * 288 + 32 * k + lane);
            const double xc0 = __ldg(x + 3 * static_cast<std::int64_t>(c));
            const double xc1 = __ldg(x + 3 * static_cast<std::int64_t>(c) + 1);
            const double xc2 = __ldg(x + 3 * static_cast<std::int64_t>(c) + 2);
            // column-major H(i,j) = h[3j+i]
            const double v0 = h[0] * xc0 + h[3] * xc1 + h[6] * xc2;
            const double v1 = h[1] * xc0 + h[4] * xc1 + h[7] * xc2;
            const double v2 = h[2] * xc0 + h[5] * xc1 + h[8] * xc2;
            a0 += v0;
            a1 += v1;
            a2 += v2;
            const bool off = c != static_cast<std::uint32_t>(r);
            if (off) {
                red_add(y + 3 * static_cast<std::int64_t>(c), h[0] * xr0 + h[1] * xr1 + h[2] * xr2);
                red_add(y + 3 * static_cast<std::int64_t>(c) + 1, h[3] * xr0 + h[4] * xr1 + h[5] * xr2);
                red_add(y + 3 * static_cast<std::int64_t>(c) + 2, h[6] * xr0 + h[7] * xr1 + h[8] * xr2);
            }
            if (kDot) dsum += (off ? 2.0 : 1.0) * (xr0 * v0 + xr1 * v1 + xr2 * v2);
        }
        if (r >= 0) {
            red_add(y + 3 * static_cast<std::int64_t>(r), a0);
            red_add(y + 3 * static_cast<std::int64_t>(r) + 1, a1);
            red_add(y + 3 * static_cast<std::int64_t>(r) + 2, a2);
        }
    }
    if (kDot) grid_sum_last_block(dsum, partials, ticket, dot_out, flags ? const_cast<int*>(flags) + F_K : nullptr);
}

}  // namespace

// (Re)build the sliced-ELL copy from the assembled (reference-numbered) A,
// with row / column ids in the solve order when it is active.
void build_sell(Ctx& c) {
    const DeviceMatrix& A = c.A;
    SellMatrix& M = c.sell;
    cudaStream_t st = c.stream;
    M.n = A.n;
    M.n_slices = static_cast<std::int32_t>(ceil_div(A.n, 32));
    M.slice_off.reserve(static_cast<std::size_t>(M.n_slices) + 1);
    c.sell_len.reserve(static_cast<std::size_t>(M.n_slices) + 1);
    if (M.n_slices > 0) {
        k_sell_len<<<grid_for(32 * static_cast<std::int64_t>(M.n_slices), 256, 64), 256, 0, st>>>(
            A.n, A.row_ptr.p, M.n_slices, c.sell_len.p);
        ADIPC_LAUNCH_CHECK();
    }
    exclusive_scan(c.sell_len.p, M.n_slices, M.slice_off.p, c.scan_scratch, st);
    std::int64_t slots = 0;
    ADIPC_CUDA(cudaMemcpyAsync(&slots, M.slice_off.p + M.n_slices, sizeof(slots), cudaMemcpyDeviceToHost, st));
    ADIPC_CUDA(cudaStreamSynchronize(st));
    M.slots = slots;
    M.cols.reserve(static_cast<std::size_t>(std::max<std::int64_t>(slots, 1)) * 32);
    M.vals.reserve(static_cast<std::size_t>(std::max<std::int64_t>(slots, 1)) * 288);
    M.row_id.reserve(32 * static_cast<std::size_t>(std::max(M.n_slices, 1)));
    const std::int32_t* perm = c.perm_active && !std::getenv("ADIPC_SELL_REF") ? c.perm.p : nullptr;  // env: experiments
    if (slots > 0) ADIPC_CUDA(cudaMemsetAsync(M.cols.p, 0xFF, sizeof(std::uint32_t) * 32 * slots, st));
    if (A.U > 0) {
        k_sell_fill<<<grid_for(A.U, 256, 16), 256, 0, st>>>(A.n, A.U, A.rows.p, A.cols.p, A.blocks.p, A.row_ptr.p,
                                                           M.slice_off.p, perm, M.cols.p, M.vals.p);
        ADIPC_LAUNCH_CHECK();
    }
    if (M.n_slices > 0) {
        k_sell_rows<<<grid_for(32 * static_cast<std::int64_t>(M.n_slices), 256, 8), 256, 0, st>>>(A.n, M.n_slices, perm,
                                                                                                 M.row_id.p);
        ADIPC_LAUNCH_CHECK();
    }
    M.a_version = A.version;
    M.perm_active = c.perm_active;
    M.levels_version = c.levels_version;
}

bool sell_current(const Ctx& c) {
    const SellMatrix& M = c.sell;
    return M.a_version == c.A.version && M.perm_active == c.perm_active &&
           (!c.perm_active || M.levels_version == c.levels_version) && M.n == c.A.n;
}

void sell_spmv_launch(Ctx& c, const double* d_x, double* d_y, const int* flags, double* partials, unsigned* ticket,
                      double* dot_out) {
    const SellMatrix& M = c.sell;
    if (M.n_slices == 0) {
        if (dot_out) ADIPC_CUDA(cudaMemsetAsync(dot_out, 0, sizeof(double), c.stream));
        return;
    }
    static int occ = 0;
    if (occ == 0) {
        ADIPC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_spmv_sell<true>, 256, 0));
        occ = std::max(occ, 1);
    }
    int sms = kSMs;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c.device);
    const int grid = static_cast<int>(std::max<std::int64_t>(
        1, std::min<std::int64_t>(static_cast<std::int64_t>(sms) * std::min(occ, 8), ceil_div(M.n_slices, 8))));
    if (dot_out)
        k_spmv_sell<true><<<grid, 256, 0, c.stream>>>(M.n_slices, M.slice_off.p, M.row_id.p, M.cols.p, M.vals.p, d_x,
                                                      d_y, partials, ticket, dot_out, flags);
    else
        k_spmv_sell<false><<<grid, 256, 0, c.stream>>>(M.n_slices, M.slice_off.p, M.row_id.p, M.cols.p, M.vals.p, d_x,
                                                       d_y, nullptr, nullptr, nullptr, flags);
    ADIPC_LAUNCH_CHECK();
}

}  // namespace adipc_gpu
