// MAS / block-Jacobi apply kernels, shared by the stand-alone preconditioner
// apply (mas.hpp:85-99 / block_jacobi.hpp:16-22) and the fused PCG iteration
// (pcg.hpp:59-85), which runs them in its "update" modes.
//
// MAS apply as a restriction tree. The reference restricts r onto every level
// directly from the slots (b[pos] += r[slot], mas.hpp:92-93). The hierarchy
// nests: every level-(l+1) node is a connected piece of ONE level-l
// subdomain, and the ids of the level-(l+1) nodes of subdomain s are
// consecutive (hierarchy.hpp:53-72 visits subdomains in order). So the warp
// that handles level-l subdomain s already holds b_l for all the children of
// its level-(l+1) nodes and emits r_{l+1} for them — one small parallel launch
// per level, no long per-lane loops over slots. Summation order is a tree
// instead of the reference's slot order (rounding-level difference).
//
// Subdomain inverses are stored symmetric-packed (packed_idx, common.cuh) and
// staged into shared memory with streaming 16-byte loads issued before the
// residual gather, so the two overlap. (These generic level kernels serve the
// stand-alone apply, the PCG start and the reference-numbering path; the
// solve-order PCG iteration uses k_precond_so, solve_order.cu.)
#pragma once

#include "context.hpp"
#include "tma.cuh"

namespace adipc_gpu {

constexpr int kMaxLevels = 8;

// Device scalars / flags of one PCG solve (PcgWork::scal / flags).
enum Scal : int {
    S_RHO0 = 0,      // rho at iteration k lives in S_RHO0 + (k & 1)
    S_RHO_INIT = 2,  // rho_0 (r0 . z0)
    S_STOP = 3,      // tol^2 * rho_0
    S_PAP = 4,       // p . A p of the current iteration
    S_REL = 5,       // rel_residual result
    S_BB = 6,        // b . b
    S_RZ = 8,        // S_RZ + l: level-l share of r . z (Jacobi: level 0)
    S_COUNT = S_RZ + kMaxLevels
};
// F_K: index (1-based) of the current iteration; advanced by the last CTA of
// the iteration's first kernel (the p.Ap SpMV), so an iteration's launch
// sequence is identical every time (captured once as a CUDA graph).
// F_ERR: an in-kernel dependency wait timed out (never expected; reported
// as a CUDA-class error instead of hanging the device)
enum Flag : int { F_DONE = 0, F_ITERS = 1, F_CONVERGED = 2, F_K = 3, F_KTICKET = 4, F_ERR = 5, F_COUNT = 8 };
// last-block tickets / partial arrays: 0 spmv, 1 b.b, 2 + l level l
enum Ticket : int { T_SPMV = 0, T_BB = 1, T_LEVEL = 2, T_COUNT = T_LEVEL + kMaxLevels };

// Gather modes of the level-0 / Jacobi kernels.
enum ApplyMode : int {
    M_APPLY = 0,    // b = r (given), z <- y
    M_INIT = 1,     // PCG start: r = b, x = 0, then as APPLY
    M_UPDATE = 2,   // PCG step: x += a p, r -= a Ap, then as APPLY
    M_RESTART = 3,  // PCG restart step: x already updated, r = b - tmp
    M_COARSE = 4,   // level >= 1: b = r_l[node] (restricted by the level below)
};

struct PcgArgs {
    double* x;
    double* r;
    const double* p;
    const double* ap;   // A p  (or A x in restart mode)
    const double* b;
    double* scal;
    int* flags;         // F_* (the current iteration index is flags[F_K])
};

// One level of the hierarchy as the apply kernels see it.
struct LevelArgs {
    std::int32_t n_parts;
    const std::int32_t* sub_ptr;    // subdomain -> first member node
    const std::int32_t* sub_nodes;  // members (level 0: slots), ascending
    const std::int64_t* inv_off;    // packed-inverse offsets (16-byte aligned)
    const double* inv;              // packed explicit inverses
    const double* r_in;             // M_COARSE: restricted residual per node (3 per node)
    double* out;                    // level 0: z per slot; coarse: y per node
    // restriction to the next level (null at the top level)
    const std::int32_t* up_first;   // subdomain -> first next-level node inside it
    const std::int32_t* upc_ptr;    // next-level node -> children range
    const std::int32_t* upc_pos;    // children as positions inside the subdomain
    double* r_next;                 // next level's restricted residual (3 per node)
};

// alpha of iteration k; returns false (and records the termination like
// pcg.hpp:61-66) when p.Ap lost positivity. All CTAs see the same scalars.
__device__ __forceinline__ bool pcg_alpha(const PcgArgs& a, double& alpha) {
    const int k = a.flags[F_K];
    const double rho = a.scal[S_RHO0 + ((k - 1) & 1)];
    const double pap = a.scal[S_PAP];
    if (!(pap > 0)) {
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            a.flags[F_DONE] = 1;
            a.flags[F_ITERS] = k - 1;
            a.scal[S_REL] = sqrt(fabs(rho) / a.scal[S_RHO_INIT]);
        }
        return false;
    }
    alpha = rho / pap;
    return true;
}

// Residual value of dof g under the gather mode (fusing the PCG vector update
// for the slots the level-0 partition owns — each slot exactly once).
template <int kMode>
__device__ __forceinline__ double gather_r(const PcgArgs& a, const double* r_in, std::int64_t g, double alpha) {
    if (kMode == M_APPLY || kMode == M_COARSE) return r_in[g];
    if (kMode == M_INIT) {
        const double rv = a.b[g];
        a.r[g] = rv;
        a.x[g] = 0.0;
        return rv;
    }
    if (kMode == M_UPDATE) {
        a.x[g] += alpha * a.p[g];
        const double rv = a.r[g] - alpha * a.ap[g];
        a.r[g] = rv;
        return rv;
    }
    const double rv = a.b[g] - a.ap[g];  // M_RESTART (x updated before the restart SpMV)
    a.r[g] = rv;
    return rv;
}

constexpr int kLevelWarps = 4;  // warps (= subdomains) per CTA of the level kernels

// y = D^-1 b for one subdomain, D^-1 symmetric-packed in shared memory (upper
// triangle by columns: D(j,k) at k(k+1)/2 + j for j <= k, packed_idx). Lane j
// holds rows j + 32 t (t < R) in b[t] / y[t]. Fully unrolled over kK >= dim
// columns, so D(j,k) is a shared load at a compile-time offset: k(k+1)/2 from
// M + j when j <= k, k from M + j(j+1)/2 when j > k — per column one
// broadcast of b_k, at most two shared loads and one FMA per row (two
// accumulation chains for ILP). Columns k >= dim need b_k = 0 and finite slot
// contents up to packed_doubles(kK); rows j >= dim come out as garbage.
template <int kK>
__device__ __forceinline__ void packed_matvec(const double* M, const double* b, double* y, int lane) {
    constexpr int R = (kK + 31) / 32;
    const double* P1[R];
    const double* P2[R];
#pragma unroll
    for (int t = 0; t < R; ++t) {
        const int j = min(lane + 32 * t, kK - 1);
        P1[t] = M + j;
        P2[t] = M + j * (j + 1) / 2;
    }
    double acc0[R], acc1[R];
#pragma unroll
    for (int t = 0; t < R; ++t) acc0[t] = acc1[t] = 0.0;
#pragma unroll
    for (int k = 0; k < kK; ++k) {
        const double bk = __shfl_sync(0xffffffffu, b[k >> 5], k & 31);
        const int ck = k * (k + 1) / 2;
#pragma unroll
        for (int t = 0; t < R; ++t) {
            double m;
            if (32 * t + 31 <= k)
                m = P1[t][ck];
            else if (32 * t > k)
                m = P2[t][k];
            else
                m = (lane + 32 * t <= k) ? P1[t][ck] : P2[t][k];
            if (k & 1)
                acc1[t] = fma(m, bk, acc1[t]);
            else
                acc0[t] = fma(m, bk, acc0[t]);
        }
    }
#pragma unroll
    for (int t = 0; t < R; ++t) y[t] = acc0[t] + acc1[t];
}

// Row handled by `lane` in register slot t of packed_matvec_rows. Rows are
// lane + 32 t from kRow0, except that for kK = 48 the upper half (rows 24..47)
// puts rows 32..47 on lanes 0..15: the transposed reads D(j,k) = P[j(j+1)/2
// + k] of a half-warp then fall in 16 distinct banks (j(j+1)/2 mod 16 is a
// permutation of 0..15 over every 16-aligned run of rows).
template <int kK, int kRow0>
__device__ __forceinline__ int matvec_row(int lane, int t) {
    if (kK == 48 && kRow0 == 24 && t == 0) return lane < 16 ? 32 + lane : 8 + lane;
    return kRow0 + lane + 32 * t;
}

// Rows [kRow0, kRow0 + kRows) of y = D^-1 b (lane i holds row
// matvec_row(i, t) in y[t]); b read from shared memory (bs, 16-byte aligned,
// kK entries, b_k = 0 for k >= dim) two entries per 128-bit broadcast load.
// Per column: all rows <= k read column k at a compile-time offset, all rows
// > k their own column, and mixed columns select the offset per lane — one
// shared load per row and column.
// independent FMA chains per row in packed_matvec_rows: 4 measured best at
// cfg5 (preconditioner 66 -> 61 us; 6: 61.7, 8: 62.0)
#ifndef ADIPC_PC_ACC
#define ADIPC_PC_ACC 4
#endif
template <int kK, int kRow0, int kRows>
__device__ __forceinline__ void packed_matvec_rows(const double* M, const double* bs, double* y, int lane) {
    constexpr int R = (kRows + 31) / 32;
    int jr[R];
    const double* P1[R];
    const double* P2[R];
#pragma unroll
    for (int t = 0; t < R; ++t) {
        jr[t] = matvec_row<kK, kRow0>(lane, t);
        const int j = min(jr[t], kK - 1);
        P1[t] = M + j;
        P2[t] = M + j * (j + 1) / 2;
    }
    // kAcc independent accumulation chains per row (fp64 FMA latency)
    constexpr int kAcc = ADIPC_PC_ACC;
    double acc[kAcc][R];
#pragma unroll
    for (int q = 0; q < kAcc; ++q)
#pragma unroll
        for (int t = 0; t < R; ++t) acc[q][t] = 0.0;
    const double2* b2 = reinterpret_cast<const double2*>(bs);
#pragma unroll
    for (int k2 = 0; k2 < kK; k2 += 2) {
        const double2 bb = b2[k2 >> 1];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int k = k2 + u;
            const double bk = u == 0 ? bb.x : bb.y;
            const int ck = k * (k + 1) / 2;
#pragma unroll
            for (int t = 0; t < R; ++t) {
                const int jlo = kRow0 + 32 * t;
                const int jhi = min(kRow0 + 32 * t + 31, kRow0 + kRows - 1);
                double m;
                if (jhi <= k)
                    m = P1[t][ck];
                else if (jlo > k)
                    m = P2[t][k];
                else
                    m = jr[t] <= k ? M[ck + jr[t]] : P2[t][k];
                acc[k % kAcc][t] = fma(m, bk, acc[k % kAcc][t]);
            }
        }
    }
#pragma unroll
    for (int t = 0; t < R; ++t) {
        double v = acc[0][t];
#pragma unroll
        for (int q = 1; q < kAcc; ++q) v += acc[q][t];
        y[t] = v;
    }
}

// One warp of a pair (half 0: rows [0, kK/2), half 1: the rest) solves its
// rows of a subdomain of dimension dim <= kK and hands each row j < dim to
// store(j, y_j); returns the warp's share of b.y. Small subdomains (coarse
// levels) take a shorter unrolled column loop.
template <int kK>
__device__ __forceinline__ int pick_cols(int dim) {
    if (kK >= 48 && dim <= 12) return 12;
    if (kK >= 48 && dim <= 24) return 24;
    return kK;
}

// kK = 48 splits the rows 32 / 16 (ADIPC_PC_SPLIT32): every shared load of
// warp 0 then serves 32 rows and warp 1's 16 rows take one wavefront, 3/4
// of the wavefronts of the 24 / 24 split whose loads each fed 24 of 32 lanes
#ifndef ADIPC_PC_SPLIT32
#define ADIPC_PC_SPLIT32 1
#endif
template <int kK>
__device__ __forceinline__ constexpr int pair_split() {
    return (kK == 48 && ADIPC_PC_SPLIT32) ? 32 : kK / 2;
}
template <int kK, class Store>
__device__ __forceinline__ double pair_rows_solve(const double* M, const double* bs, int lane, int half, int dim,
                                                  Store store) {
    constexpr int kS = pair_split<kK>();
    constexpr int RY = ((kS > kK - kS ? kS : kK - kS) + 31) / 32;
    double y[RY];
    if (half == 0)
        packed_matvec_rows<kK, 0, kS>(M, bs, y, lane);
    else
        packed_matvec_rows<kK, kS, kK - kS>(M, bs, y, lane);
    const int rows = half == 0 ? kS : kK - kS;
    double dsum = 0;
#pragma unroll
    for (int t = 0; t < RY; ++t) {
        const int i = lane + 32 * t;
        const int j = half == 0 ? matvec_row<kK, 0>(lane, t) : matvec_row<kK, kS>(lane, t);
        if (i < rows && j < dim) {
            store(j, y[t]);
            dsum += bs[j] * y[t];
        }
    }
    return dsum;
}

template <int kK, class Store>
__device__ __forceinline__ double pair_solve(const double* M, const double* bs, int lane, int half, int dim,
                                             Store store) {
    const int kc = pick_cols<kK>(dim);
    if (kK >= 48 && kc == 12) return pair_rows_solve<12>(M, bs, lane, half, dim, store);
    if (kK >= 48 && kc == 24) return pair_rows_solve<24>(M, bs, lane, half, dim, store);
    return pair_rows_solve<kK>(M, bs, lane, half, dim, store);
}

// Half-warp mat-vec: the 16 lanes of half-warp h solve one subdomain, lane i
// holding rows i + 16 t (t < kK/16). Every shared load of a column then
// serves both half-warps' subdomains with one full 256-byte access, and a
// 16-aligned run of rows reads its own columns D(j,k) = P[j(j+1)/2 + k] in 16
// distinct banks. b from bs (this half's copy), two entries per 128-bit load.
template <int kK>
__device__ __forceinline__ void packed_matvec_half(const double* M, const double* bs, double* y, int hl) {
    constexpr int T = (kK + 15) / 16;
    const double* P1[T];
    const double* P2[T];
#pragma unroll
    for (int t = 0; t < T; ++t) {
        const int j = min(hl + 16 * t, kK - 1);
        P1[t] = M + j;
        P2[t] = M + j * (j + 1) / 2;
    }
    double acc0[T], acc1[T];
#pragma unroll
    for (int t = 0; t < T; ++t) acc0[t] = acc1[t] = 0.0;
    const double2* b2 = reinterpret_cast<const double2*>(bs);
#pragma unroll
    for (int k2 = 0; k2 < kK; k2 += 2) {
        const double2 bb = b2[k2 >> 1];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int k = k2 + u;
            const double bk = u == 0 ? bb.x : bb.y;
            const int ck = k * (k + 1) / 2;
#pragma unroll
            for (int t = 0; t < T; ++t) {
                double m;
                if (16 * t + 15 <= k)
                    m = P1[t][ck];
                else if (16 * t > k)
                    m = P2[t][k];
                else
                    m = hl + 16 * t <= k ? P1[t][ck] : P2[t][k];
                if (u == 1)
                    acc1[t] = fma(m, bk, acc1[t]);
                else
                    acc0[t] = fma(m, bk, acc0[t]);
            }
        }
    }
#pragma unroll
    for (int t = 0; t < T; ++t) y[t] = acc0[t] + acc1[t];
}

// column bound of packed_matvec for subdomains of at most max_fill nodes
inline int matvec_cols(int max_fill) { return max_fill <= 8 ? 24 : (max_fill <= 16 ? 48 : (max_fill <= 32 ? 96 : 0)); }

// Bytes of dynamic shared memory per warp of k_mas_level for a level whose
// largest subdomain has dimension max_dim: packed inverse + b + mbarrier.
inline std::size_t level_warp_smem(int max_dim, int regs) {
    const std::size_t inv = static_cast<std::size_t>(packed_doubles(max_dim)) * 8;
    return ((inv + static_cast<std::size_t>(32 * regs) * 8 + 16 + 15) / 16) * 16;
}

// One warp per subdomain (dim = 3 f <= 32 kRegs), kLevelWarps per CTA:
//   the warp stages the packed inverse into its smem slot (kSolve), gathers b
//   (with the fused PCG vector update for level 0), then y = D^-1 b from
//   smem (lane j owns rows j, j+32, ...),
//   stores y, emits the next level's restricted residual, dot partial b.y.
// kSolve = false: gather (with the fused PCG vector update) + restriction
// only — the PCG's update pass, after which the level-0 solve and the coarse
// chain run concurrently.
template <int kMode, int kRegs, bool kSolve = true>
__global__ void __launch_bounds__(32 * kLevelWarps) k_mas_level(LevelArgs L, PcgArgs a, double* __restrict__ partials,
                                                                unsigned* __restrict__ ticket,
                                                                double* __restrict__ dot_out, int warp_smem) {
    extern __shared__ __align__(128) unsigned char smem[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    double* Mw = reinterpret_cast<double*>(smem + static_cast<std::size_t>(w) * warp_smem);
    double* bw = reinterpret_cast<double*>(smem + static_cast<std::size_t>(w + 1) * warp_smem) - 32 * kRegs - 2;
    double alpha = 0;
    if (a.flags && a.flags[F_DONE]) return;
    if ((kMode == M_UPDATE || kMode == M_RESTART) && !pcg_alpha(a, alpha)) return;
    double dsum = 0;
    const std::int32_t s = blockIdx.x * kLevelWarps + w;
    if (s < L.n_parts) {
        const std::int32_t s0 = L.sub_ptr[s];
        const int dim = 3 * (L.sub_ptr[s + 1] - s0);
        if (kSolve) {  // stage the packed inverse (16-byte loads, in flight during the gather)
            const double2* src = reinterpret_cast<const double2*>(L.inv + L.inv_off[s]);
            double2* dst = reinterpret_cast<double2*>(Mw);
            const int n2 = static_cast<int>(packed_doubles(dim) / 2);
            for (int i = lane; i < n2; i += 32) dst[i] = __ldcs(src + i);
        }
        double b[kRegs], y[kRegs];
        std::int64_t gi[kRegs];
#pragma unroll
        for (int t = 0; t < kRegs; ++t) {
            const int j = lane + 32 * t;
            b[t] = 0;
            y[t] = 0;
            gi[t] = -1;
            if (j < dim) {
                gi[t] = 3 * static_cast<std::int64_t>(L.sub_nodes[s0 + j / 3]) + (j % 3);
                b[t] = gather_r<kMode>(a, L.r_in, gi[t], alpha);
            }
        }
#pragma unroll
        for (int t = 0; t < kRegs; ++t) bw[lane + 32 * t] = b[t];
        __syncwarp();
        if (kSolve) {
            // y_j = sum_k D^-1(j, k) b_k over the packed upper triangle:
            // k >= j reads column k (contiguous across lanes), k < j reads
            // column j (triangular-number offsets: distinct banks per half-warp)
            for (int k = 0; k < dim; ++k) {
                const double bk = bw[k];
                const int ck = k * (k + 1) / 2;
#pragma unroll
                for (int t = 0; t < kRegs; ++t) {
                    const int j = lane + 32 * t;
                    if (j < dim) y[t] += Mw[j <= k ? ck + j : j * (j + 1) / 2 + k] * bk;
                }
            }
#pragma unroll
            for (int t = 0; t < kRegs; ++t)
                if (gi[t] >= 0) {
                    L.out[gi[t]] = y[t];
                    dsum += b[t] * y[t];
                }
        }
        if (L.r_next) {  // restriction to the nested next-level nodes
            const std::int32_t v0 = L.up_first[s];
            const int nv3 = 3 * (L.up_first[s + 1] - v0);
            for (int t = lane; t < nv3; t += 32) {
                const std::int32_t v = v0 + t / 3;
                const int comp = t % 3;
                double acc = 0;
                for (std::int32_t q = L.upc_ptr[v]; q < L.upc_ptr[v + 1]; ++q) acc += bw[3 * L.upc_pos[q] + comp];
                L.r_next[3 * static_cast<std::int64_t>(v) + comp] = acc;
            }
        }
    }
    if (dot_out) grid_sum_last_block(dsum, partials, ticket, dot_out);
}

// General-size variant (fill > 32, e.g. the exact single-domain
// preconditioner of test_solver.cpp:99-111): one CTA per subdomain, b in
// dynamic shared memory, packed inverse read from global, any dim.
template <int kMode, bool kSolve = true>
__global__ void __launch_bounds__(128) k_mas_level_big(LevelArgs L, PcgArgs a, double* __restrict__ partials,
                                                      unsigned* __restrict__ ticket, double* __restrict__ dot_out) {
    extern __shared__ double bs[];
    double alpha = 0;
    if (a.flags && a.flags[F_DONE]) return;
    if ((kMode == M_UPDATE || kMode == M_RESTART) && !pcg_alpha(a, alpha)) return;
    double dsum = 0;
    for (std::int32_t s = blockIdx.x; s < L.n_parts; s += gridDim.x) {
        const std::int32_t s0 = L.sub_ptr[s];
        const int dim = 3 * (L.sub_ptr[s + 1] - s0);
        for (int j = threadIdx.x; j < dim; j += blockDim.x)
            bs[j] = gather_r<kMode>(a, L.r_in, 3 * static_cast<std::int64_t>(L.sub_nodes[s0 + j / 3]) + (j % 3), alpha);
        __syncthreads();
        const double* M = L.inv + L.inv_off[s];
        for (int j = threadIdx.x; kSolve && j < dim; j += blockDim.x) {
            double y = 0;
            for (int k = 0; k < dim; ++k) y += M[packed_idx(j, k)] * bs[k];
            L.out[3 * static_cast<std::int64_t>(L.sub_nodes[s0 + j / 3]) + (j % 3)] = y;
            dsum += bs[j] * y;
        }
        if (L.r_next) {
            const std::int32_t v0 = L.up_first[s];
            const int nv3 = 3 * (L.up_first[s + 1] - v0);
            for (int t = threadIdx.x; t < nv3; t += blockDim.x) {
                const std::int32_t v = v0 + t / 3;
                const int comp = t % 3;
                double acc = 0;
                for (std::int32_t q = L.upc_ptr[v]; q < L.upc_ptr[v + 1]; ++q) acc += bs[3 * L.upc_pos[q] + comp];
                L.r_next[3 * static_cast<std::int64_t>(v) + comp] = acc;
            }
        }
        __syncthreads();
    }
    if (dot_out) grid_sum_last_block(dsum, partials, ticket, dot_out);
}

// Prolongation z[slot] = ((y0 + y1[agg1]) + y2[agg2]) + ... (mas.hpp:95-96
// order), then either stores z (apply) or finishes the PCG step:
// rho' = r.z; converged -> stop; else p = z + (rho'/rho) p (pcg.hpp:76-84);
// Ap is cleared for the next SpMV in the same pass.
struct ProlongArgs {
    int n_levels;  // coarse levels
    int n_rz;      // number of r.z shares to add (levels, or 1 for Jacobi)
    const std::int32_t* agg[kMaxLevels];
    const double* y[kMaxLevels];
};

enum FinalMode : int { F_APPLY = 0, F_PCG_INIT = 1, F_PCG_STEP = 2 };

template <int kFinal>
__global__ void __launch_bounds__(256) k_mas_final(std::int32_t n, ProlongArgs pa, double* __restrict__ z,
                                                  double* __restrict__ p, double* __restrict__ ap, PcgArgs a) {
    double beta = 0;
    bool write_p = false;
    if (kFinal != F_APPLY) {
        if (a.flags[F_DONE]) return;
        double rz = 0;
        for (int l = 0; l < pa.n_rz; ++l) rz += a.scal[S_RZ + l];
        if (kFinal == F_PCG_INIT) {
            // pcg.hpp:52-57: rho0 = r.z; fail if !(rho0 > 0)
            if (blockIdx.x == 0 && threadIdx.x == 0) {
                a.scal[S_RHO0] = rz;
                a.scal[S_RHO_INIT] = rz;
                a.scal[S_STOP] = a.scal[S_STOP] * rz;  // S_STOP preloaded with tol^2
                if (!(rz > 0)) {
                    a.flags[F_DONE] = 1;
                    a.flags[F_ITERS] = 0;
                    a.scal[S_REL] = 0;
                }
            }
            write_p = rz > 0;
        } else {
            const int k = a.flags[F_K];
            const double rho = a.scal[S_RHO0 + ((k - 1) & 1)];
            const double stop = a.scal[S_STOP];
            if (blockIdx.x == 0 && threadIdx.x == 0) {
                a.flags[F_ITERS] = k;
                a.scal[S_REL] = sqrt(fabs(rz) / a.scal[S_RHO_INIT]);
                if (rz <= stop) {
                    a.flags[F_DONE] = 1;
                    a.flags[F_CONVERGED] = 1;
                } else {
                    a.scal[S_RHO0 + (k & 1)] = rz;
                }
            }
            if (rz <= stop) return;
            beta = rz / rho;
            write_p = true;
        }
    }
    const std::int64_t n3 = 3 * static_cast<std::int64_t>(n);
    for (std::int64_t g = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; g < n3;
         g += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        const std::int64_t slot = g / 3;
        const int comp = static_cast<int>(g - 3 * slot);
        double zz = z[g];
        for (int l = 0; l < pa.n_levels; ++l) zz += pa.y[l][3 * static_cast<std::int64_t>(pa.agg[l][slot]) + comp];
        if (kFinal == F_APPLY) {
            z[g] = zz;
        } else if (write_p) {
            p[g] = (kFinal == F_PCG_INIT) ? zz : zz + beta * p[g];
            ap[g] = 0.0;
        }
    }
}

// Block Jacobi (block_jacobi.hpp:16-22), one thread per slot, with the same
// PCG modes as the level-0 MAS kernel. z = inv[i] r_i.
template <int kMode>
__global__ void __launch_bounds__(256) k_jacobi(std::int32_t n, const double* __restrict__ jinv,
                                               const double* __restrict__ r_in, double* __restrict__ z, PcgArgs a,
                                               double* __restrict__ partials, unsigned* __restrict__ ticket,
                                               double* __restrict__ dot_out) {
    double alpha = 0;
    if (kMode == M_UPDATE || kMode == M_RESTART) {
        if (a.flags[F_DONE]) return;
        if (!pcg_alpha(a, alpha)) return;
    }
    double dsum = 0;
    for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        double rv[3];
        for (int k = 0; k < 3; ++k) rv[k] = gather_r<kMode>(a, r_in, 3 * i + k, alpha);
        const double* M = jinv + 9 * i;
        for (int k = 0; k < 3; ++k) {
            const double zk = M[k] * rv[0] + M[3 + k] * rv[1] + M[6 + k] * rv[2];
            z[3 * i + k] = zk;
            dsum += rv[k] * zk;
        }
    }
    if (dot_out) grid_sum_last_block(dsum, partials, ticket, dot_out);
}

}  // namespace adipc_gpu
