// MAS / block-Jacobi apply kernels, shared by the stand-alone preconditioner
// apply (mas.hpp:85-99 / block_jacobi.hpp:16-22) and the fused PCG iteration
// (pcg.hpp:59-85), which runs them in its "update" modes.
#pragma once

#include "context.hpp"

namespace adipc_gpu {

// Device scalars / flags of one PCG solve (PcgWork::scal / flags).
enum Scal : int {
    S_RHO0 = 0,      // rho at iteration k lives in S_RHO0 + (k & 1)
    S_RHO_INIT = 2,  // rho_0 (r0 . z0)
    S_STOP = 3,      // tol^2 * rho_0
    S_PAP = 4,       // p . A p of the current iteration
    S_RZ_L0 = 5,     // level-0 (or Jacobi) share of r . z
    S_RZ_C = 6,      // coarse-level share of r . z
    S_REL = 7,       // rel_residual result
    S_BB = 8,        // b . b
    S_COUNT = 16
};
enum Flag : int { F_DONE = 0, F_ITERS = 1, F_CONVERGED = 2, F_COUNT = 8 };
enum Ticket : int { T_SPMV = 0, T_L0 = 1, T_C = 2, T_BB = 3, T_COUNT = 8 };

// Apply modes of the level-0 / Jacobi kernel.
enum ApplyMode : int {
    M_APPLY = 0,    // b = r (given), z <- y
    M_INIT = 1,     // PCG start: r = b, x = 0, then as APPLY
    M_UPDATE = 2,   // PCG step: x += a p, r -= a Ap, then as APPLY
    M_RESTART = 3,  // PCG restart step: x already updated, r = b - tmp
};

struct PcgArgs {
    double* x;
    double* r;
    const double* p;
    const double* ap;   // A p  (or A x in restart mode)
    const double* b;
    double* scal;
    int* flags;
    int k;              // iteration index (1-based), 0 in init
};

// alpha of iteration k; returns false (and records the termination like
// pcg.hpp:61-66) when p.Ap lost positivity. All CTAs see the same scalars.
__device__ __forceinline__ bool pcg_alpha(const PcgArgs& a, double& alpha) {
    const double rho = a.scal[S_RHO0 + ((a.k - 1) & 1)];
    const double pap = a.scal[S_PAP];
    if (!(pap > 0)) {
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            a.flags[F_DONE] = 1;
            a.flags[F_ITERS] = a.k - 1;
            a.scal[S_REL] = sqrt(fabs(rho) / a.scal[S_RHO_INIT]);
        }
        return false;
    }
    alpha = rho / pap;
    return true;
}

// Level-0 subdomain solve, one warp per subdomain: gather b (fusing the PCG
// vector update for the slots this subdomain owns — the level-0 partition
// owns every slot exactly once), y = D^-1 b with the explicit inverse read
// column by column (coalesced), z[slot] = y, dot partial b.y.
template <int kMode, int kMaxDimRegs>
__global__ void __launch_bounds__(256) k_mas_l0(std::int32_t n_parts, const std::int32_t* __restrict__ sub_ptr,
                                               const std::int32_t* __restrict__ slots,
                                               const std::int64_t* __restrict__ inv_off,
                                               const double* __restrict__ inv, const double* __restrict__ r_in,
                                               double* __restrict__ z, PcgArgs a, double* __restrict__ partials,
                                               unsigned* __restrict__ ticket, double* __restrict__ dot_out) {
    const int lane = threadIdx.x & 31;
    double alpha = 0;
    if (kMode == M_UPDATE || kMode == M_RESTART) {
        if (a.flags[F_DONE]) return;
        if (!pcg_alpha(a, alpha)) return;
    }
    double dsum = 0;
    const int wpb = blockDim.x >> 5;
    for (std::int32_t s = blockIdx.x * wpb + (threadIdx.x >> 5); s < n_parts; s += gridDim.x * wpb) {
        const std::int32_t s0 = sub_ptr[s];
        const int dim = 3 * (sub_ptr[s + 1] - s0);
        double b[kMaxDimRegs], y[kMaxDimRegs];
        std::int64_t gi[kMaxDimRegs];
#pragma unroll
        for (int t = 0; t < kMaxDimRegs; ++t) {
            const int j = lane + 32 * t;
            b[t] = 0;
            y[t] = 0;
            gi[t] = -1;
            if (j < dim) {
                const std::int32_t slot = slots[s0 + j / 3];
                const std::int64_t g = 3 * static_cast<std::int64_t>(slot) + (j % 3);
                gi[t] = g;
                double rv;
                if (kMode == M_APPLY) {
                    rv = r_in[g];
                } else if (kMode == M_INIT) {
                    rv = a.b[g];
                    a.r[g] = rv;
                    a.x[g] = 0.0;
                } else if (kMode == M_UPDATE) {
                    a.x[g] += alpha * a.p[g];
                    rv = a.r[g] - alpha * a.ap[g];
                    a.r[g] = rv;
                } else {  // M_RESTART: x was updated before the restart SpMV
                    rv = a.b[g] - a.ap[g];
                    a.r[g] = rv;
                }
                b[t] = rv;
            }
        }
        const double* M = inv + inv_off[s];
        for (int k = 0; k < dim; ++k) {
            const double bk = __shfl_sync(0xffffffffu, b[k >> 5], k & 31);
            const double* col = M + static_cast<std::int64_t>(k) * dim;
#pragma unroll
            for (int t = 0; t < kMaxDimRegs; ++t) {
                const int j = lane + 32 * t;
                if (j < dim) y[t] += __ldg(col + j) * bk;
            }
        }
#pragma unroll
        for (int t = 0; t < kMaxDimRegs; ++t)
            if (gi[t] >= 0) {
                z[gi[t]] = y[t];
                dsum += b[t] * y[t];
            }
    }
    if (dot_out) grid_sum_last_block(dsum, partials, ticket, dot_out);
}

// General-size variant (subdomain capacity > 32, e.g. the exact single-domain
// preconditioner of test_solver.cpp:99-111): one CTA per subdomain, b in
// shared memory (dim doubles, dynamic), any dim.
template <int kMode>
__global__ void __launch_bounds__(128) k_mas_l0_big(std::int32_t n_parts, const std::int32_t* __restrict__ sub_ptr,
                                                   const std::int32_t* __restrict__ slots,
                                                   const std::int64_t* __restrict__ inv_off,
                                                   const double* __restrict__ inv, const double* __restrict__ r_in,
                                                   double* __restrict__ z, PcgArgs a, double* __restrict__ partials,
                                                   unsigned* __restrict__ ticket, double* __restrict__ dot_out) {
    extern __shared__ double bs[];
    double alpha = 0;
    if (kMode == M_UPDATE || kMode == M_RESTART) {
        if (a.flags[F_DONE]) return;
        if (!pcg_alpha(a, alpha)) return;
    }
    double dsum = 0;
    for (std::int32_t s = blockIdx.x; s < n_parts; s += gridDim.x) {
        const std::int32_t s0 = sub_ptr[s];
        const int dim = 3 * (sub_ptr[s + 1] - s0);
        for (int j = threadIdx.x; j < dim; j += blockDim.x) {
            const std::int64_t g = 3 * static_cast<std::int64_t>(slots[s0 + j / 3]) + (j % 3);
            double rv;
            if (kMode == M_APPLY) {
                rv = r_in[g];
            } else if (kMode == M_INIT) {
                rv = a.b[g];
                a.r[g] = rv;
                a.x[g] = 0.0;
            } else if (kMode == M_UPDATE) {
                a.x[g] += alpha * a.p[g];
                rv = a.r[g] - alpha * a.ap[g];
                a.r[g] = rv;
            } else {
                rv = a.b[g] - a.ap[g];
                a.r[g] = rv;
            }
            bs[j] = rv;
        }
        __syncthreads();
        const double* M = inv + inv_off[s];
        for (int j = threadIdx.x; j < dim; j += blockDim.x) {
            double y = 0;
            for (int k = 0; k < dim; ++k) y += M[static_cast<std::int64_t>(k) * dim + j] * bs[k];
            z[3 * static_cast<std::int64_t>(slots[s0 + j / 3]) + (j % 3)] = y;
            dsum += bs[j] * y;
        }
        __syncthreads();
    }
    if (dot_out) grid_sum_last_block(dsum, partials, ticket, dot_out);
}

// Coarse levels (>= 1), all levels in one launch: one warp per (level,
// subdomain). b[pos] = sum of r over the node's member slots in ascending
// slot order (the reference's accumulation order, mas.hpp:92-93), y = D^-1 b,
// y stored per node for the prolongation, dot partial b.y.
struct CoarseLevelArgs {
    std::int32_t n_parts;
    const std::int32_t* sub_ptr;
    const std::int32_t* sub_nodes;
    const std::int32_t* node_ptr;
    const std::int32_t* node_slots;
    const std::int64_t* inv_off;
    const double* inv;
    double* y;
};
constexpr int kMaxCoarse = 8;
struct CoarseArgs {
    int n_levels;
    std::int32_t part_begin[kMaxCoarse + 1];  // prefix of n_parts over coarse levels
    CoarseLevelArgs lv[kMaxCoarse];
};

template <int kMaxDimRegs>
__global__ void __launch_bounds__(256) k_mas_coarse(CoarseArgs ca, const double* __restrict__ r, const int* __restrict__ flags,
                                                   double* __restrict__ partials, unsigned* __restrict__ ticket,
                                                   double* __restrict__ dot_out) {
    if (flags && flags[F_DONE]) return;
    const int lane = threadIdx.x & 31;
    const int wpb = blockDim.x >> 5;
    const std::int32_t total = ca.part_begin[ca.n_levels];
    double dsum = 0;
    for (std::int32_t gs = blockIdx.x * wpb + (threadIdx.x >> 5); gs < total; gs += gridDim.x * wpb) {
        int l = 0;
        while (gs >= ca.part_begin[l + 1]) ++l;
        const CoarseLevelArgs& L = ca.lv[l];
        const std::int32_t s = gs - ca.part_begin[l];
        const std::int32_t s0 = L.sub_ptr[s];
        const int dim = 3 * (L.sub_ptr[s + 1] - s0);
        double b[kMaxDimRegs], y[kMaxDimRegs];
#pragma unroll
        for (int t = 0; t < kMaxDimRegs; ++t) {
            const int j = lane + 32 * t;
            b[t] = 0;
            y[t] = 0;
            if (j < dim) {
                const std::int32_t node = L.sub_nodes[s0 + j / 3];
                const int comp = j % 3;
                double acc = 0;
                for (std::int32_t q = L.node_ptr[node]; q < L.node_ptr[node + 1]; ++q)
                    acc += __ldg(r + 3 * static_cast<std::int64_t>(L.node_slots[q]) + comp);
                b[t] = acc;
            }
        }
        const double* M = L.inv + L.inv_off[s];
        for (int k = 0; k < dim; ++k) {
            const double bk = __shfl_sync(0xffffffffu, b[k >> 5], k & 31);
            const double* col = M + static_cast<std::int64_t>(k) * dim;
#pragma unroll
            for (int t = 0; t < kMaxDimRegs; ++t) {
                const int j = lane + 32 * t;
                if (j < dim) y[t] += __ldg(col + j) * bk;
            }
        }
#pragma unroll
        for (int t = 0; t < kMaxDimRegs; ++t) {
            const int j = lane + 32 * t;
            if (j < dim) {
                const std::int32_t node = L.sub_nodes[s0 + j / 3];
                L.y[3 * static_cast<std::int64_t>(node) + (j % 3)] = y[t];
                dsum += b[t] * y[t];
            }
        }
    }
    if (dot_out) grid_sum_last_block(dsum, partials, ticket, dot_out);
}

// General-size coarse variant: one CTA per (level, subdomain), b in smem.
static __global__ void __launch_bounds__(128) k_mas_coarse_big(CoarseArgs ca, const double* __restrict__ r,
                                                       const int* __restrict__ flags, double* __restrict__ partials,
                                                       unsigned* __restrict__ ticket, double* __restrict__ dot_out) {
    extern __shared__ double bs[];
    if (flags && flags[F_DONE]) return;
    const std::int32_t total = ca.part_begin[ca.n_levels];
    double dsum = 0;
    for (std::int32_t gs = blockIdx.x; gs < total; gs += gridDim.x) {
        int l = 0;
        while (gs >= ca.part_begin[l + 1]) ++l;
        const CoarseLevelArgs& L = ca.lv[l];
        const std::int32_t s = gs - ca.part_begin[l];
        const std::int32_t s0 = L.sub_ptr[s];
        const int dim = 3 * (L.sub_ptr[s + 1] - s0);
        for (int j = threadIdx.x; j < dim; j += blockDim.x) {
            const std::int32_t node = L.sub_nodes[s0 + j / 3];
            double acc = 0;
            for (std::int32_t q = L.node_ptr[node]; q < L.node_ptr[node + 1]; ++q)
                acc += r[3 * static_cast<std::int64_t>(L.node_slots[q]) + (j % 3)];
            bs[j] = acc;
        }
        __syncthreads();
        const double* M = L.inv + L.inv_off[s];
        for (int j = threadIdx.x; j < dim; j += blockDim.x) {
            double y = 0;
            for (int k = 0; k < dim; ++k) y += M[static_cast<std::int64_t>(k) * dim + j] * bs[k];
            L.y[3 * static_cast<std::int64_t>(L.sub_nodes[s0 + j / 3]) + (j % 3)] = y;
            dsum += bs[j] * y;
        }
        __syncthreads();
    }
    if (dot_out) grid_sum_last_block(dsum, partials, ticket, dot_out);
}

// Prolongation z[slot] = ((y0 + y1[agg1]) + y2[agg2]) + ... (mas.hpp:95-96
// order), then either stores z (apply) or finishes the PCG step:
// rho' = r.z; converged -> stop; else p = z + (rho'/rho) p (pcg.hpp:76-84).
struct ProlongArgs {
    int n_levels;  // coarse levels
    const std::int32_t* agg[kMaxCoarse];
    const double* y[kMaxCoarse];
};

enum FinalMode : int { F_APPLY = 0, F_PCG_INIT = 1, F_PCG_STEP = 2 };

template <int kFinal>
__global__ void __launch_bounds__(256) k_mas_final(std::int32_t n, ProlongArgs pa, double* __restrict__ z, double* __restrict__ p,
                                                  PcgArgs a) {
    double beta = 0;
    bool write_p = false;
    if (kFinal != F_APPLY) {
        if (a.flags[F_DONE]) return;
        const double rz = a.scal[S_RZ_L0] + a.scal[S_RZ_C];
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
            const double rho = a.scal[S_RHO0 + ((a.k - 1) & 1)];
            const double stop = a.scal[S_STOP];
            if (blockIdx.x == 0 && threadIdx.x == 0) {
                a.flags[F_ITERS] = a.k;
                if (rz <= stop) {
                    a.flags[F_DONE] = 1;
                    a.flags[F_CONVERGED] = 1;
                    a.scal[S_REL] = sqrt(fabs(rz) / a.scal[S_RHO_INIT]);
                } else {
                    a.scal[S_RHO0 + (a.k & 1)] = rz;
                    a.scal[S_REL] = sqrt(fabs(rz) / a.scal[S_RHO_INIT]);
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
        }
    }
}

// Block Jacobi (block_jacobi.hpp:16-22), one thread per slot, with the same
// PCG modes as the level-0 MAS kernel. z = inv[i] r_i.
template <int kMode>
__global__ void __launch_bounds__(256) k_jacobi(std::int32_t n, const double* __restrict__ jinv, const double* __restrict__ r_in,
                                               double* __restrict__ z, PcgArgs a, double* __restrict__ partials,
                                               unsigned* __restrict__ ticket, double* __restrict__ dot_out) {
    double alpha = 0;
    if (kMode == M_UPDATE || kMode == M_RESTART) {
        if (a.flags[F_DONE]) return;
        if (!pcg_alpha(a, alpha)) return;
    }
    double dsum = 0;
    for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        double rv[3];
        for (int k = 0; k < 3; ++k) {
            const std::int64_t g = 3 * i + k;
            if (kMode == M_APPLY) {
                rv[k] = r_in[g];
            } else if (kMode == M_INIT) {
                rv[k] = a.b[g];
                a.r[g] = rv[k];
                a.x[g] = 0.0;
            } else if (kMode == M_UPDATE) {
                a.x[g] += alpha * a.p[g];
                rv[k] = a.r[g] - alpha * a.ap[g];
                a.r[g] = rv[k];
            } else {
                rv[k] = a.b[g] - a.ap[g];
                a.r[g] = rv[k];
            }
        }
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
