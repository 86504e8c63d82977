// MAS preconditioner construction on B200 (replaces
// TimeStepper::build_preconditioner, solver/newton.hpp:243-255:
// block_edges + build_hierarchy + MasPreconditioner::build, and
// BlockJacobiPreconditioner::build):
//   host:   block_edges (D2H of the pattern) -> build_hierarchy (host_precond)
//           -> per-level CSR metadata (sub_nodes, pos_of, node_slots)
//   device: K9 Galerkin restriction of A onto every level in ONE pass over A
//           (mas.hpp:56-64; level 0 is conflict-free and written directly,
//           coarser levels use fp64 atomics), then
//           K10 batched in-shared-memory Cholesky with the reference's
//           regularisation retry (mas.hpp:66-81: eps = 1e-8 tr/dim, shifts
//           eps, 100 eps, 1e4 eps cumulatively, failure after the 4th attempt)
//           and explicit inverse D^-1 = L^-T L^-1 (paper Alg. 1), one CTA per
//           subdomain.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <chrono>
#include <cstring>
#include <limits>

#include "mas_kernels.cuh"
#include "scan.cuh"


namespace adipc_gpu {

namespace {

struct RestrictLevel {
    const std::int32_t* agg;      // null at level 0 (identity)
    const std::int32_t* part_of;
    const std::int32_t* pos_of;
    const std::int64_t* dense_off;
    const std::int32_t* sub_ptr;
    double* dense;
};
struct RestrictArgs {
    int first, n_levels;  // levels [first, n_levels)
    RestrictLevel lv[kMaxLevels];
};

// Restricted subdomain matrices are stored packed: the lower triangle by
// columns, column j (rows j..d-1) starting at lpk_col(d, j). Only the lower
// triangle is ever read (Cholesky), so tiles above the diagonal are dropped —
// their transposes land below it.
__host__ __device__ __forceinline__ int lpk_col(int d, int j) { return j * d - (j * (j - 1)) / 2; }
__host__ __device__ __forceinline__ std::int64_t lpk_size(std::int64_t d) { return d * (d + 1) / 2; }

__device__ __forceinline__ void add_tile(double* D, int dim, int pr, int pc, const double* h, bool transpose,
                                         bool atomic) {
    // h column-major H(i,j) = h[3j+i] lands at (3pr+i, 3pc+j) when on or below the diagonal
    if (pr < pc) return;
#pragma unroll
    for (int j = 0; j < 3; ++j)
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            const int row = 3 * pr + i, col = 3 * pc + j;
            if (row < col) continue;
            const double v = transpose ? h[3 * i + j] : h[3 * j + i];
            double* dst = D + lpk_col(dim, col) + (row - col);
            if (atomic)
                atomicAdd(dst, v);
            else
                *dst += v;
        }
}

// One pass over A (solve order) restricts into every level in [first, n):
// level 0 conflict-free (each dense element receives exactly one entry);
// coarser levels by fp64 atomics, after the lanes of a warp (32 consecutive
// entries: a few rows, their columns ascending) that hit the same coarse tile
// have summed their contributions into the lowest such lane — a row's ~8
// upper entries fall into 2-3 level-1 nodes, so most atomics disappear.
// Each entry contributes ONE tile, oriented lower: H to (pr, pc) when
// pr > pc, H^T to (pc, pr) when pr < pc, H + H^T (r != c) on the diagonal.
__global__ void k_restrict(const std::uint32_t* __restrict__ rows, const std::uint32_t* __restrict__ cols,
                           const double* __restrict__ blocks, std::int64_t U, RestrictArgs ra) {
    const int lane = threadIdx.x & 31;
    const std::int64_t stride = static_cast<std::int64_t>(gridDim.x) * blockDim.x;
    for (std::int64_t e0 = (blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x) - lane; e0 < U;
         e0 += stride) {  // warp-uniform trip count: the warp intrinsics below need every lane
        const std::int64_t e = e0 + lane;
        const bool valid = e < U;
        const std::int32_t r = valid ? rows[e] : 0, c = valid ? cols[e] : 0;
        double h[9];
#pragma unroll
        for (int k = 0; k < 9; ++k) h[k] = valid ? blocks[blk(e, k)] : 0.0;
        for (int l = ra.first; l < ra.n_levels; ++l) {
            const RestrictLevel& L = ra.lv[l];
            const std::int32_t nr = L.agg ? L.agg[r] : r;
            const std::int32_t nc = L.agg ? L.agg[c] : c;
            const std::int32_t sd = L.part_of[nr];
            const bool act = valid && sd == L.part_of[nc];
            const int dim = act ? 3 * (L.sub_ptr[sd + 1] - L.sub_ptr[sd]) : 0;
            double* D = act ? L.dense + L.dense_off[sd] : nullptr;
            const int pr = act ? L.pos_of[nr] : 0, pc = act ? L.pos_of[nc] : 0;
            if (l == 0) {  // conflict-free
                if (act) {
                    add_tile(D, dim, pr, pc, h, false, false);
                    if (r != c) add_tile(D, dim, pc, pr, h, true, false);
                }
                continue;
            }
            const int pa = pr > pc ? pr : pc, pb = pr > pc ? pc : pr;
            double t[9];
#pragma unroll
            for (int j = 0; j < 3; ++j)
#pragma unroll
                for (int i = 0; i < 3; ++i) {  // t column-major, tile (pa, pb)
                    const double hij = h[3 * j + i], hji = h[3 * i + j];
                    t[3 * j + i] = pr > pc ? hij : (pr < pc ? hji : (r != c ? hij + hji : hij));
                }
            const unsigned long long key =
                act ? (static_cast<unsigned long long>(sd) << 24) | (static_cast<unsigned long long>(pa) << 12) |
                          static_cast<unsigned long long>(pb)
                    : ~0ull;
            const unsigned grp = __match_any_sync(0xffffffffu, key);
            const int rounds = __reduce_max_sync(0xffffffffu, act ? __popc(grp) : 1) - 1;
            const bool lead = act && (__ffs(grp) - 1) == lane;
            unsigned rest = grp & (grp - 1u);
            for (int k = 0; k < rounds; ++k) {
                const int src = rest ? __ffs(rest) - 1 : lane;
#pragma unroll
                for (int q = 0; q < 9; ++q) {
                    const double a = __shfl_sync(0xffffffffu, t[q], src);
                    if (lead && rest) t[q] += a;
                }
                rest &= rest - 1u;
            }
            if (lead) {
#pragma unroll
                for (int j = 0; j < 3; ++j)
#pragma unroll
                    for (int i = 0; i < 3; ++i) {
                        const int row = 3 * pa + i, col = 3 * pb + j;
                        if (row < col) continue;
                        atomicAdd(D + lpk_col(dim, col) + (row - col), t[3 * j + i]);
                    }
            }
        }
    }
}

// Deterministic coarse restriction (mas.hpp:56-64 semantics without fp
// atomics): one warp per level-l subdomain s walks its solve slots in
// ascending order and each slot's row entries in column order — the matrix's
// entry order restricted to s — and adds every entry whose both ends fall in
// s: H to tile (pr, pc), then H^T to (pc, pr), exactly the reference's
// sequence per dense element. Lanes evaluate 32 entries at a time; the adds
// are then applied entry by entry, nine lanes per 3x3 tile (lane i + 3 j owns
// element (i, j) of every tile, so an address is only ever updated by one
// lane, in program order).
__global__ void __launch_bounds__(128) k_restrict_det(std::int32_t n_parts, const std::int64_t* __restrict__ mem_ptr,
                                                      const std::int32_t* __restrict__ mem_slots,
                                                      const std::int64_t* __restrict__ row_ptr,
                                                      const std::uint32_t* __restrict__ cols,
                                                      const double* __restrict__ blocks, RestrictLevel L) {
    const int lane = threadIdx.x & 31;
    const std::int32_t s = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (s >= n_parts) return;
    const int dim = 3 * (L.sub_ptr[s + 1] - L.sub_ptr[s]);
    double* D = L.dense + L.dense_off[s];
    const int ti = lane % 3, tj = lane / 3;  // lanes 0..8: element (ti, tj) of a tile
    for (std::int64_t mi = mem_ptr[s]; mi < mem_ptr[s + 1]; ++mi) {
        const std::int32_t r = mem_slots[mi];
        const int pr = L.pos_of[L.agg[r]];
        const std::int64_t e0 = row_ptr[r], e1 = row_ptr[r + 1];
        for (std::int64_t base = e0; base < e1; base += 32) {
            const std::int64_t e = base + lane;
            int pc = -1;
            bool diag = false;
            double h[9];
            if (e < e1) {
                const std::int32_t c = static_cast<std::int32_t>(cols[e]);
                const std::int32_t nc = L.agg[c];
                if (L.part_of[nc] == s) {
                    pc = L.pos_of[nc];
                    diag = c == r;
#pragma unroll
                    for (int k = 0; k < 9; ++k) h[k] = blocks[blk(e, k)];
                }
            }
            const int nv = static_cast<int>(e1 - base < 32 ? e1 - base : 32);
            for (int q = 0; q < nv; ++q) {
                const int qpc = __shfl_sync(0xffffffffu, pc, q);
                const bool qdiag = __shfl_sync(0xffffffffu, diag ? 1 : 0, q) != 0;
                double hv[9];
#pragma unroll
                for (int k = 0; k < 9; ++k) hv[k] = __shfl_sync(0xffffffffu, h[k], q);
                if (qpc < 0 || lane >= 9) continue;
                // H to (pr, qpc); H^T to (qpc, pr) when r != c — kept where on or below the diagonal
                for (int t = 0; t < (qdiag ? 1 : 2); ++t) {
                    const int br = t == 0 ? pr : qpc, bc = t == 0 ? qpc : pr;
                    if (br < bc) continue;
                    const int row = 3 * br + ti, col = 3 * bc + tj;
                    if (row < col) continue;
                    const double v = t == 0 ? hv[3 * tj + ti] : hv[3 * ti + tj];
                    double* dst = D + lpk_col(dim, col) + (row - col);
                    *dst = __dadd_rn(*dst, v);
                }
            }
        }
    }
}

// keys (level-l subdomain of slot << 32 | slot) for the member lists
__global__ void k_member_keys(std::int32_t n, const std::int32_t* __restrict__ agg,
                              const std::int32_t* __restrict__ part_of, std::uint64_t* __restrict__ keys) {
    for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<std::int64_t>(gridDim.x) * blockDim.x)
        keys[i] = (static_cast<std::uint64_t>(part_of[agg[i]]) << 32) | static_cast<std::uint32_t>(i);
}

__global__ void k_high_words(const std::uint64_t* __restrict__ in, std::int64_t n, std::int32_t* __restrict__ out) {
    for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<std::int64_t>(gridDim.x) * blockDim.x)
        out[i] = static_cast<std::int32_t>(in[i] >> 32);
}

// One CTA per subdomain: Cholesky with retry, then explicit inverse, written
// symmetric-packed (upper triangle by columns: P[k(k+1)/2 + j] = D^-1(j,k),
// j <= k) — half the bytes the PCG streams per application.
// Work arrays S (dim x dim, column-major) + X (dim x dim) live in shared
// memory, or — for subdomains too large for it (capacity > 32) — in a global
// scratch slice per CTA (`gscratch`, 2 * max_dim^2 doubles per CTA).
__global__ void k_invert(std::int32_t n_parts, const std::int32_t* __restrict__ sub_ptr,
                         const std::int64_t* __restrict__ dense_off, const double* __restrict__ dense,
                         const std::int64_t* __restrict__ inv_off, double* __restrict__ inv,
                         int* __restrict__ status, int* __restrict__ shifts, double* __restrict__ gscratch,
                         int max_dim) {
    extern __shared__ double sm[];
    __shared__ int fail;
    __shared__ double eps0;
    double* work = gscratch ? gscratch + 2 * static_cast<std::int64_t>(max_dim) * max_dim * blockIdx.x : sm;
    for (std::int32_t s = blockIdx.x; s < n_parts; s += gridDim.x) {
        const int dim = 3 * (sub_ptr[s + 1] - sub_ptr[s]);
        if (dim == 0) continue;
        double* S = work;
        double* X = work + dim * dim;
        const double* D = dense + dense_off[s];
        double* P = inv + inv_off[s];
        const int nn = dim * dim;
        if (threadIdx.x == 0) {
            double tr = 0;
            for (int k = 0; k < dim; ++k) tr += D[lpk_col(dim, k)];
            double e = 1e-8 * tr / dim;
            if (!(e > 0)) e = 1e-12;
            eps0 = e;
        }
        __syncthreads();
        int attempt = 0;
        for (;; ++attempt) {
            for (int t = threadIdx.x; t < nn; t += blockDim.x) {  // lower triangle of the packed D
                const int i = t % dim, j = t / dim;
                if (i >= j) S[t] = D[lpk_col(dim, j) + (i - j)];
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                fail = 0;
                // cumulative shifts D += eps, D += 100 eps, ... (mas.hpp:78-79)
                double e = eps0;
                for (int a = 0; a < attempt; ++a) {
                    for (int k = 0; k < dim; ++k) S[k * dim + k] += e;
                    e *= 100;
                }
            }
            __syncthreads();
            // right-looking Cholesky on the lower triangle
            for (int k = 0; k < dim; ++k) {
                if (threadIdx.x == 0) {
                    const double x = S[k * dim + k];
                    if (x <= 0)  // Eigen LLT: non-positive pivot fails; NaN does not
                        fail = 1;
                    else
                        S[k * dim + k] = sqrt(x);
                }
                __syncthreads();
                if (fail) break;
                const double piv = S[k * dim + k];
                for (int i = k + 1 + threadIdx.x; i < dim; i += blockDim.x) S[k * dim + i] /= piv;
                __syncthreads();
                const int m = dim - k - 1;
                for (int t = threadIdx.x; t < m * m; t += blockDim.x) {
                    const int i = k + 1 + t % m, j = k + 1 + t / m;
                    if (j <= i) S[j * dim + i] -= S[k * dim + i] * S[k * dim + j];
                }
                __syncthreads();
            }
            if (!fail) break;
            __syncthreads();
            if (attempt >= 3) break;
        }
        if (fail) {
            if (threadIdx.x == 0) atomicOr(status, 1);
            __syncthreads();
            continue;
        }
        if (threadIdx.x == 0 && attempt > 0) atomicAdd(shifts, attempt);
        // X = L^-1 (lower), column j by thread j: forward substitution
        for (int j = threadIdx.x; j < dim; j += blockDim.x) {
            for (int i = 0; i < dim; ++i) {
                if (i < j) {
                    X[j * dim + i] = 0;
                    continue;
                }
                double v = (i == j) ? 1.0 : 0.0;
                for (int k = j; k < i; ++k) v -= S[k * dim + i] * X[j * dim + k];
                X[j * dim + i] = v / S[i * dim + i];
            }
        }
        __syncthreads();
        // D^-1 = X^T X, symmetric: entry (j, k), j <= k, into the packed upper
        for (int t = threadIdx.x; t < nn; t += blockDim.x) {
            const int j = t % dim, k = t / dim;
            if (j > k) continue;
            double v = 0;
            for (int q = k; q < dim; ++q) v += X[j * dim + q] * X[k * dim + q];
            P[k * (k + 1) / 2 + j] = v;
        }
        __syncthreads();
    }
}

// Warp-per-subdomain variant of k_invert for dim <= 32 R (R rows per lane),
// same semantics (Cholesky with the mas.hpp:66-81 retry rule, explicit
// inverse L^-T L^-1 written symmetric-packed). Warp-synchronous, all in ONE
// packed lower triangle per warp in shared memory (d(d+1)/2 doubles, so twice
// the warps of a full d x d work array fit an SM): right-looking Cholesky in
// place (lane i updates row i of the trailing columns), W = L^-1 in place
// column by column from the right (W(i,j) = -W(j,j) sum_{k>j} W(i,k) L(k,j),
// the trailing block already inverted), then the packed upper of W^T W
// column by column. Column accesses are lane-contiguous; the row reads of the
// product fall in distinct banks for 16 consecutive columns (triangular
// offsets).
// Every level's subdomains in one launch (the levels are independent once
// restricted): item q of the concatenated list belongs to level l with
// base[l] <= q < base[l + 1].
struct InvertLevel {
    const std::int32_t* sub_ptr;
    const std::int64_t* dense_off;
    const double* dense;
    const std::int64_t* inv_off;
    double* inv;
};
struct InvertTable {
    int n;
    std::int32_t base[kMaxLevels + 1];
    InvertLevel lv[kMaxLevels];
};

template <int R>
__global__ void __launch_bounds__(128) k_invert_warp(InvertTable tab, int* __restrict__ status,
                                                    int* __restrict__ shifts, int* __restrict__ next, int max_dim) {
    extern __shared__ double sm[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int slot = static_cast<int>(lpk_size(max_dim) + 1) & ~1;  // 16-byte aligned slots
    double* S = sm + static_cast<std::size_t>(w) * slot;
    // resident grid, items taken dynamically (their cost varies with dim and retries)
    for (;;) {
        std::int32_t q = 0;
        if (lane == 0) q = atomicAdd(next, 1);
        q = __shfl_sync(0xffffffffu, q, 0);
        if (q >= tab.base[tab.n]) break;
        int l = 0;
        while (l + 1 < tab.n && q >= tab.base[l + 1]) ++l;
        const std::int32_t s = q - tab.base[l];
        const std::int32_t* sub_ptr = tab.lv[l].sub_ptr;
        const int d = 3 * (sub_ptr[s + 1] - sub_ptr[s]);
        if (d == 0) continue;
        const double* D = tab.lv[l].dense + tab.lv[l].dense_off[s];
        const int np = static_cast<int>(lpk_size(d));
        double tr = 0;
#pragma unroll
        for (int t = 0; t < R; ++t) {
            const int i = lane + 32 * t;
            if (i < d) tr += D[lpk_col(d, i)];
        }
        for (int o = 16; o > 0; o >>= 1) tr += __shfl_xor_sync(0xffffffffu, tr, o);
        double eps0 = 1e-8 * tr / d;
        if (!(eps0 > 0)) eps0 = 1e-12;
        bool fail = true;
        int attempt = 0;
        for (; attempt < 4; ++attempt) {
            for (int e = lane; e < np; e += 32) S[e] = D[e];
            __syncwarp();
            if (attempt > 0)  // cumulative shifts eps, 100 eps, ... (mas.hpp:78-79), added in turn
                for (int i = lane; i < d; i += 32) {
                    double x = S[lpk_col(d, i)], ee = eps0;
                    for (int a = 0; a < attempt; ++a) {
                        x += ee;
                        ee *= 100;
                    }
                    S[lpk_col(d, i)] = x;
                }
            __syncwarp();
            fail = false;
            // left-looking (Crout) Cholesky, column by column: lane i forms
            // s_i = D(i,j) - sum_{k<j} L(i,k) L(j,k) in four independent FMA
            // chains (no read-modify-write of the trailing matrix), the pivot
            // is the row-j lane's s, then the column is scaled and written
            for (int j = 0; j < d; ++j) {
                const int oj = lpk_col(d, j) - j;  // column j: (i,j) at S[oj + i]
                double sc[4][R];
#pragma unroll
                for (int t = 0; t < R; ++t) {
                    const int i = lane + 32 * t;
                    sc[0][t] = (i >= j && i < d) ? S[oj + i] : 0.0;
                    sc[1][t] = sc[2][t] = sc[3][t] = 0.0;
                }
                int okc = 0;  // lpk_col(d, k) - k, from k = 0
                auto chol_step = [&](int k, double* acc) {
                    const double ljk = S[okc + j];  // L(j,k), broadcast
#pragma unroll
                    for (int t = 0; t < R; ++t) {
                        const int i = lane + 32 * t;
                        if (i >= j && i < d) acc[t] -= S[okc + i] * ljk;
                    }
                    okc += d - k - 1;
                };
                int k = 0;
                for (; k + 3 < j; k += 4) {
                    chol_step(k, sc[0]);
                    chol_step(k + 1, sc[1]);
                    chol_step(k + 2, sc[2]);
                    chol_step(k + 3, sc[3]);
                }
                for (; k < j; ++k) chol_step(k, sc[0]);
                double sv[R];
#pragma unroll
                for (int t = 0; t < R; ++t) sv[t] = (sc[0][t] + sc[1][t]) + (sc[2][t] + sc[3][t]);
                // pivot: row j lives in lane j % 32, register slot j / 32
                const double x = __shfl_sync(0xffffffffu, j < 32 ? sv[0] : sv[R - 1], j & 31);
                if (x <= 0) {  // Eigen LLT: a non-positive pivot fails; NaN does not
                    fail = true;
                    break;
                }
                const double piv = sqrt(x);
#pragma unroll
                for (int t = 0; t < R; ++t) {
                    const int i = lane + 32 * t;
                    if (i > j && i < d) S[oj + i] = sv[t] / piv;
                }
                if (lane == 0) S[oj + j] = piv;
                __syncwarp();  // column j complete before later columns read it
            }
            if (!fail) break;
            __syncwarp();  // every lane's reads of the failed attempt before the next one rewrites S
        }
        if (fail) {
            if (lane == 0) atomicOr(status, 1);
            __syncwarp();
            continue;
        }
        if (lane == 0 && attempt > 0) atomicAdd(shifts, attempt);
        // W = L^-1 in place, columns from the right
        for (int j = d - 1; j >= 0; --j) {
            const int oj = lpk_col(d, j) - j;
            const double wjj = 1.0 / S[oj + j];
            double a[4][R];  // four independent fp64 FMA chains (static indices)
#pragma unroll
            for (int q = 0; q < 4; ++q)
#pragma unroll
                for (int t = 0; t < R; ++t) a[q][t] = 0.0;
            int okk = lpk_col(d, j + 1) - (j + 1);
            auto inv_step = [&](int k, double* acc) {
                const double lkj = S[oj + k];  // L(k,j), broadcast
#pragma unroll
                for (int t = 0; t < R; ++t) {
                    const int i = lane + 32 * t;
                    if (i >= k && i < d) acc[t] += S[okk + i] * lkj;  // W(i,k)
                }
                okk += d - k - 1;
            };
            int k = j + 1;
            for (; k + 3 < d; k += 4) {
                inv_step(k, a[0]);
                inv_step(k + 1, a[1]);
                inv_step(k + 2, a[2]);
                inv_step(k + 3, a[3]);
            }
            for (; k < d; ++k) inv_step(k, a[0]);
            __syncwarp();  // every read of column j done before it is overwritten
#pragma unroll
            for (int t = 0; t < R; ++t) {
                const int i = lane + 32 * t;
                if (i > j && i < d) S[oj + i] = -wjj * ((a[0][t] + a[1][t]) + (a[2][t] + a[3][t]));
            }
            if (lane == 0) S[oj + j] = wjj;
            __syncwarp();
        }
        // D^-1 = W^T W: packed column k, lanes j <= k: sum_{q >= k} W(q,j) W(q,k)
        double* P = tab.lv[l].inv + tab.lv[l].inv_off[s];
        int oc[R];  // W(q, j) of lane j at S[oc + q]
#pragma unroll
        for (int t = 0; t < R; ++t) {
            const int j = min(lane + 32 * t, d - 1);
            oc[t] = lpk_col(d, j) - j;
        }
        for (int k = 0; k < d; ++k) {
            const int ok = lpk_col(d, k) - k;
            const double wkk = S[ok + k];
            double v[4][R];  // four independent fp64 FMA chains
#pragma unroll
            for (int t = 0; t < R; ++t) {
                const int j = lane + 32 * t;  // q = k term
                v[0][t] = j < k ? S[oc[t] + k] * wkk : (j == k ? wkk * wkk : 0.0);
                v[1][t] = v[2][t] = v[3][t] = 0.0;
            }
            auto prod_step = [&](int q2, double* acc) {
                const double wqk = S[ok + q2];  // broadcast
#pragma unroll
                for (int t = 0; t < R; ++t) {
                    const int j = lane + 32 * t;
                    if (j <= k) {
                        const double wqj = j == k ? wqk : S[oc[t] + q2];
                        acc[t] += wqj * wqk;
                    }
                }
            };
            int q2 = k + 1;
            for (; q2 + 3 < d; q2 += 4) {
                prod_step(q2, v[0]);
                prod_step(q2 + 1, v[1]);
                prod_step(q2 + 2, v[2]);
                prod_step(q2 + 3, v[3]);
            }
            for (; q2 < d; ++q2) prod_step(q2, v[0]);
#pragma unroll
            for (int t = 0; t < R; ++t) {
                const int j = lane + 32 * t;
                if (j <= k) P[k * (k + 1) / 2 + j] = (v[0][t] + v[1][t]) + (v[2][t] + v[3][t]);
            }
        }
        __syncwarp();
    }
}

__global__ void k_jacobi_build(std::int32_t n, const std::uint32_t* __restrict__ cols, const double* __restrict__ blocks,
                               std::int64_t U, const std::int64_t* __restrict__ row_ptr, double* __restrict__ jinv) {
    for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        double a[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
        for (std::int64_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e)
            if (cols[e] == static_cast<std::uint32_t>(i)) {
                for (int k = 0; k < 9; ++k) a[k] = blocks[blk(e, k)];
                // Mat3::inverse as Eigen computes a fixed 3x3 (block_jacobi.hpp:13):
                // cyclic cofactors, det down column 0, times 1/det; explicit
                // _rn ops so nvcc cannot contract into FMAs (bitwise with CPU)
                auto A = [&](int r, int c) { return a[3 * c + r]; };
                auto cof = [&](int i, int j) {
                    const int i1 = (i + 1) % 3, i2 = (i + 2) % 3, j1 = (j + 1) % 3, j2 = (j + 2) % 3;
                    return __dsub_rn(__dmul_rn(A(i1, j1), A(i2, j2)), __dmul_rn(A(i1, j2), A(i2, j1)));
                };
                const double det = __dadd_rn(__dadd_rn(__dmul_rn(cof(0, 0), A(0, 0)), __dmul_rn(cof(1, 0), A(1, 0))),
                                             __dmul_rn(cof(2, 0), A(2, 0)));
                const double invdet = __ddiv_rn(1.0, det);
                double inv[9];
                for (int i = 0; i < 3; ++i)
                    for (int j = 0; j < 3; ++j) inv[3 * j + i] = __dmul_rn(cof(j, i), invdet);
                for (int k = 0; k < 9; ++k) a[k] = inv[k];
                break;
            }
        for (int k = 0; k < 9; ++k) jinv[9 * i + k] = a[k];
    }
}

template <class T>
void upload(DBuf<T>& d, const std::vector<T>& h, cudaStream_t st) {
    d.reserve(h.size());
    if (!h.empty()) ADIPC_CUDA(cudaMemcpyAsync(d.p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice, st));
}

// Per-level CSR metadata from a hierarchy level (mas.hpp:42-54 semantics:
// pos_of = rank of the node among its subdomain's nodes in ascending id).
void build_level(Ctx& c, DeviceLevel& L, const host::Level& hl, int level, std::int32_t n_slots, bool upload_agg = true) {
    cudaStream_t st = c.stream;
    L.n_nodes = hl.n_nodes;
    L.n_parts = hl.n_parts;
    std::vector<std::int32_t> sub_ptr(hl.n_parts + 1, 0), pos_of(hl.n_nodes), sub_nodes(hl.n_nodes);
    for (std::int32_t v = 0; v < hl.n_nodes; ++v) pos_of[v] = sub_ptr[hl.part_of[v] + 1]++;
    int max_fill = 0;
    for (std::int32_t s = 0; s < hl.n_parts; ++s) max_fill = std::max(max_fill, sub_ptr[s + 1]);
    for (std::int32_t s = 0; s < hl.n_parts; ++s) sub_ptr[s + 1] += sub_ptr[s];
    for (std::int32_t v = 0; v < hl.n_nodes; ++v) sub_nodes[sub_ptr[hl.part_of[v]] + pos_of[v]] = v;
    // restricted matrices (build scratch, packed lower triangle) and the packed
    // inverses (d(d+1)/2, padded to 16 B so each is one TMA bulk copy)
    std::vector<std::int64_t> inv_off(hl.n_parts + 1, 0), dense_off(hl.n_parts + 1, 0);
    for (std::int32_t s = 0; s < hl.n_parts; ++s) {
        const std::int64_t d = 3 * static_cast<std::int64_t>(sub_ptr[s + 1] - sub_ptr[s]);
        dense_off[s + 1] = dense_off[s] + lpk_size(d);  // packed lower triangle
        inv_off[s + 1] = inv_off[s] + packed_doubles(static_cast<int>(d));
    }
    L.max_fill = max_fill;
    L.inv_doubles = inv_off[hl.n_parts];
    L.dense_doubles = dense_off[hl.n_parts];
    upload(L.part_of, hl.part_of, st);
    upload(L.pos_of, pos_of, st);
    upload(L.sub_ptr, sub_ptr, st);
    upload(L.sub_nodes, sub_nodes, st);
    upload(L.inv_off, inv_off, st);
    upload(L.dense_off, dense_off, st);
    L.inv_off_host = std::move(inv_off);
    if (level > 0) {
        if (upload_agg)
            upload(L.agg, hl.agg, st);
        else
            L.agg.reserve(static_cast<std::size_t>(n_slots));
        L.y.reserve(3 * static_cast<std::size_t>(hl.n_nodes));
        L.rr.reserve(3 * static_cast<std::size_t>(hl.n_nodes));
    }
    L.pos_host = std::move(pos_of);
    L.inv.reserve(static_cast<std::size_t>(L.inv_doubles));
    ADIPC_CUDA(cudaMemsetAsync(L.inv.p, 0, sizeof(double) * std::max<std::int64_t>(L.inv_doubles, 1), st));
    L.dense.reserve(static_cast<std::size_t>(L.dense_doubles));
    ADIPC_CUDA(cudaMemsetAsync(L.dense.p, 0, sizeof(double) * std::max<std::int64_t>(L.dense_doubles, 1), st));
}

// Restriction metadata from level l to l+1 (see mas_kernels.cuh): the
// level-(l+1) nodes inside each level-l subdomain are consecutive ids; their
// children are given as positions inside that subdomain.
void link_levels(Ctx& c, const host::MasHierarchy& h) {
    cudaStream_t st = c.stream;
    std::vector<std::vector<std::int32_t>> ups(h.n_levels());
    for (int l = 0; l + 1 < h.n_levels(); ++l) {
        const host::Level& cur = h.levels[l];
        const host::Level& nxt = h.levels[l + 1];
        DeviceLevel& L = *c.levels[l];
        std::vector<std::int32_t> up(cur.n_nodes, -1);
        if (l == 0) {
#pragma omp parallel for schedule(static)
            for (std::int32_t slot = 0; slot < h.n_slots; ++slot) up[slot] = nxt.agg[slot];
        } else {
            for (std::int32_t slot = 0; slot < h.n_slots; ++slot) up[cur.agg[slot]] = nxt.agg[slot];
        }
        std::vector<std::int32_t> first(cur.n_parts + 1, std::numeric_limits<std::int32_t>::max());
        std::vector<std::int32_t> cnt(nxt.n_nodes + 1, 0);
        for (std::int32_t v = 0; v < cur.n_nodes; ++v) {
            first[cur.part_of[v]] = std::min(first[cur.part_of[v]], up[v]);
            ++cnt[up[v] + 1];
        }
        first[cur.n_parts] = nxt.n_nodes;
        for (std::int32_t s = cur.n_parts - 1; s >= 0; --s)
            if (first[s] == std::numeric_limits<std::int32_t>::max()) first[s] = first[s + 1];  // empty subdomain
        for (std::int32_t v = 0; v < nxt.n_nodes; ++v) cnt[v + 1] += cnt[v];
        std::vector<std::int32_t> pos(cur.n_nodes), node(cur.n_nodes), fill(cnt.begin(), cnt.end() - 1);
        for (std::int32_t v = 0; v < cur.n_nodes; ++v) {  // children ascending
            node[fill[up[v]]] = v;
            pos[fill[up[v]]++] = L.pos_host[v];
        }
        upload(L.up_first, first, st);
        upload(L.upc_ptr, cnt, st);
        upload(L.upc_pos, pos, st);
        upload(L.upc_node, node, st);
        upload(L.up_node, up, st);
        ups[l] = std::move(up);
    }
    // ancestors of the level-1 nodes at every level >= 2 (update-pass RED targets)
    if (h.n_levels() > 2) {
        std::vector<std::int32_t> a = ups[1];
        for (int l = 2; l < h.n_levels(); ++l) {
            upload(c.levels[l]->anc, a, st);
            if (l + 1 < h.n_levels())
                for (auto& v : a) v = ups[l][v];
        }
    }
}

// A in solve order as a triplet stream: (perm[r], perm[c]) re-canonicalised to
// the upper triangle (the block transposed when the order flips, as
// BlockTripletStream::emit does, block_coo.hpp:36-43), AoS column-major values.
__global__ void k_permute_stream(const std::uint32_t* __restrict__ rows, const std::uint32_t* __restrict__ cols,
                                 const double* __restrict__ blocks, std::int64_t U,
                                 const std::int32_t* __restrict__ perm, std::uint64_t* __restrict__ keys,
                                 double* __restrict__ vals) {
    for (std::int64_t e = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; e < U;
         e += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        const std::uint32_t r = static_cast<std::uint32_t>(perm[rows[e]]);
        const std::uint32_t c = static_cast<std::uint32_t>(perm[cols[e]]);
        double h[9];
#pragma unroll
        for (int k = 0; k < 9; ++k) h[k] = blocks[blk(e, k)];
        const bool flip = r > c;
        keys[e] = flip ? (static_cast<std::uint64_t>(c) << 32 | r) : (static_cast<std::uint64_t>(r) << 32 | c);
#pragma unroll
        for (int j = 0; j < 3; ++j)
#pragma unroll
            for (int i = 0; i < 3; ++i) vals[9 * e + 3 * j + i] = flip ? h[3 * i + j] : h[3 * j + i];
    }
}

// Solve order of a hierarchy: slots renumbered so each level-0 subdomain is a
// contiguous range, members in ascending reference id (= pos_of order).
// Uploads the slot map to c.perm and returns the hierarchy in solve order
// (level 0: part_of by solve slot, agg identity; coarser levels: agg by solve
// slot; node-level data unchanged).
host::MasHierarchy to_solve_order(Ctx& c, const host::MasHierarchy& h) {
    const host::Level& l0 = h.levels[0];
    const std::int32_t n = h.n_slots;
    std::vector<std::int32_t> start(static_cast<std::size_t>(l0.n_parts) + 1, 0), perm(n);
    for (std::int32_t i = 0; i < n; ++i) ++start[l0.part_of[i] + 1];
    for (std::int32_t s = 0; s < l0.n_parts; ++s) start[s + 1] += start[s];
    for (std::int32_t i = 0; i < n; ++i) perm[i] = start[l0.part_of[i]]++;
    upload(c.perm, perm, c.stream);
    // built directly (no copy of the slot-sized arrays): level 0's agg is the
    // identity and never read in solve order
    host::MasHierarchy hp;
    hp.capacity = h.capacity;
    hp.n_slots = n;
    hp.levels.resize(h.levels.size());
    for (std::size_t l = 0; l < h.levels.size(); ++l) {
        hp.levels[l].n_nodes = h.levels[l].n_nodes;
        hp.levels[l].n_parts = h.levels[l].n_parts;
        if (l > 0) hp.levels[l].part_of = h.levels[l].part_of;
    }
    hp.levels[0].part_of.resize(n);
#pragma omp parallel for schedule(static)
    for (std::int32_t i = 0; i < n; ++i) hp.levels[0].part_of[perm[i]] = l0.part_of[i];
    for (std::size_t l = 1; l < h.levels.size(); ++l) {
        std::vector<std::int32_t>& agg = hp.levels[l].agg;
        agg.resize(n);
        const std::vector<std::int32_t>& src = h.levels[l].agg;
#pragma omp parallel for schedule(static)
        for (std::int32_t i = 0; i < n; ++i) agg[perm[i]] = src[i];
    }
    return hp;
}

// (Re)build the device levels of hierarchy h, in solve order when enabled.
void set_levels(Ctx& c, const host::MasHierarchy& h) {
    const bool dbg = std::getenv("ADIPC_DEBUG_HIER") != nullptr;
    auto lap = [&, t = std::chrono::steady_clock::now()](const char* what) mutable {
        if (!dbg) return;
        ADIPC_CUDA(cudaStreamSynchronize(c.stream));
        const auto now = std::chrono::steady_clock::now();
        std::fprintf(stderr, "set_levels %s %.1f ms\n", what, std::chrono::duration<double, std::milli>(now - t).count());
        t = now;
    };
    // level objects (and their device buffers, which only grow) are reused
    // across rebuilds: a new sparsity pattern costs no cudaFree / cudaMalloc
    // of the ~400 MB of level storage
    const std::size_t n_lv = static_cast<std::size_t>(h.n_levels());
    if (c.levels.size() > n_lv) c.levels.resize(n_lv);
    while (c.levels.size() < n_lv) c.levels.emplace_back(new DeviceLevel());
    c.l0_levels_version = ~0ull;  // level 0 rebuilt from h: the per-scene cache no longer holds
    lap("levels");
    const bool perm = c.solve_order && h.n_levels() > 0 && h.n_slots > 0;
    const host::MasHierarchy hp = perm ? to_solve_order(c, h) : host::MasHierarchy{};
    const host::MasHierarchy& hl = perm ? hp : h;
    lap("to_solve_order");
    for (int l = 0; l < hl.n_levels(); ++l) {
        build_level(c, *c.levels[l], hl.levels[l], l, c.A.n);
        lap("build_level");
    }
    link_levels(c, hl);
    lap("link_levels");
    c.levels_permuted = perm;
    ++c.levels_version;
}

// Level 0 in solve order from the level-0 partition alone (per scene): the
// slot permutation, its device copy and the level-0 metadata, kept across
// cold rebuilds until the partition, the size or the mode changes.
void ensure_level0(Ctx& c) {
    const std::int32_t n = static_cast<std::int32_t>(c.l0.part_of.size());
    if (c.l0_levels_version == c.l0_version && !c.levels.empty() && c.levels[0]->n_nodes == n &&
        static_cast<std::int32_t>(c.perm_host.size()) == n)
        return;
    const host::Partition& l0 = c.l0;
    std::vector<std::int32_t> start(static_cast<std::size_t>(l0.n_parts) + 1, 0);
    c.perm_host.resize(n);
    for (std::int32_t i = 0; i < n; ++i) ++start[l0.part_of[i] + 1];
    for (std::int32_t s = 0; s < l0.n_parts; ++s) start[s + 1] += start[s];
    for (std::int32_t i = 0; i < n; ++i) c.perm_host[i] = start[l0.part_of[i]]++;
    upload(c.perm, c.perm_host, c.stream);
    host::Level lv;
    lv.n_nodes = n;
    lv.n_parts = l0.n_parts;
    lv.part_of.resize(n);
    for (std::int32_t i = 0; i < n; ++i) lv.part_of[c.perm_host[i]] = l0.part_of[i];
    if (c.levels.empty()) c.levels.emplace_back(new DeviceLevel());
    build_level(c, *c.levels[0], lv, 0, n);
    c.l0_solve_part_of = std::move(lv.part_of);
    c.l0_levels_version = c.l0_version;
    ++c.levels_version;
}

__global__ void k_perm_scatter(std::int32_t n, const std::int32_t* __restrict__ perm,
                               const std::int32_t* __restrict__ src, std::int32_t* __restrict__ dst) {
    for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<std::int64_t>(gridDim.x) * blockDim.x)
        dst[perm[i]] = src[i];
}
__global__ void k_map_through(std::int32_t n, const std::int32_t* __restrict__ map,
                              const std::int32_t* __restrict__ src, std::int32_t* __restrict__ dst) {
    for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<std::int64_t>(gridDim.x) * blockDim.x)
        dst[i] = map[src[i]];
}

// Restriction links level 0 -> 1 in solve order (link_levels' level-0 part):
// one warp per level-0 subdomain (<= 32 slots, contiguous in solve order,
// lane j = slot sub_ptr[s] + j); its level-1 nodes are consecutive ids from
// agg1 of its first slot, so the children lists (ascending slots) and their
// CSR offsets follow from ballots inside the warp.
__global__ void k_l0_links(std::int32_t n_parts, std::int32_t n, std::int32_t n1,
                           const std::int32_t* __restrict__ sub_ptr, const std::int32_t* __restrict__ agg1,
                           std::int32_t* __restrict__ up_first, std::int32_t* __restrict__ upc_ptr,
                           std::int32_t* __restrict__ upc_pos, std::int32_t* __restrict__ upc_node) {
    const int lane = threadIdx.x & 31;
    const std::int64_t w = (blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x) >> 5;
    if (w >= n_parts) return;
    const std::int32_t s = static_cast<std::int32_t>(w);
    const std::int32_t a = sub_ptr[s], m = sub_ptr[s + 1] - a;
    const bool act = lane < m;
    // the subdomain's smallest level-1 node (an empty subdomain: the next one's)
    const std::int32_t base = a < n ? agg1[a] : n1;
    const std::int32_t loc = act ? agg1[a + lane] - base : 0x7FFFFFFF;
    const unsigned lt = (1u << lane) - 1u;
    const unsigned same = __match_any_sync(0xffffffffu, loc);
    // offset of node base + loc: slots of the subdomain in nodes < loc
    int n_below = 0;
    for (int j = 0; j < m; ++j) n_below += (__shfl_sync(0xffffffffu, loc, j) < loc) ? 1 : 0;
    if (act) {
        const int q = a + n_below + __popc(same & lt);
        upc_node[q] = a + lane;
        upc_pos[q] = lane;
        if ((same & lt) == 0) upc_ptr[base + loc] = a + n_below;  // first child of its node
    }
    if (lane == 0) up_first[s] = base;
    if (s == n_parts - 1 && lane == 0) upc_ptr[n1] = n;
}

// The coarse levels (>= 1) of hierarchy h in solve order on top of the
// cached level 0, and the restriction links of every level. The slot-sized
// parts are built on the device: level-1 agg from the level-1 pass's map
// through perm, levels >= 2 through the (small) level-1 -> level-l ancestor
// maps, the level-0 links by k_l0_links; the host links the small coarse
// levels.
void set_coarse_levels(Ctx& c, const host::MasHierarchy& h) {
    cudaStream_t st = c.stream;
    const std::int32_t n = h.n_slots;
    const std::size_t n_lv = static_cast<std::size_t>(h.n_levels());
    if (c.levels.size() > std::max<std::size_t>(n_lv, 1)) c.levels.resize(std::max<std::size_t>(n_lv, 1));
    while (c.levels.size() < n_lv) c.levels.emplace_back(new DeviceLevel());
    for (std::size_t l = 1; l < n_lv; ++l) build_level(c, *c.levels[l], h.levels[l], static_cast<int>(l), n, false);
    if (n_lv < 2) {
        c.levels_permuted = true;
        ++c.levels_version;
        return;
    }
    // agg of level 1 in solve order, then levels >= 2 through the ancestors
    DeviceLevel& L1 = *c.levels[1];
    k_perm_scatter<<<grid_for(n, 256, 16), 256, 0, st>>>(n, c.perm.p, c.l1_up.p, L1.agg.p);
    ADIPC_LAUNCH_CHECK();
    std::vector<std::int32_t> anc;  // level-1 node -> level-l node
    for (std::size_t l = 2; l < n_lv; ++l) {
        const std::vector<std::int32_t>& up = h.levels[l - 1].up;
        if (l == 2) {
            anc = up;
        } else {
            for (auto& v : anc) v = up[v];
        }
        DeviceLevel& Ll = *c.levels[l];
        upload(Ll.anc, anc, st);
        k_map_through<<<grid_for(n, 256, 16), 256, 0, st>>>(n, Ll.anc.p, L1.agg.p, Ll.agg.p);
        ADIPC_LAUNCH_CHECK();
    }
    // level-0 links on the device
    DeviceLevel& L0 = *c.levels[0];
    const std::int32_t n1 = h.levels[1].n_nodes;
    L0.up_first.reserve(static_cast<std::size_t>(h.levels[0].n_parts) + 1);
    L0.upc_ptr.reserve(static_cast<std::size_t>(n1) + 1);
    L0.upc_pos.reserve(static_cast<std::size_t>(n));
    L0.upc_node.reserve(static_cast<std::size_t>(n));
    L0.up_node.reserve(static_cast<std::size_t>(n));
    k_l0_links<<<static_cast<int>(ceil_div(h.levels[0].n_parts, 8)), 256, 0, st>>>(
        h.levels[0].n_parts, n, n1, L0.sub_ptr.p, L1.agg.p, L0.up_first.p, L0.upc_ptr.p, L0.upc_pos.p, L0.upc_node.p);
    ADIPC_LAUNCH_CHECK();
    ADIPC_CUDA(cudaMemcpyAsync(L0.up_node.p, L1.agg.p, sizeof(std::int32_t) * n, cudaMemcpyDeviceToDevice, st));
    ADIPC_CUDA(cudaMemcpyAsync(L0.up_first.p + h.levels[0].n_parts, &n1, sizeof(n1), cudaMemcpyHostToDevice, st));
    // levels >= 1: the host links from the stored node maps (link_levels' rule)
    for (std::size_t l = 1; l + 1 < n_lv; ++l) {
        const host::Level& cur = h.levels[l];
        const host::Level& nxt = h.levels[l + 1];
        DeviceLevel& L = *c.levels[l];
        const std::vector<std::int32_t>& up = cur.up;
        std::vector<std::int32_t> first(cur.n_parts + 1, std::numeric_limits<std::int32_t>::max());
        std::vector<std::int32_t> cnt(nxt.n_nodes + 1, 0);
        for (std::int32_t v = 0; v < cur.n_nodes; ++v) {
            first[cur.part_of[v]] = std::min(first[cur.part_of[v]], up[v]);
            ++cnt[up[v] + 1];
        }
        first[cur.n_parts] = nxt.n_nodes;
        for (std::int32_t s = cur.n_parts - 1; s >= 0; --s)
            if (first[s] == std::numeric_limits<std::int32_t>::max()) first[s] = first[s + 1];
        for (std::int32_t v = 0; v < nxt.n_nodes; ++v) cnt[v + 1] += cnt[v];
        std::vector<std::int32_t> pos(cur.n_nodes), node(cur.n_nodes), fill(cnt.begin(), cnt.end() - 1);
        for (std::int32_t v = 0; v < cur.n_nodes; ++v) {
            node[fill[up[v]]] = v;
            pos[fill[up[v]]++] = L.pos_host[v];
        }
        upload(L.up_first, first, st);
        upload(L.upc_ptr, cnt, st);
        upload(L.upc_pos, pos, st);
        upload(L.upc_node, node, st);
        upload(L.up_node, up, st);
    }
    c.levels_permuted = true;
    ++c.levels_version;
}

// As entry i <- A entry src (the bucket sort's emission index: the permuted
// stream has no repeated keys, so sorted position i IS As entry i), bit 31 when
// the block is stored transposed
__global__ void k_solve_map(const std::uint64_t* __restrict__ sorted, std::int64_t U,
                            const std::uint32_t* __restrict__ rows, const std::uint32_t* __restrict__ cols,
                            const std::int32_t* __restrict__ perm, std::uint32_t* __restrict__ src) {
    for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < U;
         i += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        const std::uint32_t e = static_cast<std::uint32_t>(sorted[i] & 0xFFFFFFFFu);
        const bool flip = perm[rows[e]] > perm[cols[e]];
        src[i] = e | (flip ? 0x80000000u : 0u);
    }
}

// As values from A through the map (pattern unchanged since the map was built)
__global__ void k_solve_gather(const double* __restrict__ blocks, const std::uint32_t* __restrict__ src,
                               std::int64_t U, double* __restrict__ out) {
    for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < U;
         i += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        const std::uint32_t m = src[i];
        const std::int64_t e = m & 0x7FFFFFFFu;
        double h[9];
#pragma unroll
        for (int k = 0; k < 9; ++k) h[k] = blocks[blk(e, k)];
        const bool flip = (m >> 31) != 0;
#pragma unroll
        for (int j = 0; j < 3; ++j)
#pragma unroll
            for (int i2 = 0; i2 < 3; ++i2) out[blk(i, 3 * j + i2)] = flip ? h[3 * i2 + j] : h[3 * j + i2];
    }
}

}  // namespace

// As = P A P^T in solve order (sorted upper block triangle, the same layout
// as A), rebuilt from the current A values on every preconditioner build:
// while the pattern and the levels are unchanged (`reuse`), one gather
// through the As -> A map; otherwise permute stream + the assembly
// sort/reduce, and the map is taken from the sort.
void build_solve_matrix(Ctx& c, bool reuse) {
    const DeviceMatrix& A = c.A;
    if (reuse && c.as_src_version == c.levels_version && c.As.U == A.U && c.As.n == A.n) {
        if (A.U > 0) {
            k_solve_gather<<<grid_for(A.U, 256, 16), 256, 0, c.stream>>>(A.blocks.p, c.as_src.p, A.U, c.As.blocks.p);
            ADIPC_LAUNCH_CHECK();
        }
        ++c.As.version;
        c.as_a_version = A.version;
        return;
    }
    c.perm_keys.reserve(static_cast<std::size_t>(std::max<std::int64_t>(A.U, 1)));
    c.perm_vals.reserve(9 * static_cast<std::size_t>(std::max<std::int64_t>(A.U, 1)));
    if (A.U > 0) {
        k_permute_stream<<<grid_for(A.U, 256, 16), 256, 0, c.stream>>>(A.rows.p, A.cols.p, A.blocks.p, A.U, c.perm.p,
                                                                      c.perm_keys.p, c.perm_vals.p);
        ADIPC_LAUNCH_CHECK();
    }
    sort_reduce(c, c.perm_keys.p, c.perm_vals.p, A.U, A.n, c.As);
    c.as_a_version = A.version;
    c.as_src_version = ~0ull;
    if (c.As.U != A.U) return;  // cannot happen for a permutation; no map then
    c.as_src.reserve(static_cast<std::size_t>(std::max<std::int64_t>(A.U, 1)));
    if (A.U > 0) {
        k_solve_map<<<grid_for(A.U, 256, 16), 256, 0, c.stream>>>(c.sorted.p, A.U, A.rows.p, A.cols.p, c.perm.p,
                                                                 c.as_src.p);
        ADIPC_LAUNCH_CHECK();
    }
    c.as_src_version = c.levels_version;
}

// The solve-order PCG multiplies by As: if A was reassembled (or uploaded)
// since As was built, rebuild As from the current A, as the reference's
// pcg_solve always uses the A it is given (pcg.hpp:34) whatever matrix the
// preconditioner was built on. A different size cannot be preconditioned.
static void check_precond_size(const Ctx& c) {
    if (c.pkind == kNone) throw StatusError(kInvalidArgument, "no preconditioner built");
    if ((c.pkind == kMas && (c.levels.empty() || c.levels[0]->n_nodes != c.A.n)) ||
        (c.pkind == kJacobi && c.jinv_n != c.A.n))
        throw StatusError(kInvalidArgument, "preconditioner built for a matrix of a different size");
}

void check_solve_matrix(Ctx& c) {
    check_precond_size(c);
    if (c.pkind == kMas && c.perm_active && c.as_a_version != c.A.version) build_solve_matrix(c, false);
}

// K9 restriction + K10 batched factorisation/inversion, in three steps so a
// cold build can factor level 0 while the host builds the coarse levels:
// factor_begin (status counters), factor_levels over a level range,
// factor_end (the one synchronisation: failure flag and shift count).
static void factor_begin(Ctx& c) {
    c.build_status.reserve(3);  // failure flag, shifts applied, work counter
    ADIPC_CUDA(cudaMemsetAsync(c.build_status.p, 0, 3 * sizeof(int), c.stream));
}

static void factor_levels(Ctx& c, int lb, int le) {
    cudaStream_t st = c.stream;
    const DeviceMatrix& A = c.S();
    for (int l = lb; l < le; ++l) {
        DeviceLevel& L = *c.levels[l];
        ADIPC_CUDA(cudaMemsetAsync(L.dense.p, 0, sizeof(double) * std::max<std::int64_t>(L.dense_doubles, 1), st));
    }
    RestrictArgs ra{};
    ra.first = lb;
    ra.n_levels = le;
    for (int l = 0; l < le; ++l) {
        DeviceLevel& L = *c.levels[l];
        ra.lv[l] = RestrictLevel{l > 0 ? L.agg.p : nullptr, L.part_of.p, L.pos_of.p, L.dense_off.p, L.sub_ptr.p,
                                 L.dense.p};
    }
    // deterministic mode: the atomics-free k_restrict pass covers level 0
    // only (conflict-free: one entry per dense element); coarse levels in a
    // fixed order per subdomain (k_restrict_det)
    if (c.deterministic) ra.n_levels = std::min(le, 1);
    if (A.U > 0 && ra.first < ra.n_levels) {
        k_restrict<<<grid_for(A.U, 256, 16), 256, 0, st>>>(A.rows.p, A.cols.p, A.blocks.p, A.U, ra);
        ADIPC_LAUNCH_CHECK();
    }
    for (int l = std::max(lb, 1); c.deterministic && l < le && A.U > 0; ++l) {
        DeviceLevel& L = *c.levels[l];
        if (L.det_version != c.levels_version) {  // solve slots of each subdomain, ascending
            c.perm_keys.reserve(static_cast<std::size_t>(A.n));
            k_member_keys<<<grid_for(A.n, 256, 16), 256, 0, st>>>(A.n, L.agg.p, L.part_of.p, c.perm_keys.p);
            ADIPC_LAUNCH_CHECK();
            bucket_sort(c, c.perm_keys.p, A.n, L.n_parts, nullptr);
            L.det_ptr.reserve(static_cast<std::size_t>(L.n_parts) + 1);
            L.det_slots.reserve(static_cast<std::size_t>(A.n));
            ADIPC_CUDA(cudaMemcpyAsync(L.det_ptr.p, c.row_start.p, sizeof(std::int64_t) * (L.n_parts + 1),
                                       cudaMemcpyDeviceToDevice, st));
            k_high_words<<<grid_for(A.n, 256, 16), 256, 0, st>>>(c.sorted.p, A.n, L.det_slots.p);
            ADIPC_LAUNCH_CHECK();
            L.det_version = c.levels_version;
        }
        k_restrict_det<<<static_cast<int>(ceil_div(L.n_parts, 4)), 128, 0, st>>>(
            L.n_parts, L.det_ptr.p, L.det_slots.p, A.row_ptr.p, A.cols.p, A.blocks.p, ra.lv[l]);
        ADIPC_LAUNCH_CHECK();
    }
    // warp-per-subdomain levels (dim <= 64): one launch for all of them
    InvertTable tab{};
    int wdim = 0;
    for (int l = lb; l < le; ++l) {
        DeviceLevel& L = *c.levels[l];
        const int dim = 3 * L.max_fill;
        if (L.n_parts == 0 || dim > 64) continue;
        tab.lv[tab.n] = InvertLevel{L.sub_ptr.p, L.dense_off.p, L.dense.p, L.inv_off.p, L.inv.p};
        tab.base[tab.n + 1] = tab.base[tab.n] + L.n_parts;
        ++tab.n;
        wdim = std::max(wdim, dim);
    }
    if (tab.n > 0) {
        // the warps take subdomains from a work counter (build_status[2]): reset
        // per launch, as a build may invert its levels in two launches
        ADIPC_CUDA(cudaMemsetAsync(c.build_status.p + 2, 0, sizeof(int), st));
        const int nw = 4;
        const std::size_t wsm = sizeof(double) * nw * static_cast<std::size_t>((lpk_size(wdim) + 1) & ~1);
        int sms = kSMs;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c.device);
        auto run = [&](auto kernel) {
            ADIPC_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(wsm)));
            int occ = 0;
            ADIPC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, 32 * nw, wsm));
            const int grid = static_cast<int>(std::max<std::int64_t>(
                1, std::min<std::int64_t>(ceil_div(tab.base[tab.n], nw), static_cast<std::int64_t>(sms) * std::max(occ, 1))));
            kernel<<<grid, 32 * nw, wsm, st>>>(tab, c.build_status.p, c.build_status.p + 1, c.build_status.p + 2, wdim);
        };
        if (wdim <= 32)
            run(k_invert_warp<1>);
        else
            run(k_invert_warp<2>);
        ADIPC_LAUNCH_CHECK();
    }
    for (int l = lb; l < le; ++l) {
        DeviceLevel& L = *c.levels[l];
        if (L.n_parts == 0) continue;
        const int dim = 3 * L.max_fill;
        if (dim <= 64) continue;  // done above
        const std::size_t need = 2 * sizeof(double) * dim * dim;
        const bool in_smem = need <= 200 * 1024;
        const int threads = dim <= 48 ? 128 : 256;
        const int grid = static_cast<int>(std::min<std::int64_t>(L.n_parts, in_smem ? kSMs * 16 : kSMs * 2));
        if (!in_smem) c.invert_scratch.reserve(need / sizeof(double) * grid);
        const std::size_t smem = in_smem ? need : 0;
        ADIPC_CUDA(cudaFuncSetAttribute(k_invert, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        k_invert<<<grid, threads, smem, st>>>(L.n_parts, L.sub_ptr.p, L.dense_off.p, L.dense.p, L.inv_off.p, L.inv.p,
                                              c.build_status.p,
                                              c.build_status.p + 1, in_smem ? nullptr : c.invert_scratch.p, dim);
        ADIPC_LAUNCH_CHECK();
    }
}

static void factor_end(Ctx& c) {
    int h_status[2] = {0, 0};
    ADIPC_CUDA(cudaMemcpyAsync(h_status, c.build_status.p, sizeof(h_status), cudaMemcpyDeviceToHost, c.stream));
    ADIPC_CUDA(cudaStreamSynchronize(c.stream));
    c.shifts_applied = h_status[1];
    if (h_status[0]) {
        c.pkind = kNone;
        throw StatusError(kIndefinite, "subdomain matrix stayed indefinite after regularization");
    }
    c.pkind = kMas;
}

void factorize(Ctx& c) {
    factor_begin(c);
    factor_levels(c, 0, static_cast<int>(c.levels.size()));
    factor_end(c);
}


namespace {
__device__ __forceinline__ std::uint64_t mix64(std::uint64_t z) {  // splitmix64 finaliser
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
// order-sensitive 64-bit hash of the pattern: sum_i mix(i, row_i, col_i)
__global__ void k_pattern_hash(const std::uint32_t* __restrict__ rows, const std::uint32_t* __restrict__ cols,
                               std::int64_t U, unsigned long long* __restrict__ out) {
    std::uint64_t h = 0;
    for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < U;
         i += static_cast<std::int64_t>(gridDim.x) * blockDim.x)
        h += mix64((static_cast<std::uint64_t>(rows[i]) << 32 | cols[i]) ^ mix64(static_cast<std::uint64_t>(i)));
    for (int o = 16; o > 0; o >>= 1) h += __shfl_xor_sync(0xffffffffu, h, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(out, static_cast<unsigned long long>(h));
}
}  // namespace

std::uint64_t pattern_hash(Ctx& c) {
    c.build_status.reserve(4);
    unsigned long long* d = reinterpret_cast<unsigned long long*>(c.build_status.p + 2);
    ADIPC_CUDA(cudaMemsetAsync(d, 0, sizeof(unsigned long long), c.stream));
    if (c.A.U > 0) {
        k_pattern_hash<<<grid_for(c.A.U, 256, 8), 256, 0, c.stream>>>(c.A.rows.p, c.A.cols.p, c.A.U, d);
        ADIPC_LAUNCH_CHECK();
    }
    unsigned long long h = 0;
    ADIPC_CUDA(cudaMemcpyAsync(&h, d, sizeof(h), cudaMemcpyDeviceToHost, c.stream));
    ADIPC_CUDA(cudaStreamSynchronize(c.stream));
    return (h ^ (static_cast<std::uint64_t>(c.A.n) << 1) ^ static_cast<std::uint64_t>(c.A.U) * 0x9e3779b97f4a7c15ull) |
           1ull;  // never equals the ~0 "invalid" marker's complement pattern; non-zero
}

namespace {

// Level-0 graph of build_hierarchy (hierarchy.hpp:30-100 -> partition.hpp:37-50)
// straight from the device matrix's pattern: node i's neighbours are the
// off-diagonal blocks of row i and of column i (block_edges, mas.hpp:19-25),
// every list sorted ascending and duplicate-free, as std::set-per-node makes
// them. Both directions of every entry become a key (a << 32 | b) for the
// assembly's bucket sort (any row length: contact scenes give affine-body
// rows tens of thousands of neighbours), then per row the unique
// neighbours without the node itself are counted and emitted.
__global__ void k_graph_keys(const std::uint32_t* __restrict__ rows, const std::uint32_t* __restrict__ cols,
                             std::int64_t U, std::uint64_t* __restrict__ keys) {
    for (std::int64_t e = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; e < U;
         e += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        const std::uint64_t r = rows[e], c = cols[e];
        keys[2 * e] = r << 32 | c;  // a diagonal entry gives self keys, dropped below
        keys[2 * e + 1] = c << 32 | r;
    }
}

// per row of the bucket sort: unique neighbour count without the row itself
// (one warp per row: rows of affine bodies in contact scenes are long)
__global__ void k_adj_count(std::int32_t n, const std::uint64_t* __restrict__ sorted,
                            const std::int64_t* __restrict__ row_start, std::int32_t* __restrict__ cnt) {
    const int lane = threadIdx.x & 31;
    for (std::int64_t r = (blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x) >> 5; r < n;
         r += (static_cast<std::int64_t>(gridDim.x) * blockDim.x) >> 5) {
        const std::int64_t b = row_start[r], e = row_start[r + 1];
        int u = 0;
        for (std::int64_t q = b + lane; q < e; q += 32) {
            const std::uint32_t v = static_cast<std::uint32_t>(sorted[q] >> 32);
            const bool head = q == b || static_cast<std::uint32_t>(sorted[q - 1] >> 32) != v;
            u += (head && v != static_cast<std::uint32_t>(r)) ? 1 : 0;
        }
        for (int o = 16; o > 0; o >>= 1) u += __shfl_xor_sync(0xffffffffu, u, o);
        if (lane == 0) cnt[r] = u;
    }
}

__global__ void k_adj_emit(std::int32_t n, const std::uint64_t* __restrict__ sorted,
                           const std::int64_t* __restrict__ row_start, const std::int64_t* __restrict__ ptr,
                           std::int32_t* __restrict__ adj) {
    const int lane = threadIdx.x & 31;
    for (std::int64_t r = (blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x) >> 5; r < n;
         r += (static_cast<std::int64_t>(gridDim.x) * blockDim.x) >> 5) {
        const std::int64_t b = row_start[r], e = row_start[r + 1];
        std::int64_t o = ptr[r];
        for (std::int64_t q0 = b; q0 < e; q0 += 32) {
            const std::int64_t q = q0 + lane;
            std::uint32_t v = 0;
            bool keep = false;
            if (q < e) {
                v = static_cast<std::uint32_t>(sorted[q] >> 32);
                keep = (q == b || static_cast<std::uint32_t>(sorted[q - 1] >> 32) != v) &&
                       v != static_cast<std::uint32_t>(r);
            }
            const unsigned m = __ballot_sync(0xffffffffu, keep);
            if (keep) adj[o + __popc(m & ((1u << lane) - 1u))] = static_cast<std::int32_t>(v);
            o += __popc(m);
        }
    }
}

struct DeviceGraph {
    const std::int64_t* ptr = nullptr;
    const std::int32_t* adj = nullptr;
    std::int64_t E = 0;
};

DeviceGraph level0_graph_device(Ctx& c) {
    const DeviceMatrix& A = c.A;
    cudaStream_t st = c.stream;
    const std::int32_t n = A.n;
    c.l1_keys.reserve(static_cast<std::size_t>(std::max<std::int64_t>(2 * A.U, 1)));
    if (A.U > 0) {
        k_graph_keys<<<grid_for(A.U, 256, 16), 256, 0, st>>>(A.rows.p, A.cols.p, A.U, c.l1_keys.p);
        ADIPC_LAUNCH_CHECK();
    }
    bucket_sort(c, c.l1_keys.p, 2 * A.U, n, nullptr);
    c.graph_deg.reserve(static_cast<std::size_t>(std::max(n, 1)));
    c.graph_ptr.reserve(static_cast<std::size_t>(n) + 1);
    if (n > 0) {
        k_adj_count<<<grid_for(n, 8, 16), 256, 0, st>>>(n, c.sorted.p, c.row_start.p, c.graph_deg.p);
        ADIPC_LAUNCH_CHECK();
    }
    exclusive_scan(c.graph_deg.p, n, c.graph_ptr.p, c.scan_scratch, st);
    std::int64_t E = 0;
    ADIPC_CUDA(cudaMemcpyAsync(&E, c.graph_ptr.p + n, sizeof(E), cudaMemcpyDeviceToHost, st));
    ADIPC_CUDA(cudaStreamSynchronize(st));
    c.graph_adj.reserve(static_cast<std::size_t>(std::max<std::int64_t>(E, 1)));
    if (n > 0 && E > 0) {
        k_adj_emit<<<grid_for(n, 8, 16), 256, 0, st>>>(n, c.sorted.p, c.row_start.p, c.graph_ptr.p, c.graph_adj.p);
        ADIPC_LAUNCH_CHECK();
    }
    return DeviceGraph{c.graph_ptr.p, c.graph_adj.p, E};
}

// into g, reusing its capacity (the host graphs are kept in the context, so a
// rebuild does not page-fault fresh vectors)
void graph_to_host(Ctx& c, const DeviceGraph& dg, std::int32_t n, host::Graph& g) {
    g.ptr.resize(static_cast<std::size_t>(n) + 1);
    g.adj.resize(static_cast<std::size_t>(dg.E));
    const std::size_t bp = sizeof(std::int64_t) * (static_cast<std::size_t>(n) + 1);
    const std::size_t ba = sizeof(std::int32_t) * static_cast<std::size_t>(dg.E);
    unsigned char* st = static_cast<unsigned char*>(c.stage.reserve(bp + ba));
    ADIPC_CUDA(cudaMemcpyAsync(st, dg.ptr, bp, cudaMemcpyDeviceToHost, c.stream));
    if (dg.E > 0) ADIPC_CUDA(cudaMemcpyAsync(st + bp, dg.adj, ba, cudaMemcpyDeviceToHost, c.stream));
    ADIPC_CUDA(cudaStreamSynchronize(c.stream));
    std::memcpy(g.ptr.data(), st, bp);
    if (ba) std::memcpy(g.adj.data(), st + bp, ba);
}
host::Graph graph_to_host(Ctx& c, const DeviceGraph& dg, std::int32_t n) {
    host::Graph g;
    graph_to_host(c, dg, n, g);
    return g;
}

// ---- the first aggregation pass of build_hierarchy on the device -------------
// (hierarchy.hpp:53-85 for level 0 -> 1): connected components inside each
// level-0 subdomain, numbered in the order of their smallest member (= BFS
// seeds in ascending node order), and the sorted unique super-node graph.
// One warp per subdomain (<= 32 members): lane i = i-th member in ascending
// node order; in-subdomain neighbours as a bit mask; min-label propagation.
__global__ void k_l1_components(std::int32_t n_parts, const std::int32_t* __restrict__ mem_ptr,
                                const std::int32_t* __restrict__ members, const std::int32_t* __restrict__ part_of,
                                const std::int32_t* __restrict__ pos, const std::int64_t* __restrict__ gptr,
                                const std::int32_t* __restrict__ gadj, std::int32_t* __restrict__ up_local,
                                std::int32_t* __restrict__ ncomp) {
    const int lane = threadIdx.x & 31;
    const std::int64_t w = (blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x) >> 5;
    if (w >= n_parts) return;
    const std::int32_t s = static_cast<std::int32_t>(w);
    const std::int32_t m0 = mem_ptr[s], m = mem_ptr[s + 1] - m0;
    const bool act = lane < m;
    const std::int32_t node = act ? members[m0 + lane] : -1;
    unsigned nb = 0;
    if (act) {
        // in-subdomain neighbours lie in [first member, last member] of the
        // sorted adjacency: binary-search the window (affine-body slots have
        // tens of thousands of neighbours, their subdomain a handful)
        const std::int32_t lo = members[m0], hi = members[m0 + m - 1];
        std::int64_t a = gptr[node], b = gptr[node + 1];
        while (a < b) {
            const std::int64_t mid = (a + b) >> 1;
            if (gadj[mid] < lo) a = mid + 1;
            else b = mid;
        }
        std::int64_t z = a, zb = gptr[node + 1];  // end of the window: first neighbour > hi
        while (z < zb) {
            const std::int64_t mid = (z + zb) >> 1;
            if (gadj[mid] <= hi) z = mid + 1;
            else zb = mid;
        }
        if (z - a <= 4 * m) {  // short window: scan it
            for (std::int64_t e2 = a; e2 < z; ++e2) {
                const std::int32_t v = gadj[e2];
                if (part_of[v] == s) nb |= 1u << pos[v];
            }
        } else {  // long window (coarse levels: members spread in id): look each member up
            for (int j = 0; j < m; ++j) {
                const std::int32_t v = members[m0 + j];
                std::int64_t x = a, y = z;
                while (x < y) {
                    const std::int64_t mid = (x + y) >> 1;
                    if (gadj[mid] < v) x = mid + 1;
                    else y = mid;
                }
                if (x < z && gadj[x] == v) nb |= 1u << j;
            }
        }
    }
    int lab = lane;
    for (;;) {
        int best = lab;
        for (int j = 0; j < m; ++j) {
            const int lj = __shfl_sync(0xffffffffu, lab, j);
            if ((nb >> j) & 1u) best = min(best, lj);
        }
        const bool changed = act && best != lab;
        lab = act ? best : lab;
        if (!__any_sync(0xffffffffu, changed)) break;
    }
    const unsigned roots = __ballot_sync(0xffffffffu, act && lab == lane);
    if (act) up_local[node] = __popc(roots & ((1u << lab) - 1u));
    if (lane == 0) ncomp[s] = __popc(roots);
}

__global__ void k_l1_up(std::int32_t n, const std::int32_t* __restrict__ part_of, const std::int64_t* __restrict__ base,
                        std::int32_t* __restrict__ up) {
    for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<std::int64_t>(gridDim.x) * blockDim.x)
        up[i] = static_cast<std::int32_t>(base[part_of[i]] + up[i]);
}


// The super-node keys without the ones the unique pass would drop anyway:
// self loops (up[b] == up[a]) and a repeat of the previous neighbour's super
// node (the adjacency is sorted by fine id, and fine neighbours of one super
// node are mostly consecutive) — about a third of the fine edges survive, so
// the bucket sort moves a third of the keys. One warp per fine node (affine-
// body slots have tens of thousands of neighbours); count, then emit at a
// scanned offset in the same order.
__device__ __forceinline__ bool l1_key_kept(const std::int64_t* gptr, const std::int32_t* gadj, const std::int32_t* up,
                                            std::int64_t a, std::int64_t e, std::int32_t ua, std::int32_t* ub) {
    *ub = up[gadj[e]];
    return *ub != ua && (e == gptr[a] || up[gadj[e - 1]] != *ub);
}
__global__ void k_l1_keycount(std::int32_t n, const std::int64_t* __restrict__ gptr, const std::int32_t* __restrict__ gadj,
                              const std::int32_t* __restrict__ up, std::int32_t* __restrict__ cnt) {
    const int lane = threadIdx.x & 31;
    for (std::int64_t a = (blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x) >> 5; a < n;
         a += (static_cast<std::int64_t>(gridDim.x) * blockDim.x) >> 5) {
        const std::int32_t ua = up[a];
        int c = 0;
        for (std::int64_t e0 = gptr[a]; e0 < gptr[a + 1]; e0 += 32) {
            const std::int64_t e = e0 + lane;
            std::int32_t ub;
            const bool keep = e < gptr[a + 1] && l1_key_kept(gptr, gadj, up, a, e, ua, &ub);
            c += __popc(__ballot_sync(0xffffffffu, keep));
        }
        if (lane == 0) cnt[a] = c;
    }
}
__global__ void k_l1_keyemit(std::int32_t n, const std::int64_t* __restrict__ gptr, const std::int32_t* __restrict__ gadj,
                             const std::int32_t* __restrict__ up, const std::int64_t* __restrict__ off,
                             std::uint64_t* __restrict__ keys) {
    const int lane = threadIdx.x & 31;
    for (std::int64_t a = (blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x) >> 5; a < n;
         a += (static_cast<std::int64_t>(gridDim.x) * blockDim.x) >> 5) {
        const std::int32_t ua = up[a];
        std::int64_t o = off[a];
        for (std::int64_t e0 = gptr[a]; e0 < gptr[a + 1]; e0 += 32) {
            const std::int64_t e = e0 + lane;
            std::int32_t ub = 0;
            const bool keep = e < gptr[a + 1] && l1_key_kept(gptr, gadj, up, a, e, ua, &ub);
            const unsigned m = __ballot_sync(0xffffffffu, keep);
            if (keep)
                keys[o + __popc(m & ((1u << lane) - 1u))] =
                    (static_cast<std::uint64_t>(ua) << 32) | static_cast<std::uint32_t>(ub);
            o += __popc(m);
        }
    }
}

// the compacted super-node keys of graph (gptr, gadj) under the map up into
// c.l1_keys; returns their count
std::int64_t super_keys(Ctx& c, std::int32_t n, const std::int64_t* gptr, const std::int32_t* gadj,
                        const std::int32_t* up) {
    cudaStream_t st = c.stream;
    c.ag_kcnt.reserve(static_cast<std::size_t>(std::max(n, 1)));
    c.ag_koff.reserve(static_cast<std::size_t>(n) + 1);
    k_l1_keycount<<<grid_for(n, 8, 16), 256, 0, st>>>(n, gptr, gadj, up, c.ag_kcnt.p);
    ADIPC_LAUNCH_CHECK();
    exclusive_scan(c.ag_kcnt.p, n, c.ag_koff.p, c.scan_scratch, st);
    std::int64_t k = 0;
    ADIPC_CUDA(cudaMemcpyAsync(&k, c.ag_koff.p + n, sizeof(k), cudaMemcpyDeviceToHost, st));
    ADIPC_CUDA(cudaStreamSynchronize(st));
    c.l1_keys.reserve(static_cast<std::size_t>(std::max<std::int64_t>(k, 1)));
    if (k > 0) {
        k_l1_keyemit<<<grid_for(n, 8, 16), 256, 0, st>>>(n, gptr, gadj, up, c.ag_koff.p, c.l1_keys.p);
        ADIPC_LAUNCH_CHECK();
    }
    return k;
}

// Level 0 -> 1 on the device; false when a level-0 subdomain has more than 32
// members (the host pass handles any size).
bool level1_device(Ctx& c, const DeviceGraph& g0, std::vector<std::int32_t>& up1, std::int32_t& n1,
                   host::Graph& g1) {
    const host::Partition& l0 = c.l0;
    const bool dbg = std::getenv("ADIPC_DEBUG_HIER") != nullptr;
    auto t = std::chrono::steady_clock::now();
    auto lap = [&](const char* what) {
        if (!dbg) return;
        ADIPC_CUDA(cudaStreamSynchronize(c.stream));
        const auto now = std::chrono::steady_clock::now();
        std::fprintf(stderr, "    level-1 pass: %s %.2f ms\n", what, std::chrono::duration<double, std::milli>(now - t).count());
        t = now;
    };
    const std::int32_t n = static_cast<std::int32_t>(l0.part_of.size());
    cudaStream_t st = c.stream;
    if (c.l0_dev_version != c.l0_version) {  // per scene: members of each subdomain, ascending
        std::vector<std::int32_t> mem_ptr(static_cast<std::size_t>(l0.n_parts) + 1, 0), members(n), pos(n);
        for (std::int32_t i = 0; i < n; ++i) pos[i] = mem_ptr[l0.part_of[i] + 1]++;
        c.l0_max_members = 0;
        for (std::int32_t s = 0; s < l0.n_parts; ++s) c.l0_max_members = std::max(c.l0_max_members, mem_ptr[s + 1]);
        for (std::int32_t s = 0; s < l0.n_parts; ++s) mem_ptr[s + 1] += mem_ptr[s];
        for (std::int32_t i = 0; i < n; ++i) members[mem_ptr[l0.part_of[i]] + pos[i]] = i;
        upload(c.l0_part, l0.part_of, st);
        upload(c.l0_mem_ptr, mem_ptr, st);
        upload(c.l0_members, members, st);
        upload(c.l0_pos, pos, st);
        c.l0_dev_version = c.l0_version;
    }
    if (c.l0_max_members > 32 || n == 0 || l0.n_parts == 0) return false;
    c.l1_up.reserve(static_cast<std::size_t>(n));
    c.l1_ncomp.reserve(static_cast<std::size_t>(l0.n_parts));
    c.l1_base.reserve(static_cast<std::size_t>(l0.n_parts) + 1);
    k_l1_components<<<static_cast<int>(ceil_div(l0.n_parts, 8)), 256, 0, st>>>(
        l0.n_parts, c.l0_mem_ptr.p, c.l0_members.p, c.l0_part.p, c.l0_pos.p, g0.ptr, g0.adj, c.l1_up.p, c.l1_ncomp.p);
    ADIPC_LAUNCH_CHECK();
    exclusive_scan(c.l1_ncomp.p, l0.n_parts, c.l1_base.p, c.scan_scratch, st);
    std::int64_t total = 0;
    ADIPC_CUDA(cudaMemcpyAsync(&total, c.l1_base.p + l0.n_parts, sizeof(total), cudaMemcpyDeviceToHost, st));
    ADIPC_CUDA(cudaStreamSynchronize(st));
    n1 = static_cast<std::int32_t>(total);
    lap("components + scan");
    k_l1_up<<<grid_for(n, 256, 16), 256, 0, st>>>(n, c.l0_part.p, c.l1_base.p, c.l1_up.p);
    ADIPC_LAUNCH_CHECK();
    up1.resize(static_cast<std::size_t>(n));
    void* up_stage = c.stage_up.reserve(sizeof(std::int32_t) * static_cast<std::size_t>(n));
    ADIPC_CUDA(cudaMemcpyAsync(up_stage, c.l1_up.p, sizeof(std::int32_t) * n, cudaMemcpyDeviceToHost, st));
    if (n1 == n) {  // no merge: the hierarchy stops at level 0
        ADIPC_CUDA(cudaStreamSynchronize(st));
        std::memcpy(up1.data(), up_stage, sizeof(std::int32_t) * n);
        return true;
    }
    lap("map + D2H");
    // super-node graph: bucket-sort the mapped adjacency, drop repeats and self loops
    const std::int64_t nk = super_keys(c, n, g0.ptr, g0.adj, c.l1_up.p);
    bucket_sort(c, c.l1_keys.p, nk, n1, nullptr);
    lap("keys + bucket sort");
    c.l1_cnt.reserve(static_cast<std::size_t>(n1) + 1);
    c.l1_ptr.reserve(static_cast<std::size_t>(n1) + 1);
    k_adj_count<<<grid_for(n1, 8, 16), 256, 0, st>>>(n1, c.sorted.p, c.row_start.p, c.l1_cnt.p);
    ADIPC_LAUNCH_CHECK();
    exclusive_scan(c.l1_cnt.p, n1, c.l1_ptr.p, c.scan_scratch, st);
    std::int64_t E1 = 0;
    ADIPC_CUDA(cudaMemcpyAsync(&E1, c.l1_ptr.p + n1, sizeof(E1), cudaMemcpyDeviceToHost, st));
    ADIPC_CUDA(cudaStreamSynchronize(st));
    c.l1_adj.reserve(static_cast<std::size_t>(std::max<std::int64_t>(E1, 1)));
    k_adj_emit<<<grid_for(n1, 8, 16), 256, 0, st>>>(n1, c.sorted.p, c.row_start.p, c.l1_ptr.p, c.l1_adj.p);
    ADIPC_LAUNCH_CHECK();
    lap("unique count / emit");
    graph_to_host(c, DeviceGraph{c.l1_ptr.p, c.l1_adj.p, E1}, n1, g1);  // synchronises: up1 has landed too
    std::memcpy(up1.data(), up_stage, sizeof(std::int32_t) * n);
    lap("graph D2H");
    c.l1_E = E1;
    return true;
}

// One aggregation pass (hierarchy.hpp:53-85) above level 1 on the device, for
// a level whose subdomains have <= 32 members: the components inside each
// subdomain (numbered as the BFS seeds), the node map up (to the host too)
// and the next level's sorted unique graph into ag_ptr / ag_adj[out]. False
// when a subdomain is too large (the host continues then).
bool agg_pass_device(Ctx& c, const host::Level& lv, const DeviceGraph& g, int out, std::vector<std::int32_t>& up,
                     std::int32_t& n_next, DeviceGraph& g_next) {
    cudaStream_t st = c.stream;
    const std::int32_t n = lv.n_nodes, np = lv.n_parts;
    const bool dbg = std::getenv("ADIPC_DEBUG_HIER") != nullptr;
    auto t = std::chrono::steady_clock::now();
    auto lap = [&](const char* what) {
        if (!dbg) return;
        ADIPC_CUDA(cudaStreamSynchronize(c.stream));
        const auto now = std::chrono::steady_clock::now();
        std::fprintf(stderr, "      pass (n=%d): %s %.2f ms\n", n, what, std::chrono::duration<double, std::milli>(now - t).count());
        t = now;
    };
    std::vector<std::int32_t> mem_ptr(static_cast<std::size_t>(np) + 1, 0), members(n), pos(n);
    for (std::int32_t i = 0; i < n; ++i) pos[i] = mem_ptr[lv.part_of[i] + 1]++;
    for (std::int32_t s = 0; s < np; ++s)
        if (mem_ptr[s + 1] > 32) return false;
    for (std::int32_t s = 0; s < np; ++s) mem_ptr[s + 1] += mem_ptr[s];
    for (std::int32_t i = 0; i < n; ++i) members[mem_ptr[lv.part_of[i]] + pos[i]] = i;
    upload(c.ag_part, lv.part_of, st);
    upload(c.ag_mem_ptr, mem_ptr, st);
    upload(c.ag_members, members, st);
    upload(c.ag_pos, pos, st);
    lap("member lists + uploads");
    c.ag_up.reserve(static_cast<std::size_t>(n));
    c.ag_ncomp.reserve(static_cast<std::size_t>(np));
    c.ag_base.reserve(static_cast<std::size_t>(np) + 1);
    k_l1_components<<<static_cast<int>(ceil_div(np, 8)), 256, 0, st>>>(np, c.ag_mem_ptr.p, c.ag_members.p, c.ag_part.p,
                                                                     c.ag_pos.p, g.ptr, g.adj, c.ag_up.p, c.ag_ncomp.p);
    ADIPC_LAUNCH_CHECK();
    lap("components kernel");
    exclusive_scan(c.ag_ncomp.p, np, c.ag_base.p, c.scan_scratch, st);
    lap("scan");
    k_l1_up<<<grid_for(n, 256, 16), 256, 0, st>>>(n, c.ag_part.p, c.ag_base.p, c.ag_up.p);
    ADIPC_LAUNCH_CHECK();
    std::int64_t total = 0;
    up.resize(static_cast<std::size_t>(n));
    ADIPC_CUDA(cudaMemcpyAsync(&total, c.ag_base.p + np, sizeof(total), cudaMemcpyDeviceToHost, st));
    ADIPC_CUDA(cudaMemcpyAsync(up.data(), c.ag_up.p, sizeof(std::int32_t) * n, cudaMemcpyDeviceToHost, st));
    ADIPC_CUDA(cudaStreamSynchronize(st));
    n_next = static_cast<std::int32_t>(total);
    lap("components + map + D2H");
    if (n_next == n) return true;
    const std::int64_t nk = super_keys(c, n, g.ptr, g.adj, c.ag_up.p);
    lap("keys");
    bucket_sort(c, c.l1_keys.p, nk, n_next, nullptr);
    lap("bucket sort");
    c.ag_cnt.reserve(static_cast<std::size_t>(n_next) + 1);
    c.ag_ptr[out].reserve(static_cast<std::size_t>(n_next) + 1);
    k_adj_count<<<grid_for(n_next, 8, 16), 256, 0, st>>>(n_next, c.sorted.p, c.row_start.p, c.ag_cnt.p);
    ADIPC_LAUNCH_CHECK();
    exclusive_scan(c.ag_cnt.p, n_next, c.ag_ptr[out].p, c.scan_scratch, st);
    std::int64_t E = 0;
    ADIPC_CUDA(cudaMemcpyAsync(&E, c.ag_ptr[out].p + n_next, sizeof(E), cudaMemcpyDeviceToHost, st));
    ADIPC_CUDA(cudaStreamSynchronize(st));
    c.ag_adj[out].reserve(static_cast<std::size_t>(std::max<std::int64_t>(E, 1)));
    k_adj_emit<<<grid_for(n_next, 8, 16), 256, 0, st>>>(n_next, c.sorted.p, c.row_start.p, c.ag_ptr[out].p,
                                                      c.ag_adj[out].p);
    ADIPC_LAUNCH_CHECK();
    g_next = DeviceGraph{c.ag_ptr[out].p, c.ag_adj[out].p, E};
    return true;
}

// build_hierarchy from the device level-1 pass (hierarchy.hpp:30-100): the
// partitions (sequential carving) on the host, every aggregation pass above
// level 1 on the device while its subdomains fit a warp
host::MasHierarchy hierarchy_from_level1(Ctx& c, std::vector<std::int32_t> up1, std::int32_t n1, const host::Graph& g1) {
    host::MasHierarchy h = host::hierarchy_base(c.l0);
    if (h.n_levels() >= c.max_levels || c.l0.n_parts <= 1 || n1 == h.n_slots) return h;
    const bool dbg = std::getenv("ADIPC_DEBUG_HIER") != nullptr;
    auto t = std::chrono::steady_clock::now();
    auto lap = [&](const char* what, int l) {
        if (!dbg) return;
        const auto now = std::chrono::steady_clock::now();
        std::fprintf(stderr, "  level %d %s %.2f ms\n", l, what, std::chrono::duration<double, std::milli>(now - t).count());
        t = now;
    };
    host::append_level(h, std::move(up1), n1, g1);  // level-1 partition (host carve)
    lap("partition", 1);
    DeviceGraph gcur{c.l1_ptr.p, c.l1_adj.p, c.l1_E};
    int out = 0;
    while (h.n_levels() < c.max_levels && h.levels.back().n_parts > 1) {
        std::vector<std::int32_t> up;
        std::int32_t n_next = 0;
        DeviceGraph gn{};
        if (!agg_pass_device(c, h.levels.back(), gcur, out, up, n_next, gn)) {  // subdomains beyond a warp
            host::Graph gh = graph_to_host(c, gcur, h.levels.back().n_nodes);
            host::extend_from(h, std::move(gh), c.max_levels);
            break;
        }
        if (n_next == h.levels.back().n_nodes) break;
        host::Graph& ghn = c.host_graph[out];
        graph_to_host(c, gn, n_next, ghn);
        lap("aggregation (device)", h.n_levels());
        host::append_level(h, std::move(up), n_next, ghn);
        lap("partition", h.n_levels() - 1);
        gcur = gn;
        out ^= 1;
    }
    return h;
}

}  // namespace

void build_preconditioner(Ctx& c, PrecondKind kind) {
    cudaStream_t st = c.stream;
    const DeviceMatrix& A = c.A;
    if (kind == kJacobi) {
        c.jinv.reserve(9 * static_cast<std::size_t>(A.n));
        if (A.n > 0) {
            k_jacobi_build<<<grid_for(A.n, 256, 16), 256, 0, st>>>(A.n, A.cols.p, A.blocks.p, A.U, A.row_ptr.p, c.jinv.p);
            ADIPC_LAUNCH_CHECK();
        }
        c.pkind = kJacobi;
        c.jinv_n = A.n;
        c.perm_active = false;
        return;
    }
    if (!c.have_l0) throw StatusError(kInvalidArgument, "level-0 partition not set (adipc_gpu_set_level0_partition)");
    if (static_cast<std::int32_t>(c.l0.part_of.size()) != A.n)
        throw StatusError(kInvalidArgument, "level-0 partition size differs from n_block_rows");
    const auto t0 = std::chrono::steady_clock::now();
    // The hierarchy is a pure function of (level-0 partition, sparsity
    // pattern, max_levels): with ADIPC_OPT_CACHE_HIERARCHY it is reused while
    // the pattern hash is unchanged (e.g. Newton iterations without contact
    // changes); restriction and inversion always rerun on the new values.
    const std::uint64_t phash = c.cache_hierarchy ? pattern_hash(c) : 0;
    const bool reuse = c.cache_hierarchy && c.hier_version == phash && !c.levels.empty();
    // block_edges(A) (mas.hpp:19-25): off-diagonal (row, col) pairs, in order
    if (!reuse) {
        // the level-0 graph built on the device from A's pattern and — for
        // subdomains of <= 32 members — the first aggregation pass too; the
        // host continues from the (small) level-1 graph
        const DeviceGraph g0 = level0_graph_device(c);
        const auto tg = std::chrono::steady_clock::now();
        std::vector<std::int32_t> up1;
        std::int32_t n1 = 0;
        host::Graph& g1 = c.host_graph[2];
        const bool dev_l1 = c.max_levels > 1 && c.l0.n_parts > 1 && level1_device(c, g0, up1, n1, g1);
        const auto ta = std::chrono::steady_clock::now();
        if (std::getenv("ADIPC_DEBUG_HIER"))
            std::fprintf(stderr, "  level-0 graph (device, E=%lld) %.2f ms, level-1 pass + D2H %.2f ms\n",
                         static_cast<long long>(g0.E), std::chrono::duration<double, std::milli>(tg - t0).count(),
                         std::chrono::duration<double, std::milli>(ta - tg).count());
        if (dev_l1 && c.solve_order && A.n > 0) {
            // level 0 (cached per scene) is factored on the device while the
            // host builds the coarse levels: As, restriction and inversion of
            // level 0 are queued before the host hierarchy and overlap it
            ensure_level0(c);
            c.perm_active = true;
            build_solve_matrix(c, false);
            factor_begin(c);
            factor_levels(c, 0, 1);
            const auto tq = std::chrono::steady_clock::now();
            c.hier = hierarchy_from_level1(c, std::move(up1), n1, g1);
            if (c.hier.n_levels() > kMaxLevels) throw StatusError(kInvalidArgument, "too many MAS levels");
            const auto tb = std::chrono::steady_clock::now();
            set_coarse_levels(c, c.hier);
            c.as_src_version = c.levels_version;  // the As map depends on perm and the pattern only
            c.hier_version = c.cache_hierarchy ? phash : ~0ull;
            c.ms_build_host = std::chrono::duration<float, std::milli>(std::chrono::steady_clock::now() - t0).count();
            if (std::getenv("ADIPC_DEBUG_HIER")) {
                auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
                std::fprintf(stderr, "cold MAS host (level 0 overlapped): block_edges %.1f ms, level 0 + As queued %.1f ms, "
                                     "build_hierarchy %.1f ms, coarse levels %.1f ms\n",
                             ms(t0, ta), ms(ta, tq), ms(tq, tb), ms(tb, std::chrono::steady_clock::now()));
            }
            factor_levels(c, 1, static_cast<int>(c.levels.size()));
            factor_end(c);
            return;
        }
        if (dev_l1)
            c.hier = host::build_hierarchy_l1(c.l0, std::move(up1), n1, std::move(g1), c.max_levels);
        else
            c.hier = host::build_hierarchy(c.l0, graph_to_host(c, g0, A.n), c.max_levels);
        if (c.hier.n_levels() > kMaxLevels) throw StatusError(kInvalidArgument, "too many MAS levels");
        const auto tb = std::chrono::steady_clock::now();
        set_levels(c, c.hier);
        c.hier_version = c.cache_hierarchy ? phash : ~0ull;
        if (std::getenv("ADIPC_DEBUG_HIER")) {
            const auto tc = std::chrono::steady_clock::now();
            auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
            std::fprintf(stderr, "cold MAS host: block_edges %.1f ms, build_hierarchy %.1f ms, device levels %.1f ms\n",
                         ms(t0, ta), ms(ta, tb), ms(tb, tc));
        }
    }
    const auto t1 = std::chrono::steady_clock::now();
    c.ms_build_host = std::chrono::duration<float, std::milli>(t1 - t0).count();
    c.perm_active = c.levels_permuted;
    if (c.perm_active) build_solve_matrix(c, reuse);
    factorize(c);
}

void build_mas_from_hierarchy(Ctx& c, const host::MasHierarchy& h) {
    const auto t0 = std::chrono::steady_clock::now();
    if (h.n_levels() > kMaxLevels) throw StatusError(kInvalidArgument, "too many MAS levels");
    c.hier = h;
    set_levels(c, c.hier);
    c.hier_version = ~0ull;  // explicit hierarchies are never reused by the cache
    c.ms_build_host = std::chrono::duration<float, std::milli>(std::chrono::steady_clock::now() - t0).count();
    c.perm_active = c.levels_permuted;
    if (c.perm_active) build_solve_matrix(c, false);
    factorize(c);
}

// ---------------------------------------------------------------------------
// launch helpers shared with pcg.cu
int level_grid(const Ctx& c, int l) {
    const DeviceLevel& L = *c.levels[l];
    // one subdomain per warp (kLevelWarps per CTA), no grid-stride: the block
    // scheduler balances the memory-bound warps; fills > 32 take a CTA each
    const std::int64_t per = L.max_fill > 32 ? 1 : kLevelWarps;
    return static_cast<int>(std::max<std::int64_t>(1, ceil_div(L.n_parts, per)));
}
int slot_grid(const Ctx& c) { return grid_for(3 * static_cast<std::int64_t>(c.A.n), 256, 8); }
int jacobi_grid(const Ctx& c) { return grid_for(c.A.n, 256, 8); }

// lanes hold dims j = lane + 32 t, t < regs; fills above 32 use the CTA kernel
static int dim_regs(int max_fill) { return max_fill <= 10 ? 1 : (max_fill <= 21 ? 2 : (max_fill <= 32 ? 3 : 0)); }

LevelArgs level_args(Ctx& c, int l, const double* r_in, double* out) {
    DeviceLevel& L = *c.levels[l];
    const bool top = l + 1 >= static_cast<int>(c.levels.size());
    LevelArgs la{};
    la.n_parts = L.n_parts;
    la.sub_ptr = L.sub_ptr.p;
    la.sub_nodes = L.sub_nodes.p;
    la.inv_off = L.inv_off.p;
    la.inv = L.inv.p;
    la.r_in = l == 0 ? r_in : L.rr.p;
    la.out = l == 0 ? out : L.y.p;
    la.up_first = top ? nullptr : L.up_first.p;
    la.upc_ptr = top ? nullptr : L.upc_ptr.p;
    la.upc_pos = top ? nullptr : L.upc_pos.p;
    la.r_next = top ? nullptr : c.levels[l + 1]->rr.p;
    return la;
}

// Level-l MAS solve (+ restriction to level l+1). Level 0 uses `kMode`
// (apply / PCG gather modes); coarser levels read their restricted residual.
// kSolve = false: gather + restriction only (the PCG update pass);
// restrict_next = false: no restriction (the level-0 solve of the PCG, whose
// restriction was done by the update pass).
template <int kMode, bool kSolve>
void launch_level(Ctx& c, int l, const double* r_in, double* z, const PcgArgs& a, double* partials,
                  unsigned* ticket, double* dot_out, cudaStream_t st, bool restrict_next) {
    LevelArgs la = level_args(c, l, r_in, z);
    if (!restrict_next) la.r_next = nullptr;
    const DeviceLevel& L = *c.levels[l];
    const int regs = dim_regs(L.max_fill);
    const int grid = level_grid(c, l);
    if (regs == 0) {
        const std::size_t smem = sizeof(double) * 3 * L.max_fill;
        ADIPC_CUDA(cudaFuncSetAttribute(k_mas_level_big<kMode, kSolve>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(smem)));
        k_mas_level_big<kMode, kSolve><<<grid, 128, smem, st>>>(la, a, partials, ticket, dot_out);
    } else {
        const int ws = static_cast<int>(level_warp_smem(kSolve ? 3 * L.max_fill : 0, regs));
        const std::size_t smem = static_cast<std::size_t>(kLevelWarps) * ws;
        const int block = 32 * kLevelWarps;
#define ADIPC_LVL(R)                                                                                           \
    do {                                                                                                       \
        /* per-device attribute: set on every launch (cheap, legal while capturing) */                        \
        ADIPC_CUDA(cudaFuncSetAttribute(k_mas_level<kMode, R, kSolve>,                                         \
                                        cudaFuncAttributeMaxDynamicSharedMemorySize,                           \
                                        static_cast<int>(kLevelWarps * level_warp_smem(32 * R, R))));          \
        k_mas_level<kMode, R, kSolve><<<grid, block, smem, st>>>(la, a, partials, ticket, dot_out, ws);        \
    } while (0)
        if (regs == 1)
            ADIPC_LVL(1);
        else if (regs == 2)
            ADIPC_LVL(2);
        else
            ADIPC_LVL(3);
#undef ADIPC_LVL
    }
    ADIPC_LAUNCH_CHECK();
}
#define ADIPC_INST(M, S)                                                                                      \
    template void launch_level<M, S>(Ctx&, int, const double*, double*, const PcgArgs&, double*, unsigned*, \
                                     double*, cudaStream_t, bool);
ADIPC_INST(M_APPLY, true)
ADIPC_INST(M_COARSE, true)
ADIPC_INST(M_INIT, false)
ADIPC_INST(M_UPDATE, false)
ADIPC_INST(M_RESTART, false)
#undef ADIPC_INST

ProlongArgs prolong_args(const Ctx& c) {
    ProlongArgs pa{};
    pa.n_levels = c.pkind == kMas ? static_cast<int>(c.levels.size()) - 1 : 0;
    pa.n_rz = c.pkind == kMas ? static_cast<int>(c.levels.size()) : 1;
    for (int l = 0; l < pa.n_levels; ++l) {
        pa.agg[l] = c.levels[l + 1]->agg.p;
        pa.y[l] = c.levels[l + 1]->y.p;
    }
    return pa;
}

template <int kFinal>
void launch_final(Ctx& c, double* z, double* p, double* ap, const PcgArgs& a) {
    k_mas_final<kFinal><<<slot_grid(c), 256, 0, c.stream>>>(c.A.n, prolong_args(c), z, p, ap, a);
    ADIPC_LAUNCH_CHECK();
}
template void launch_final<F_APPLY>(Ctx&, double*, double*, double*, const PcgArgs&);
template void launch_final<F_PCG_INIT>(Ctx&, double*, double*, double*, const PcgArgs&);
template void launch_final<F_PCG_STEP>(Ctx&, double*, double*, double*, const PcgArgs&);

template <int kMode>
void launch_jacobi(Ctx& c, const double* r_in, double* z, const PcgArgs& a, double* partials, unsigned* ticket,
                   double* dot_out) {
    k_jacobi<kMode><<<jacobi_grid(c), 256, 0, c.stream>>>(c.A.n, c.jinv.p, r_in, z, a, partials, ticket, dot_out);
    ADIPC_LAUNCH_CHECK();
}
template void launch_jacobi<M_APPLY>(Ctx&, const double*, double*, const PcgArgs&, double*, unsigned*, double*);
template void launch_jacobi<M_INIT>(Ctx&, const double*, double*, const PcgArgs&, double*, unsigned*, double*);
template void launch_jacobi<M_UPDATE>(Ctx&, const double*, double*, const PcgArgs&, double*, unsigned*, double*);
template void launch_jacobi<M_RESTART>(Ctx&, const double*, double*, const PcgArgs&, double*, unsigned*, double*);

namespace {
__global__ void k_permute_vec(std::int32_t n, const std::int32_t* __restrict__ perm, const double* __restrict__ src,
                              double* __restrict__ dst, bool to_solve) {
    const std::int64_t n3 = 3 * static_cast<std::int64_t>(n);
    for (std::int64_t g = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; g < n3;
         g += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        const std::int64_t i = g / 3, k = g - 3 * i;
        const std::int64_t q = 3 * static_cast<std::int64_t>(perm[i]) + k;
        if (to_solve)
            dst[q] = src[g];
        else
            dst[g] = src[q];
    }
}
}  // namespace

void permute_vec(Ctx& c, const double* src, double* dst, bool to_solve) {
    if (c.A.n == 0) return;
    k_permute_vec<<<slot_grid(c), 256, 0, c.stream>>>(c.A.n, c.perm.p, src, dst, to_solve);
    ADIPC_LAUNCH_CHECK();
}

// z = M r (MasPreconditioner::apply / BlockJacobiPreconditioner::apply).
void precond_apply(Ctx& c, const double* d_r, double* d_z) {
    PcgArgs a{};
    check_precond_size(c);
    if (c.A.n == 0) return;
    if (c.pkind == kMas && c.perm_active) {  // run in solve order
        const std::size_t n3 = 3 * static_cast<std::size_t>(c.A.n);
        c.pv_in.reserve(n3);
        c.pv_out.reserve(n3);
        permute_vec(c, d_r, c.pv_in.p, true);
        launch_level<M_APPLY, true>(c, 0, c.pv_in.p, c.pv_out.p, a, nullptr, nullptr, nullptr, c.stream, true);
        for (int l = 1; l < static_cast<int>(c.levels.size()); ++l)
            launch_level<M_COARSE, true>(c, l, nullptr, nullptr, a, nullptr, nullptr, nullptr, c.stream, true);
        launch_final<F_APPLY>(c, c.pv_out.p, nullptr, nullptr, a);
        permute_vec(c, c.pv_out.p, d_z, false);
        return;
    }
    if (c.pkind == kJacobi) {
        launch_jacobi<M_APPLY>(c, d_r, d_z, a, nullptr, nullptr, nullptr);
    } else if (c.pkind == kMas) {
        launch_level<M_APPLY, true>(c, 0, d_r, d_z, a, nullptr, nullptr, nullptr, c.stream, true);
        for (int l = 1; l < static_cast<int>(c.levels.size()); ++l)
            launch_level<M_COARSE, true>(c, l, nullptr, nullptr, a, nullptr, nullptr, nullptr, c.stream, true);
        launch_final<F_APPLY>(c, d_z, nullptr, nullptr, a);
    } else {
        throw StatusError(kInvalidArgument, "no preconditioner built");
    }
}

}  // namespace adipc_gpu
