// PCG iteration kernels of the solve order (Ctx::perm active: every level-0
// subdomain is a contiguous slot range, slots in pos_of order). The iteration
// (pcg.hpp:59-85) becomes:
//   1. SpMV + p.Ap                                  (spmv.cu)
//   2. k_update_so: alpha, x += alpha p, r -= alpha Ap as a unit-stride stream
//      over each CTA's run of level-0 subdomains; the level-1 restricted
//      residual from the CTA's shared-memory copy of r (children in ascending
//      order, as the tree restriction of mas_kernels.cuh); levels >= 2 get the
//      level-1 sums by fp64 RED up the nesting (r_{l+1}[w] = sum of r_l over
//      the level-l nodes inside w, hierarchy.hpp:53-72), so every coarse level
//      is ready at once
//   3. k_l0_solve_so (level-0 dense solves, persistent warps, each streaming
//      its run of packed inverses through a ring of TMA bulk copies) on the
//      solve stream, concurrently with k_coarse_so (all coarse levels in ONE
//      launch, one warp per subdomain of any level) on the side stream
//   4. k_final_so: z = ((z0 + y1[agg1]) + y2[agg2]) + ... (mas.hpp:95-96
//      order), the convergence test, p = z + beta p, Ap cleared, the RED
//      targets of step 2 cleared for the next iteration.
// r.z comes from the per-level partial dots b_l.y_l of step 3 (the same
// quantity: r.z = sum_l (P_l r).(D_l^-1 P_l r)).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include <cooperative_groups.h>

#include "mas_kernels.cuh"

namespace adipc_gpu {

namespace {

constexpr int kUpdThreads = 256;
constexpr int kUpdSubs = 32;  // level-0 subdomains per CTA of the update pass

struct SoRestrict {
    int n_levels;                        // total levels L (>= 2 when used)
    std::int32_t n0_parts;               // level-0 subdomains
    const std::int32_t* sub_ptr0;        // level-0 subdomain -> first solve slot
    const std::int32_t* up_first0;       // level-0 subdomain -> first level-1 node
    const std::int32_t* upc_ptr0;        // level-1 node -> children range
    const std::int32_t* upc_node0;       // children (solve slots), ascending
    double* rr[kMaxLevels];              // restricted residual of level l >= 1 (3 per node)
    const std::int32_t* up_node[kMaxLevels];  // level-l node -> level-(l+1) node, l >= 1
    const std::int32_t* anc[kMaxLevels];      // level-1 node -> its level-l node, l >= 2
    int max_fill0;                            // largest level-0 subdomain (tile smem sizing)
    int subs;                                 // level-0 subdomains per tile
};

// One tile of kUpdSubs level-0 subdomains of the update pass (solve order):
// the vector update as a unit-stride stream, r kept in shared memory, then
// the level-1 restricted residual of the level-1 nodes nested in the tile.
// In solve order the tile's slots are [sub_ptr0[s0], sub_ptr0[s1]) and the
// children lists of its level-1 nodes are exactly upc_node0 over that same
// range (CSR in node order), so all restriction metadata is fetched with
// coalesced loads issued together with the vector stream. Levels >= 2 take
// the level-1 sums by RED through the precomputed ancestors (no dependent
// chain). smem: 3 * slots doubles, then (slots + 1 + slots) ints.
template <int kMode, int kThreads>
__device__ __forceinline__ void update_tile(const SoRestrict& so, const PcgArgs& a, double alpha,
                                            const double* __restrict__ apv, std::int32_t tile, double* smem) {
    const std::int32_t s0 = tile * so.subs;
    const std::int32_t s1 = min(s0 + so.subs, so.n0_parts);
    const std::int32_t slot0 = so.sub_ptr0[s0], slot1 = so.sub_ptr0[s1];
    const std::int32_t v0 = so.up_first0[s0], v1 = so.up_first0[s1];
    const std::int64_t g0 = 3 * static_cast<std::int64_t>(slot0);
    const std::int64_t g1 = 3 * static_cast<std::int64_t>(slot1);
    const int cap = so.subs * so.max_fill0;
    double* sr = smem;
    int* uptr = reinterpret_cast<int*>(smem + 3 * cap);
    int* child = uptr + cap + 1;
    for (int i = threadIdx.x; i <= v1 - v0; i += kThreads) uptr[i] = so.upc_ptr0[v0 + i] - slot0;
    for (int i = threadIdx.x; i < slot1 - slot0; i += kThreads) child[i] = so.upc_node0[slot0 + i] - slot0;
    constexpr int kU = 4;
    for (std::int64_t gb = g0 + threadIdx.x; gb < g1; gb += kU * kThreads) {
        double rv[kU], pv[kU], av[kU], xv[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const std::int64_t g = gb + u * kThreads;
            if (g < g1) {
                av[u] = apv[g];
                if (kMode == M_UPDATE) {
                    rv[u] = a.r[g];
                    pv[u] = a.p[g];
                    xv[u] = a.x[g];
                } else {
                    rv[u] = a.b[g];
                }
            }
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const std::int64_t g = gb + u * kThreads;
            if (g < g1) {
                double nr;
                if (kMode == M_UPDATE) {
                    a.x[g] = xv[u] + alpha * pv[u];
                    nr = rv[u] - alpha * av[u];
                } else {  // M_RESTART: r = b - A x (x updated before the restart SpMV)
                    nr = rv[u] - av[u];
                }
                a.r[g] = nr;
                sr[g - g0] = nr;
            }
        }
    }
    __syncthreads();
    for (int t = threadIdx.x; t < 3 * (v1 - v0); t += kThreads) {
        const int i = t / 3, comp = t % 3;
        const std::int32_t v = v0 + i;
        std::int32_t w[kMaxLevels];
#pragma unroll
        for (int l = 2; l < kMaxLevels; ++l)
            if (l < so.n_levels) w[l] = so.anc[l][v];
        double acc = 0;
        for (int q = uptr[i]; q < uptr[i + 1]; ++q) acc += sr[3 * child[q] + comp];
        so.rr[1][3 * static_cast<std::int64_t>(v) + comp] = acc;
#pragma unroll
        for (int l = 2; l < kMaxLevels; ++l)
            if (l < so.n_levels) red_add(so.rr[l] + 3 * static_cast<std::int64_t>(w[l]) + comp, acc);
    }
    __syncthreads();
}

inline std::size_t update_tile_smem(int max_fill0, int subs) {
    const std::size_t cap = static_cast<std::size_t>(subs) * max_fill0;
    return sizeof(double) * 3 * cap + sizeof(int) * (2 * cap + 1);
}

template <int kMode>
__global__ void __launch_bounds__(kUpdThreads) k_update_so(SoRestrict so, PcgArgs a) {
    extern __shared__ double sr[];
    double alpha = 0;
    pdl_wait();
    if (a.flags[F_DONE]) return;
    if (!pcg_alpha(a, alpha)) return;
    pdl_launch();
    update_tile<kMode, kUpdThreads>(so, a, alpha, a.ap, blockIdx.x, sr);
}

// ---- level-0 solve: persistent warp pairs, TMA ring of packed inverses -------
// Each pair of warps owns a contiguous run of subdomains and keeps kStages
// packed inverses in flight (cp.async.bulk, L2 evict-first) in its shared
// ring; the two warps split the rows of every subdomain (kK/2 each), so the
// ring's shared memory feeds twice the warps and each warp's unrolled
// mat-vec is half as long. The residual of the next subdomain is loaded one
// subdomain ahead. Pairs per CTA = blockDim.x / 64 (sized to the ring).
__device__ __forceinline__ void pair_sync(int pair) {
    asm volatile("bar.sync %0, 64;" ::"r"(pair + 1) : "memory");
}

// Every level of the preconditioner in one persistent launch: the work list
// is level 0's subdomains followed by each coarse level's (their restricted
// residuals were all produced by the update pass), so there is no side stream
// and no second kernel competing for the shared memory of the rings.
struct PrecondTable {
    int n;                                   // levels
    std::int32_t base[kMaxLevels + 1];       // prefix sums of subdomain counts
    const std::int32_t* sub_ptr[kMaxLevels];
    const std::int32_t* sub_nodes[kMaxLevels];  // null at level 0 (solve order: contiguous slots)
    const std::int64_t* inv_off[kMaxLevels];
    const double* inv[kMaxLevels];
    const double* rin[kMaxLevels];           // level 0: r; coarse: restricted residual
    double* out[kMaxLevels];                 // level 0: z; coarse: y
    int dbg_nomath;                          // timing experiments only
    std::int64_t l0_keep;                    // level-0 inverse doubles below this offset stream L2 evict-last
    // byte-balanced work split: split[l * (np + 1) + p] = first subdomain of
    // level l for work unit p (np units), cut at equal packed-inverse bytes
    const std::int32_t* split;
    int np;
};

template <int kK, int kStages>
__global__ void __launch_bounds__(320) k_precond_so(PrecondTable pt, double* __restrict__ partials,
                                                   unsigned* __restrict__ ticket, double* __restrict__ dot_out,
                                                   const int* __restrict__ flags, int slot_doubles) {
    constexpr int RB = (kK + 31) / 32;  // b entries per lane
    extern __shared__ __align__(128) unsigned char smem[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, pair = w >> 1, half = w & 1;
    const int npc = blockDim.x >> 6;
    double* ring = reinterpret_cast<double*>(smem) + static_cast<std::size_t>(pair) * kStages * slot_doubles;
    // one b per pair: both warps write the same values into it after the
    // pair barrier that ends the previous item, then read it after their own
    // __syncwarp (no cross-warp dependency)
    double* bs = reinterpret_cast<double*>(smem) + static_cast<std::size_t>(npc) * kStages * slot_doubles +
                 static_cast<std::size_t>(pair) * kK;
    std::uint64_t* bar = reinterpret_cast<std::uint64_t*>(
                             reinterpret_cast<double*>(smem) + static_cast<std::size_t>(npc) * kStages * slot_doubles +
                             static_cast<std::size_t>(npc) * kK) +
                         pair * kStages;
    // every pair takes an even share of EACH level (a contiguous run per
    // level, level 0 first): the coarse items, cheap in bytes but with a
    // longer gather chain, are spread over all pairs instead of piling up at
    // the end of the work list
    const std::int64_t gp = static_cast<std::int64_t>(blockIdx.x) * npc + pair;
    const std::int64_t np = static_cast<std::int64_t>(gridDim.x) * npc;
    std::int32_t lv_lo[kMaxLevels], lv_n[kMaxLevels];
    int nloc = 0;
#pragma unroll
    for (int l = 0; l < kMaxLevels; ++l) {
        lv_lo[l] = lv_n[l] = 0;
        if (l < pt.n) {
            std::int32_t a, b;
            if (pt.split && pt.np == np) {
                a = pt.split[l * (np + 1) + gp];
                b = pt.split[l * (np + 1) + gp + 1];
            } else {
                const std::int64_t nl = pt.base[l + 1] - pt.base[l];
                a = static_cast<std::int32_t>(gp * nl / np);
                b = static_cast<std::int32_t>((gp + 1) * nl / np);
            }
            lv_lo[l] = pt.base[l] + a;
            lv_n[l] = b - a;
            nloc += lv_n[l];
        }
    }
    auto item = [&](int i) -> std::int32_t {
#pragma unroll
        for (int l = 0; l < kMaxLevels; ++l) {
            if (i < lv_n[l]) return lv_lo[l] + i;
            i -= lv_n[l];
        }
        return 0;
    };
    auto level_of = [&](std::int32_t q) {
        int l = 0;
        while (l + 1 < pt.n && q >= pt.base[l + 1]) ++l;
        return l;
    };
    // finite slot contents beyond each inverse (packed_matvec reads them x 0)
    for (int i = half * 32 + lane; i < kStages * slot_doubles; i += 64) ring[i] = 0.0;
    fence_proxy_async();
    pair_sync(pair);
    auto issue = [&](std::int32_t q, int st) {  // one thread of the pair
        const int l = level_of(q);
        const std::int32_t s = q - pt.base[l];
        const std::int64_t o = pt.inv_off[l][s];
        const std::uint32_t bytes = static_cast<std::uint32_t>((pt.inv_off[l][s + 1] - o) * 8);
        mbar_arrive_expect_tx(&bar[st], bytes);
        if (l == 0 && o >= pt.l0_keep)  // streamed once per application
            bulk_g2s_evict_first(ring + static_cast<std::size_t>(st) * slot_doubles, pt.inv[0] + o, bytes, &bar[st]);
        else  // coarse inverses (~26 MB at cfg5) and the kept share of level 0 stay L2-resident across iterations
            bulk_g2s_evict_last(ring + static_cast<std::size_t>(st) * slot_doubles, pt.inv[l] + o, bytes, &bar[st]);
    };
    if (half == 0 && lane == 0) {
        for (int st = 0; st < kStages; ++st) mbar_init(&bar[st], 1);
        fence_mbar_init();
        for (int st = 0; st < kStages && st < nloc; ++st) issue(item(st), st);
    }
    pair_sync(pair);
    // the inverses are constant during the solve: the ring above fills while
    // the predecessor (update pass) drains; its outputs are read from here on
    pdl_wait();
    if (flags && flags[F_DONE]) {  // PCG already finished: drain the issued copies, leave
        if (half == 0 && lane == 0)
            for (int st = 0; st < kStages && st < nloc; ++st) mbar_wait(&bar[st], 0);
        return;
    }
    pdl_launch();
    // b of a work item and the addresses of its rows (gathered for coarse levels)
    struct Item {
        int l;
        std::int32_t s0, dim;
    };
    auto row_index = [&](const Item& it, int j) -> std::int64_t {
        if (it.l == 0) return 3 * static_cast<std::int64_t>(it.s0) + j;
        return 3 * static_cast<std::int64_t>(pt.sub_nodes[it.l][it.s0 + j / 3]) + (j % 3);
    };
    auto load_b = [&](std::int32_t q, Item& it, double* bb) {
        it.l = level_of(q);
        const std::int32_t s = q - pt.base[it.l];
        it.s0 = pt.sub_ptr[it.l][s];
        it.dim = 3 * (pt.sub_ptr[it.l][s + 1] - it.s0);
#pragma unroll
        for (int t = 0; t < RB; ++t) {
            const int j = lane + 32 * t;
            bb[t] = j < it.dim ? ldg_issue(pt.rin[it.l] + row_index(it, j)) : 0.0;
        }
    };
    Item cur{0, 0, 0};
    double b[RB];
    if (nloc > 0) load_b(item(0), cur, b);
    double dsum = 0;
    int st = 0;
    std::uint32_t par = 0;
    for (int i = 0; i < nloc; ++i) {
#pragma unroll
        for (int t = 0; t < RB; ++t)
            if (lane + 32 * t < kK) bs[lane + 32 * t] = b[t];
        Item nxt{0, 0, 0};
        double bn[RB];
        if (i + 1 < nloc) load_b(item(i + 1), nxt, bn);
        __syncwarp();
        mbar_wait(&bar[st], par);
        const double* M = ring + static_cast<std::size_t>(st) * slot_doubles;
        double* out = pt.out[cur.l];
        auto refill = [&] {
            pair_sync(pair);  // both warps are done with the slot
            if (half == 0 && lane == 0 && i + kStages < nloc) {  // refill kStages items ahead
                fence_proxy_async();
                issue(item(i + kStages), st);
            }
        };
        if (pt.dbg_nomath)  // timing experiments: stream the inverses, skip the mat-vec
            dsum += M[lane] * bs[lane];
        else
            dsum += pair_solve<kK>(M, bs, lane, half, cur.dim,
                                   [&](int j, double v) { out[row_index(cur, j)] = v; });
        refill();  // also orders the next item's bs writes after both warps' reads
        if (++st == kStages) {
            st = 0;
            par ^= 1u;
        }
        cur = nxt;
#pragma unroll
        for (int t = 0; t < RB; ++t) b[t] = bn[t];
    }
    grid_sum_last_block(dsum, partials, ticket, dot_out);
}

// ---- prolongation + p update, one thread per solve slot ------------------------
struct FinalSo {
    int n_coarse;                            // coarse levels
    const std::int32_t* agg[kMaxLevels];     // solve slot -> level-(l+1) node
    const double* y[kMaxLevels];
    double* clear[kMaxLevels];               // RED targets of k_update_so (levels >= 2)
    std::int64_t clear_n[kMaxLevels];
    int n_clear;
    double* p4;                              // optional copy of p padded to 4 doubles per slot
};

template <int kFinal, int kPer>
__global__ void __launch_bounds__(512) k_final_so(std::int32_t n, FinalSo fa, const double* __restrict__ z,
                                                 double* __restrict__ p, double* __restrict__ ap, PcgArgs a) {
    double beta = 0;
    pdl_wait();
    if (a.flags[F_DONE]) return;
    pdl_launch();
    const double rz = a.scal[S_RZ];  // r.z = sum over all levels of b_l.y_l (k_precond_so)
    if (kFinal == F_PCG_INIT) {
        if (blockIdx.x == 0 && threadIdx.x == 0) {  // pcg.hpp:52-57
            a.scal[S_RHO0] = rz;
            a.scal[S_RHO_INIT] = rz;
            a.scal[S_STOP] = a.scal[S_STOP] * rz;  // S_STOP preloaded with tol^2
            if (!(rz > 0)) {
                a.flags[F_DONE] = 1;
                a.flags[F_ITERS] = 0;
                a.scal[S_REL] = 0;
            }
        }
        if (!(rz > 0)) return;
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
    }
    // two slots (6 doubles, three 128-bit accesses per vector) per thread
    const std::int64_t nthreads = static_cast<std::int64_t>(gridDim.x) * blockDim.x;
    const std::int64_t tid = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x;
    (void)kPer;
    for (std::int64_t pr = tid; 2 * pr < n; pr += nthreads) {
        const std::int64_t sl0 = 2 * pr;
        const bool two = sl0 + 1 < n;
        std::int32_t nd[kMaxLevels][2];
#pragma unroll
        for (int l = 0; l < kMaxLevels; ++l)
            if (l < fa.n_coarse) {
                if (two) {
                    const int2 v = *reinterpret_cast<const int2*>(fa.agg[l] + sl0);
                    nd[l][0] = v.x;
                    nd[l][1] = v.y;
                } else {
                    nd[l][0] = fa.agg[l][sl0];
                    nd[l][1] = nd[l][0];
                }
            }
        double zz[6], pp[6];
        if (two) {
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                const double2 zv = reinterpret_cast<const double2*>(z)[3 * pr + q];
                zz[2 * q] = zv.x;
                zz[2 * q + 1] = zv.y;
                if (kFinal != F_PCG_INIT) {
                    const double2 pv = reinterpret_cast<const double2*>(p)[3 * pr + q];
                    pp[2 * q] = pv.x;
                    pp[2 * q + 1] = pv.y;
                } else {
                    pp[2 * q] = pp[2 * q + 1] = 0.0;
                }
            }
        } else {
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                zz[q] = z[3 * sl0 + q];
                pp[q] = kFinal != F_PCG_INIT ? p[3 * sl0 + q] : 0.0;
                zz[3 + q] = pp[3 + q] = 0.0;
            }
        }
#pragma unroll
        for (int l = 0; l < kMaxLevels; ++l)
            if (l < fa.n_coarse) {
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const double* yl = fa.y[l] + 3 * static_cast<std::int64_t>(nd[l][u]);
                    zz[3 * u] += yl[0];
                    zz[3 * u + 1] += yl[1];
                    zz[3 * u + 2] += yl[2];
                }
            }
        double pn[6];
#pragma unroll
        for (int q = 0; q < 6; ++q) pn[q] = zz[q] + beta * pp[q];
        if (two) {
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                reinterpret_cast<double2*>(p)[3 * pr + q] = make_double2(pn[2 * q], pn[2 * q + 1]);
                reinterpret_cast<double2*>(ap)[3 * pr + q] = make_double2(0.0, 0.0);
            }
        } else {
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                p[3 * sl0 + q] = pn[q];
                ap[3 * sl0 + q] = 0.0;
            }
        }
        if (fa.p4) {
#pragma unroll
            for (int u = 0; u < 2; ++u)
                if (u == 0 || two)
#pragma unroll
                    for (int q = 0; q < 3; ++q) fa.p4[4 * (sl0 + u) + q] = pn[3 * u + q];
        }
    }
    // clear the RED targets of the next update pass
    for (int l = 0; l < fa.n_clear; ++l)
        for (std::int64_t i = tid; i < fa.clear_n[l]; i += nthreads) fa.clear[l][i] = 0.0;
}

// Variant of k_precond_so with ONE warp per item (rows 0..31 on the lanes,
// rows 32..47 on lanes 0..15 of a second register slot): every column is
// three full 128-byte shared wavefronts instead of the pair split's partial
// ones, and b is broadcast once per item instead of once per warp. Each warp
// owns its ring of kStages slots; warps per CTA = blockDim.x / 32.
template <int kK, int kStages>
__global__ void __launch_bounds__(128) k_precond_so1(PrecondTable pt, double* __restrict__ partials,
                                                    unsigned* __restrict__ ticket, double* __restrict__ dot_out,
                                                    const int* __restrict__ flags, int slot_doubles) {
    constexpr int RB = (kK + 31) / 32;
    if (flags && flags[F_DONE]) return;
    extern __shared__ __align__(128) unsigned char smem[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nwc = blockDim.x >> 5;
    double* ring = reinterpret_cast<double*>(smem) + static_cast<std::size_t>(w) * kStages * slot_doubles;
    double* bs = reinterpret_cast<double*>(smem) + static_cast<std::size_t>(nwc) * kStages * slot_doubles +
                 static_cast<std::size_t>(w) * kK;
    std::uint64_t* bar = reinterpret_cast<std::uint64_t*>(
                             reinterpret_cast<double*>(smem) + static_cast<std::size_t>(nwc) * kStages * slot_doubles +
                             static_cast<std::size_t>(nwc) * kK) +
                         w * kStages;
    const std::int64_t gp = static_cast<std::int64_t>(blockIdx.x) * nwc + w;
    const std::int64_t np = static_cast<std::int64_t>(gridDim.x) * nwc;
    std::int32_t lv_lo[kMaxLevels], lv_n[kMaxLevels];
    int nloc = 0;
#pragma unroll
    for (int l = 0; l < kMaxLevels; ++l) {
        lv_lo[l] = lv_n[l] = 0;
        if (l < pt.n) {
            std::int32_t a, b;
            if (pt.split && pt.np == np) {
                a = pt.split[l * (np + 1) + gp];
                b = pt.split[l * (np + 1) + gp + 1];
            } else {
                const std::int64_t nl = pt.base[l + 1] - pt.base[l];
                a = static_cast<std::int32_t>(gp * nl / np);
                b = static_cast<std::int32_t>((gp + 1) * nl / np);
            }
            lv_lo[l] = pt.base[l] + a;
            lv_n[l] = b - a;
            nloc += lv_n[l];
        }
    }
    auto item = [&](int i) -> std::int32_t {
#pragma unroll
        for (int l = 0; l < kMaxLevels; ++l) {
            if (i < lv_n[l]) return lv_lo[l] + i;
            i -= lv_n[l];
        }
        return 0;
    };
    auto level_of = [&](std::int32_t q) {
        int l = 0;
        while (l + 1 < pt.n && q >= pt.base[l + 1]) ++l;
        return l;
    };
    for (int i = lane; i < kStages * slot_doubles; i += 32) ring[i] = 0.0;  // finite slot tails
    fence_proxy_async();
    __syncwarp();
    auto issue = [&](std::int32_t q, int st) {  // lane 0
        const int l = level_of(q);
        const std::int32_t s = q - pt.base[l];
        const std::int64_t o = pt.inv_off[l][s];
        const std::uint32_t bytes = static_cast<std::uint32_t>((pt.inv_off[l][s + 1] - o) * 8);
        mbar_arrive_expect_tx(&bar[st], bytes);
        if (l == 0)
            bulk_g2s_evict_first(ring + static_cast<std::size_t>(st) * slot_doubles, pt.inv[0] + o, bytes, &bar[st]);
        else
            bulk_g2s_evict_last(ring + static_cast<std::size_t>(st) * slot_doubles, pt.inv[l] + o, bytes, &bar[st]);
    };
    if (lane == 0) {
        for (int st = 0; st < kStages; ++st) mbar_init(&bar[st], 1);
        fence_mbar_init();
        for (int st = 0; st < kStages && st < nloc; ++st) issue(item(st), st);
    }
    __syncwarp();
    struct Item {
        int l;
        std::int32_t s0, dim;
    };
    auto row_index = [&](const Item& it, int j) -> std::int64_t {
        if (it.l == 0) return 3 * static_cast<std::int64_t>(it.s0) + j;
        return 3 * static_cast<std::int64_t>(pt.sub_nodes[it.l][it.s0 + j / 3]) + (j % 3);
    };
    auto load_b = [&](std::int32_t q, Item& it, double* bb) {
        it.l = level_of(q);
        const std::int32_t s = q - pt.base[it.l];
        it.s0 = pt.sub_ptr[it.l][s];
        it.dim = 3 * (pt.sub_ptr[it.l][s + 1] - it.s0);
#pragma unroll
        for (int t = 0; t < RB; ++t) {
            const int j = lane + 32 * t;
            bb[t] = j < it.dim ? ldg_issue(pt.rin[it.l] + row_index(it, j)) : 0.0;
        }
    };
    Item cur{0, 0, 0};
    double b[RB];
    if (nloc > 0) load_b(item(0), cur, b);
    double dsum = 0;
    int st = 0;
    std::uint32_t par = 0;
    for (int i = 0; i < nloc; ++i) {
#pragma unroll
        for (int t = 0; t < RB; ++t)
            if (lane + 32 * t < kK) bs[lane + 32 * t] = b[t];
        Item nxt{0, 0, 0};
        double bn[RB];
        if (i + 1 < nloc) load_b(item(i + 1), nxt, bn);
        __syncwarp();
        mbar_wait(&bar[st], par);
        const double* M = ring + static_cast<std::size_t>(st) * slot_doubles;
        constexpr int R = (kK + 31) / 32;
        double y[R];
        const int kc = pick_cols<kK>(cur.dim);
        double* out = pt.out[cur.l];
        auto emit = [&](auto kc_tag) {
            constexpr int K2 = decltype(kc_tag)::value;
            constexpr int R2 = (K2 + 31) / 32;
            double yy[R2];
            packed_matvec_rows<K2, 0, K2>(M, bs, yy, lane);
#pragma unroll
            for (int t = 0; t < R2; ++t) {
                const int j = matvec_row<K2, 0>(lane, t);
                if (j < cur.dim) {
                    out[row_index(cur, j)] = yy[t];
                    dsum += bs[j] * yy[t];
                }
            }
        };
        (void)y;
        if (kK >= 48 && kc == 12)
            emit(std::integral_constant<int, 12>{});
        else if (kK >= 48 && kc == 24)
            emit(std::integral_constant<int, 24>{});
        else
            emit(std::integral_constant<int, kK>{});
        __syncwarp();
        if (lane == 0 && i + kStages < nloc) {
            fence_proxy_async();
            issue(item(i + kStages), st);
        }
        if (++st == kStages) {
            st = 0;
            par ^= 1u;
        }
        cur = nxt;
#pragma unroll
        for (int t = 0; t < RB; ++t) b[t] = bn[t];
    }
    grid_sum_last_block(dsum, partials, ticket, dot_out);
}

// Variant with TWO items per warp, one per half-warp (lane i of the half
// holds rows i + 16 t): every column's shared load is a full 256-byte access
// serving both items, and the transposed reads of each 16-aligned run of rows
// hit 16 distinct banks (~4x fewer shared wavefronts per item than the pair
// split). Each warp streams its items two at a time through a ring of kStages
// double slots.
template <int kK, int kStages>
__global__ void __launch_bounds__(128) k_precond_so2(PrecondTable pt, double* __restrict__ partials,
                                                    unsigned* __restrict__ ticket, double* __restrict__ dot_out,
                                                    const int* __restrict__ flags, int slot_doubles) {
    constexpr int T = (kK + 15) / 16;
    constexpr int kBs = kK + 2;  // per-half b copy (padded: the halves' broadcasts hit different banks)
    if (flags && flags[F_DONE]) return;
    extern __shared__ __align__(128) unsigned char smem[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nwc = blockDim.x >> 5;
    const int half = lane >> 4, hl = lane & 15;
    double* ring = reinterpret_cast<double*>(smem) + static_cast<std::size_t>(w) * kStages * 2 * slot_doubles;
    double* bsw = reinterpret_cast<double*>(smem) + static_cast<std::size_t>(nwc) * kStages * 2 * slot_doubles +
                  static_cast<std::size_t>(w) * 2 * kBs;
    double* bs = bsw + half * kBs;
    std::uint64_t* bar = reinterpret_cast<std::uint64_t*>(
                             reinterpret_cast<double*>(smem) + static_cast<std::size_t>(nwc) * kStages * 2 * slot_doubles +
                             static_cast<std::size_t>(nwc) * 2 * kBs) +
                         w * kStages;
    const std::int64_t gp = static_cast<std::int64_t>(blockIdx.x) * nwc + w;
    const std::int64_t np = static_cast<std::int64_t>(gridDim.x) * nwc;
    std::int32_t lv_lo[kMaxLevels], lv_n[kMaxLevels];
    int nloc = 0;
#pragma unroll
    for (int l = 0; l < kMaxLevels; ++l) {
        lv_lo[l] = lv_n[l] = 0;
        if (l < pt.n) {
            std::int32_t a, b;
            if (pt.split && pt.np == np) {
                a = pt.split[l * (np + 1) + gp];
                b = pt.split[l * (np + 1) + gp + 1];
            } else {
                const std::int64_t nl = pt.base[l + 1] - pt.base[l];
                a = static_cast<std::int32_t>(gp * nl / np);
                b = static_cast<std::int32_t>((gp + 1) * nl / np);
            }
            lv_lo[l] = pt.base[l] + a;
            lv_n[l] = b - a;
            nloc += lv_n[l];
        }
    }
    auto item = [&](int i) -> std::int32_t {
#pragma unroll
        for (int l = 0; l < kMaxLevels; ++l) {
            if (i < lv_n[l]) return lv_lo[l] + i;
            i -= lv_n[l];
        }
        return 0;
    };
    auto level_of = [&](std::int32_t q) {
        int l = 0;
        while (l + 1 < pt.n && q >= pt.base[l + 1]) ++l;
        return l;
    };
    const int nsteps = (nloc + 1) / 2;
    for (int i = lane; i < kStages * 2 * slot_doubles; i += 32) ring[i] = 0.0;  // finite slot tails
    for (int i = lane; i < 2 * kBs; i += 32) bsw[i] = 0.0;
    fence_proxy_async();
    __syncwarp();
    auto issue = [&](int step, int st) {  // lane 0: both items of a step on one barrier
        std::uint32_t total = 0;
        std::int64_t off[2];
        std::uint32_t bytes[2] = {0, 0};
        int lv[2] = {0, 0};
        for (int h = 0; h < 2; ++h) {
            const int i = 2 * step + h;
            if (i >= nloc) continue;
            const std::int32_t q = item(i);
            lv[h] = level_of(q);
            const std::int32_t s = q - pt.base[lv[h]];
            off[h] = pt.inv_off[lv[h]][s];
            bytes[h] = static_cast<std::uint32_t>((pt.inv_off[lv[h]][s + 1] - off[h]) * 8);
            total += bytes[h];
        }
        mbar_arrive_expect_tx(&bar[st], total);
        for (int h = 0; h < 2; ++h) {
            if (!bytes[h]) continue;
            double* dst = ring + (static_cast<std::size_t>(st) * 2 + h) * slot_doubles;
            if (lv[h] == 0)
                bulk_g2s_evict_first(dst, pt.inv[0] + off[h], bytes[h], &bar[st]);
            else
                bulk_g2s_evict_last(dst, pt.inv[lv[h]] + off[h], bytes[h], &bar[st]);
        }
    };
    if (lane == 0) {
        for (int st = 0; st < kStages; ++st) mbar_init(&bar[st], 1);
        fence_mbar_init();
        for (int st = 0; st < kStages && st < nsteps; ++st) issue(st, st);
    }
    __syncwarp();
    struct Item {
        int l;
        std::int32_t s0, dim;
    };
    auto row_index = [&](const Item& it, int j) -> std::int64_t {
        if (it.l == 0) return 3 * static_cast<std::int64_t>(it.s0) + j;
        return 3 * static_cast<std::int64_t>(pt.sub_nodes[it.l][it.s0 + j / 3]) + (j % 3);
    };
    // this half's item of a step (dim 0 when the step has a single item)
    auto load_b = [&](int step, Item& it, double* bb) {
        const int i = 2 * step + half;
        it.l = 0;
        it.s0 = 0;
        it.dim = 0;
        if (i < nloc) {
            const std::int32_t q = item(i);
            it.l = level_of(q);
            const std::int32_t s = q - pt.base[it.l];
            it.s0 = pt.sub_ptr[it.l][s];
            it.dim = 3 * (pt.sub_ptr[it.l][s + 1] - it.s0);
        }
#pragma unroll
        for (int t = 0; t < T; ++t) {
            const int j = hl + 16 * t;
            bb[t] = j < it.dim ? ldg_issue(pt.rin[it.l] + row_index(it, j)) : 0.0;
        }
    };
    Item cur{0, 0, 0};
    double b[T];
    if (nsteps > 0) load_b(0, cur, b);
    double dsum = 0;
    int st = 0;
    std::uint32_t par = 0;
    for (int step = 0; step < nsteps; ++step) {
#pragma unroll
        for (int t = 0; t < T; ++t) bs[hl + 16 * t] = b[t];
        Item nxt{0, 0, 0};
        double bn[T];
        if (step + 1 < nsteps) load_b(step + 1, nxt, bn);
        __syncwarp();
        mbar_wait(&bar[st], par);
        const double* M = ring + (static_cast<std::size_t>(st) * 2 + half) * slot_doubles;
        const int dmax = max(cur.dim, __shfl_xor_sync(0xffffffffu, cur.dim, 16));
        const int kc = pick_cols<kK>(dmax);
        double* out = pt.out[cur.l];
        auto emit = [&](auto kc_tag) {
            constexpr int K2 = decltype(kc_tag)::value;
            constexpr int T2 = (K2 + 15) / 16;
            double yy[T2];
            packed_matvec_half<K2>(M, bs, yy, hl);
#pragma unroll
            for (int t = 0; t < T2; ++t) {
                const int j = hl + 16 * t;
                if (j < cur.dim) {
                    out[row_index(cur, j)] = yy[t];
                    dsum += bs[j] * yy[t];
                }
            }
        };
        if (kK >= 48 && kc == 12)
            emit(std::integral_constant<int, 12>{});
        else if (kK >= 48 && kc == 24)
            emit(std::integral_constant<int, 24>{});
        else
            emit(std::integral_constant<int, kK>{});
        __syncwarp();
        if (lane == 0 && step + kStages < nsteps) {
            fence_proxy_async();
            issue(step + kStages, st);
        }
        if (++st == kStages) {
            st = 0;
            par ^= 1u;
        }
        cur = nxt;
#pragma unroll
        for (int t = 0; t < T; ++t) b[t] = bn[t];
    }
    grid_sum_last_block(dsum, partials, ticket, dot_out);
}

// ============================================================================
// Warp-specialised preconditioner (k_precond_ws): one CTA per SM, one producer
// warp streaming the CTA's packed inverses in order through a CTA-wide ring of
// kSlots shared slots (cp.async.bulk; full/empty mbarriers per slot), and
// kCons consumer warps, each solving two items at a time (one per half-warp,
// packed_matvec_half: full 256-byte shared loads, conflict-free transposed
// reads). Staging depth (slots in flight) and compute concurrency are sized
// independently, so neither the TMA latency nor the mat-vec latency is
// exposed per item as in the per-pair rings.
__device__ __forceinline__ void mbar_arrive(std::uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

template <int kK, int kSlots, int kCons>
__global__ void __launch_bounds__(32 * (kCons + 1)) k_precond_ws(PrecondTable pt, double* __restrict__ partials,
                                                                unsigned* __restrict__ ticket,
                                                                double* __restrict__ dot_out,
                                                                const int* __restrict__ flags, int slot_doubles) {
    constexpr int T = (kK + 15) / 16;
    constexpr int kBs = kK + 2;
    if (flags && flags[F_DONE]) return;
    extern __shared__ __align__(128) unsigned char smem[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    double* ring = reinterpret_cast<double*>(smem);
    double* bsw = ring + static_cast<std::size_t>(kSlots) * slot_doubles;  // kCons x 2 x kBs
    std::uint64_t* full = reinterpret_cast<std::uint64_t*>(bsw + static_cast<std::size_t>(kCons) * 2 * kBs);
    std::uint64_t* empty = full + kSlots;
    // this CTA's items: an even share of each level, level 0 first
    const std::int64_t gp = blockIdx.x, np = gridDim.x;
    std::int32_t lv_lo[kMaxLevels], lv_n[kMaxLevels];
    int nloc = 0;
#pragma unroll
    for (int l = 0; l < kMaxLevels; ++l) {
        lv_lo[l] = lv_n[l] = 0;
        if (l < pt.n) {
            const std::int64_t nl = pt.base[l + 1] - pt.base[l];
            const std::int32_t a = static_cast<std::int32_t>(gp * nl / np);
            const std::int32_t b = static_cast<std::int32_t>((gp + 1) * nl / np);
            lv_lo[l] = pt.base[l] + a;
            lv_n[l] = b - a;
            nloc += lv_n[l];
        }
    }
    auto item = [&](int i) -> std::int32_t {
#pragma unroll
        for (int l = 0; l < kMaxLevels; ++l) {
            if (i < lv_n[l]) return lv_lo[l] + i;
            i -= lv_n[l];
        }
        return 0;
    };
    auto level_of = [&](std::int32_t q) {
        int l = 0;
        while (l + 1 < pt.n && q >= pt.base[l + 1]) ++l;
        return l;
    };
    // finite slot tails (the unrolled mat-vec multiplies them by b_k = 0)
    for (int i = threadIdx.x; i < kSlots * slot_doubles; i += blockDim.x) ring[i] = 0.0;
    for (int i = threadIdx.x; i < kCons * 2 * kBs; i += blockDim.x) bsw[i] = 0.0;
    fence_proxy_async();
    if (threadIdx.x == 0) {
        for (int sl = 0; sl < kSlots; ++sl) {
            mbar_init(&full[sl], 1);
            mbar_init(&empty[sl], 1);
        }
        fence_mbar_init();
    }
    __syncthreads();
    double dsum = 0;
    if (w == kCons) {  // ---- producer warp ----
        if (lane == 0) {
            for (int i = 0; i < nloc; ++i) {
                const int sl = i % kSlots;
                const std::uint32_t ph = static_cast<std::uint32_t>(i / kSlots) & 1u;
                if (i >= kSlots) mbar_wait(&empty[sl], ph ^ 1u);  // consumed item i - kSlots
                const std::int32_t q = item(i);
                const int l = level_of(q);
                const std::int32_t s = q - pt.base[l];
                const std::int64_t o = pt.inv_off[l][s];
                const std::uint32_t bytes = static_cast<std::uint32_t>((pt.inv_off[l][s + 1] - o) * 8);
                mbar_arrive_expect_tx(&full[sl], bytes);
                double* dst = ring + static_cast<std::size_t>(sl) * slot_doubles;
                if (l == 0)
                    bulk_g2s_evict_first(dst, pt.inv[0] + o, bytes, &full[sl]);
                else
                    bulk_g2s_evict_last(dst, pt.inv[l] + o, bytes, &full[sl]);
            }
        }
    } else {  // ---- consumer warps: items (2p, 2p+1) for p = w, w + kCons, ... ----
        const int half = lane >> 4, hl = lane & 15;
        double* bs = bsw + (static_cast<std::size_t>(w) * 2 + half) * kBs;
        struct Item {
            int l;
            std::int32_t s0, dim;
        };
        auto row_index = [&](const Item& it, int j) -> std::int64_t {
            if (it.l == 0) return 3 * static_cast<std::int64_t>(it.s0) + j;
            return 3 * static_cast<std::int64_t>(pt.sub_nodes[it.l][it.s0 + j / 3]) + (j % 3);
        };
        auto load_b = [&](int i, Item& it, double* bb) {
            it.l = 0;
            it.s0 = 0;
            it.dim = 0;
            if (i < nloc) {
                const std::int32_t q = item(i);
                it.l = level_of(q);
                const std::int32_t s = q - pt.base[it.l];
                it.s0 = pt.sub_ptr[it.l][s];
                it.dim = 3 * (pt.sub_ptr[it.l][s + 1] - it.s0);
            }
#pragma unroll
            for (int t = 0; t < T; ++t) {
                const int j = hl + 16 * t;
                bb[t] = j < it.dim ? ldg_issue(pt.rin[it.l] + row_index(it, j)) : 0.0;
            }
        };
        const int npairs = (nloc + 1) / 2;
        Item cur{0, 0, 0};
        double b[T];
        if (w < npairs) load_b(2 * w + half, cur, b);
        for (int pi = w; pi < npairs; pi += kCons) {
            const int i = 2 * pi + half;  // this half's item
#pragma unroll
            for (int t = 0; t < T; ++t) bs[hl + 16 * t] = b[t];
            Item nxt{0, 0, 0};
            double bn[T];
            if (pi + kCons < npairs) load_b(2 * (pi + kCons) + half, nxt, bn);
            __syncwarp();
            const bool have = i < nloc;
            const int sl = i % kSlots;
            if (have) mbar_wait(&full[sl], static_cast<std::uint32_t>(i / kSlots) & 1u);
            __syncwarp();
            const double* M = ring + static_cast<std::size_t>(have ? sl : (i - 1) % kSlots) * slot_doubles;
            const int dmax = max(cur.dim, __shfl_xor_sync(0xffffffffu, cur.dim, 16));
            const int kc = pick_cols<kK>(dmax);
            double* out = pt.out[cur.l];
            auto emit = [&](auto kc_tag) {
                constexpr int K2 = decltype(kc_tag)::value;
                constexpr int T2 = (K2 + 15) / 16;
                double yy[T2];
                packed_matvec_half<K2>(M, bs, yy, hl);
#pragma unroll
                for (int t = 0; t < T2; ++t) {
                    const int j = hl + 16 * t;
                    if (j < cur.dim) {
                        out[row_index(cur, j)] = yy[t];
                        dsum += bs[j] * yy[t];
                    }
                }
            };
            if (kK >= 48 && kc == 12)
                emit(std::integral_constant<int, 12>{});
            else if (kK >= 48 && kc == 24)
                emit(std::integral_constant<int, 24>{});
            else
                emit(std::integral_constant<int, kK>{});
            __syncwarp();
            if (have && hl == 0) mbar_arrive(&empty[sl]);  // this half is done with its slot
            cur = nxt;
#pragma unroll
            for (int t = 0; t < T; ++t) b[t] = bn[t];
        }
    }
    grid_sum_last_block(dsum, partials, ticket, dot_out);
}

// ============================================================================
// One PCG iteration after the SpMV as ONE cooperative kernel (k_iter_so):
//   items   level-0 subdomains first: warp 0 of the pair applies the vector
//           update to the subdomain's slots (x += alpha p, r -= alpha Ap, or
//           r = b - A x on restart iterations, pcg.hpp:67-74) and hands the
//           new residual to both warps through shared memory as b; warp 1
//           restricts it to the subdomain's level-1 nodes (and REDs the sums
//           to their coarser ancestors); both solve the packed inverse.
//           Then the coarse items, once every pair has finished its level-0
//           items (a global arrival counter: the coarse restricted residuals
//           are complete).
//   final   once every CTA has published its share of r.z (second counter),
//           every CTA sums the shares in the same order, applies the stop test
//           and beta, and prolongs + updates p for its slice of the slots.
// Two kernels per iteration (SpMV, this) instead of four; r is read once.
// The counters are monotone (target = iteration index x participants, the
// iteration index advanced by the SpMV), so nothing needs re-arming.
struct IterArgs {
    PrecondTable pt;
    FinalSo fa;
    // update (solve order)
    double* x;
    double* r;
    const double* p;
    const double* ap;   // A p, or A x_new on restart iterations
    const double* b;
    double* z;
    double* pout;       // p (updated in place by the final phase)
    double* apclear;    // A p buffer, cleared for the next SpMV
    double* tmpclear;   // A x buffer of the next restart iteration (or null)
    // restriction metadata (level 0 -> 1 and ancestors)
    const std::int32_t* up_first0;
    const std::int32_t* upc_ptr0;
    const std::int32_t* upc_node0;
    double* rr1;
    double* rr[kMaxLevels];
    const std::int32_t* anc[kMaxLevels];
    int n_levels;
    std::int32_t n_slots;
    double* scal;
    int* flags;
    unsigned* counters;  // [0] level-0 pairs done, [1] CTAs done
    double* partials;    // per-CTA r.z shares
    int restart_mode;    // 1: r = b - A x (restart iteration)
};

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void spin_until(const unsigned* p, unsigned target, int* err) {
    long long n = 0;
    while (static_cast<int>(ld_acquire(p) - target) < 0) {
        __nanosleep(64);
        if (++n > (1ll << 26)) {  // ~seconds: never expected; fail loudly instead of hanging
            atomicExch(err, 1);
            break;
        }
    }
}

template <int kK, int kStages>
__global__ void __launch_bounds__(256) k_iter_so(IterArgs ia, int slot_doubles) {
    constexpr int RB = (kK + 31) / 32;
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ double red[32];
    int* flags = ia.flags;
    if (flags[F_DONE]) return;
    const int k_it = flags[F_K];
    double alpha = 0;
    {
        PcgArgs pa{};
        pa.scal = ia.scal;
        pa.flags = flags;
        if (!pcg_alpha(pa, alpha)) return;  // every CTA sees the same p.Ap
    }
    const PrecondTable& pt = ia.pt;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, pair = w >> 1, half = w & 1;
    const int npc = blockDim.x >> 6;
    double* ring = reinterpret_cast<double*>(smem) + static_cast<std::size_t>(pair) * kStages * slot_doubles;
    double* bs = reinterpret_cast<double*>(smem) + static_cast<std::size_t>(npc) * kStages * slot_doubles +
                 static_cast<std::size_t>(pair) * kK;  // one b per pair (written by warp 0)
    int* meta = reinterpret_cast<int*>(reinterpret_cast<double*>(smem) +
                                       static_cast<std::size_t>(npc) * kStages * slot_doubles +
                                       static_cast<std::size_t>(npc) * kK) +
                pair * 80;  // [0..32] level-1 CSR offsets, [40..71] children
    std::uint64_t* bar = reinterpret_cast<std::uint64_t*>(reinterpret_cast<double*>(smem) +
                                                          static_cast<std::size_t>(npc) * kStages * slot_doubles +
                                                          static_cast<std::size_t>(npc) * kK + npc * 40) +
                         pair * kStages;
    const std::int64_t gp = static_cast<std::int64_t>(blockIdx.x) * npc + pair;
    const std::int64_t np = static_cast<std::int64_t>(gridDim.x) * npc;
    std::int32_t lv_lo[kMaxLevels], lv_n[kMaxLevels];
    int nloc = 0;
#pragma unroll
    for (int l = 0; l < kMaxLevels; ++l) {
        lv_lo[l] = lv_n[l] = 0;
        if (l < pt.n) {
            std::int32_t a, b;
            if (pt.split && pt.np == np) {
                a = pt.split[l * (np + 1) + gp];
                b = pt.split[l * (np + 1) + gp + 1];
            } else {
                const std::int64_t nl = pt.base[l + 1] - pt.base[l];
                a = static_cast<std::int32_t>(gp * nl / np);
                b = static_cast<std::int32_t>((gp + 1) * nl / np);
            }
            lv_lo[l] = pt.base[l] + a;
            lv_n[l] = b - a;
            nloc += lv_n[l];
        }
    }
    const int n0 = lv_n[0];  // this pair's level-0 items come first
    auto item = [&](int i) -> std::int32_t {
#pragma unroll
        for (int l = 0; l < kMaxLevels; ++l) {
            if (i < lv_n[l]) return lv_lo[l] + i;
            i -= lv_n[l];
        }
        return 0;
    };
    auto level_of = [&](std::int32_t q) {
        int l = 0;
        while (l + 1 < pt.n && q >= pt.base[l + 1]) ++l;
        return l;
    };
    for (int i = half * 32 + lane; i < kStages * slot_doubles; i += 64) ring[i] = 0.0;  // finite slot tails
    fence_proxy_async();
    pair_sync(pair);
    auto issue = [&](std::int32_t q, int st) {
        const int l = level_of(q);
        const std::int32_t s = q - pt.base[l];
        const std::int64_t o = pt.inv_off[l][s];
        const std::uint32_t bytes = static_cast<std::uint32_t>((pt.inv_off[l][s + 1] - o) * 8);
        mbar_arrive_expect_tx(&bar[st], bytes);
        if (l == 0)
            bulk_g2s_evict_first(ring + static_cast<std::size_t>(st) * slot_doubles, pt.inv[0] + o, bytes, &bar[st]);
        else
            bulk_g2s_evict_last(ring + static_cast<std::size_t>(st) * slot_doubles, pt.inv[l] + o, bytes, &bar[st]);
    };
    if (half == 0 && lane == 0) {
        for (int st = 0; st < kStages; ++st) mbar_init(&bar[st], 1);
        fence_mbar_init();
        for (int st = 0; st < kStages && st < nloc; ++st) issue(item(st), st);
    }
    pair_sync(pair);
    struct Item {
        int l;
        std::int32_t s, s0, dim;
    };
    auto row_index = [&](const Item& it, int j) -> std::int64_t {
        if (it.l == 0) return 3 * static_cast<std::int64_t>(it.s0) + j;
        return 3 * static_cast<std::int64_t>(pt.sub_nodes[it.l][it.s0 + j / 3]) + (j % 3);
    };
    // Per item, prefetched one item ahead into registers:
    //   level 0, warp 0: the update operands -> new residual in b (x, r written)
    //   level 0, warp 1: level-1 node range, CSR offsets and children
    //   coarse: both warps gather b from the restricted residual
    std::int32_t v0 = 0, nv = 0, my_uptr = 0, my_child = 0;
    auto load = [&](int i, Item& it, double* bb, std::int32_t& av0, std::int32_t& anv, std::int32_t& aup,
                    std::int32_t& ach) {
        const std::int32_t q = item(i);
        it.l = level_of(q);
        it.s = q - pt.base[it.l];
        it.s0 = pt.sub_ptr[it.l][it.s];
        it.dim = 3 * (pt.sub_ptr[it.l][it.s + 1] - it.s0);
        if (it.l == 0) {
            if (half == 0) {
                double pv[RB], av[RB], xv[RB], rv[RB];
#pragma unroll
                for (int t = 0; t < RB; ++t) {
                    const int j = lane + 32 * t;
                    if (j < it.dim) {
                        const std::int64_t g = 3 * static_cast<std::int64_t>(it.s0) + j;
                        av[t] = ldg_issue(ia.ap + g);
                        if (ia.restart_mode) {
                            rv[t] = ldg_issue(ia.b + g);
                        } else {
                            rv[t] = ldg_issue(ia.r + g);
                            pv[t] = ldg_issue(ia.p + g);
                            xv[t] = ldg_issue(ia.x + g);
                        }
                    }
                }
#pragma unroll
                for (int t = 0; t < RB; ++t) {
                    const int j = lane + 32 * t;
                    bb[t] = 0.0;
                    if (j < it.dim) {
                        const std::int64_t g = 3 * static_cast<std::int64_t>(it.s0) + j;
                        double nr;
                        if (ia.restart_mode) {
                            nr = rv[t] - av[t];
                        } else {
                            ia.x[g] = xv[t] + alpha * pv[t];
                            nr = rv[t] - alpha * av[t];
                        }
                        ia.r[g] = nr;
                        bb[t] = nr;
                    }
                }
            } else {
                av0 = ia.up_first0[it.s];
                anv = ia.up_first0[it.s + 1] - av0;
                aup = lane < anv ? ia.upc_ptr0[av0 + lane] - it.s0 : 0;
                ach = lane < it.dim / 3 ? ia.upc_node0[it.s0 + lane] - it.s0 : 0;
            }
        } else {
#pragma unroll
            for (int t = 0; t < RB; ++t) {
                const int j = lane + 32 * t;
                bb[t] = j < it.dim ? ldg_issue(pt.rin[it.l] + row_index(it, j)) : 0.0;
            }
        }
    };
    Item cur{0, 0, 0, 0};
    double b[RB];
    if (nloc > 0 && n0 > 0) load(0, cur, b, v0, nv, my_uptr, my_child);
    double dsum = 0;
    int st = 0;
    std::uint32_t par = 0;
    for (int i = 0; i < nloc; ++i) {
        if (i == n0) {
            // every pair's level-0 items (and restrictions) must be complete
            // before the coarse residuals are read
            __threadfence();
            pair_sync(pair);
            if (half == 0 && lane == 0) {
                atomicAdd(ia.counters + 0, 1u);
                spin_until(ia.counters + 0, static_cast<unsigned>(k_it) * static_cast<unsigned>(np), flags + F_ERR);
            }
            pair_sync(pair);
            load(i, cur, b, v0, nv, my_uptr, my_child);
        }
        // b into shared memory: warp 0 for level-0 items (it holds the updated
        // residual), both warps otherwise (same values)
        if (cur.l > 0 || half == 0) {
#pragma unroll
            for (int t = 0; t < RB; ++t)
                if (lane + 32 * t < kK) bs[lane + 32 * t] = b[t];
        }
        if (cur.l == 0 && half == 1) {
            if (lane < nv) meta[lane] = my_uptr;
            if (lane < cur.dim / 3) meta[40 + lane] = my_child;
            if (lane == 0) meta[nv] = cur.dim / 3;  // end of the last node's children
        }
        Item nxt{0, 0, 0, 0};
        double bn[RB];
        std::int32_t nv0 = 0, nnv = 0, nup = 0, nch = 0;
        if (i + 1 < nloc && i + 1 != n0) load(i + 1, nxt, bn, nv0, nnv, nup, nch);
        pair_sync(pair);  // bs (and meta) ready for both warps
        if (cur.l == 0 && half == 1) {  // level-1 restriction of this subdomain (children ascending)
            for (int t = lane; t < 3 * nv; t += 32) {
                const int vi = t / 3, comp = t % 3;
                double acc = 0;
                for (int q = meta[vi]; q < meta[vi + 1]; ++q) acc += bs[3 * meta[40 + q] + comp];
                const std::int32_t v = v0 + vi;
                ia.rr1[3 * static_cast<std::int64_t>(v) + comp] = acc;
#pragma unroll
                for (int l = 2; l < kMaxLevels; ++l)
                    if (l < ia.n_levels) red_add(ia.rr[l] + 3 * static_cast<std::int64_t>(ia.anc[l][v]) + comp, acc);
            }
        }
        mbar_wait(&bar[st], par);
        const double* M = ring + static_cast<std::size_t>(st) * slot_doubles;
        double* out = pt.out[cur.l];
        dsum += pair_solve<kK>(M, bs, lane, half, cur.dim,
                               [&](int j, double v) { out[row_index(cur, j)] = v; });
        pair_sync(pair);  // both warps are done with the slot, bs and meta
        if (half == 0 && lane == 0 && i + kStages < nloc) {
            fence_proxy_async();
            issue(item(i + kStages), st);
        }
        if (++st == kStages) {
            st = 0;
            par ^= 1u;
        }
        cur = nxt;
        v0 = nv0;
        nv = nnv;
        my_uptr = nup;
        my_child = nch;
#pragma unroll
        for (int t = 0; t < RB; ++t) b[t] = bn[t];
    }
    if (n0 == nloc) {  // a pair without coarse items still arrives
        __threadfence();
        pair_sync(pair);
        if (half == 0 && lane == 0) atomicAdd(ia.counters + 0, 1u);
    }
    // ---- final: r.z from every CTA, stop test, beta, prolongation + p ----
    const double bsum = block_sum(dsum, red);
    if (threadIdx.x == 0) {
        ia.partials[blockIdx.x] = bsum;
        __threadfence();
        atomicAdd(ia.counters + 1, 1u);
        spin_until(ia.counters + 1, static_cast<unsigned>(k_it) * gridDim.x, flags + F_ERR);
    }
    __syncthreads();
    if (threadIdx.x < 32) {
        double v = 0;
        for (unsigned q = threadIdx.x; q < gridDim.x; q += 32) v += __ldcg(ia.partials + q);
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (threadIdx.x == 0) red[0] = v;
    }
    __syncthreads();
    const double rz = red[0];
    const double rho = ia.scal[S_RHO0 + ((k_it - 1) & 1)];
    const double stop = ia.scal[S_STOP];
    if (blockIdx.x == 0 && threadIdx.x == 0) {  // pcg.hpp:76-82
        flags[F_ITERS] = k_it;
        ia.scal[S_REL] = sqrt(fabs(rz) / ia.scal[S_RHO_INIT]);
        if (rz <= stop) {
            flags[F_DONE] = 1;
            flags[F_CONVERGED] = 1;
        } else {
            ia.scal[S_RHO0 + (k_it & 1)] = rz;
        }
    }
    if (rz <= stop) return;
    const double beta = rz / rho;
    const FinalSo& fa = ia.fa;
    const std::int64_t stride = static_cast<std::int64_t>(gridDim.x) * blockDim.x;
    const std::int64_t tid = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x;
    for (std::int64_t sl = tid; sl < ia.n_slots; sl += stride) {
        const std::int64_t g = 3 * sl;
        std::int32_t nd[kMaxLevels];
#pragma unroll
        for (int l = 0; l < kMaxLevels; ++l)
            if (l < fa.n_coarse) nd[l] = fa.agg[l][sl];
        double z0 = ia.z[g], z1 = ia.z[g + 1], z2 = ia.z[g + 2];
        const double p0 = ia.pout[g], p1 = ia.pout[g + 1], p2 = ia.pout[g + 2];
#pragma unroll
        for (int l = 0; l < kMaxLevels; ++l)
            if (l < fa.n_coarse) {
                const double* yl = fa.y[l] + 3 * static_cast<std::int64_t>(nd[l]);
                z0 += yl[0];
                z1 += yl[1];
                z2 += yl[2];
            }
        ia.pout[g] = z0 + beta * p0;
        ia.pout[g + 1] = z1 + beta * p1;
        ia.pout[g + 2] = z2 + beta * p2;
        ia.apclear[g] = 0.0;
        ia.apclear[g + 1] = 0.0;
        ia.apclear[g + 2] = 0.0;
        if (ia.tmpclear) {
            ia.tmpclear[g] = 0.0;
            ia.tmpclear[g + 1] = 0.0;
            ia.tmpclear[g + 2] = 0.0;
        }
    }
    for (int l = 0; l < fa.n_clear; ++l)
        for (std::int64_t q = tid; q < fa.clear_n[l]; q += stride) fa.clear[l][q] = 0.0;
}

// ============================================================================
// The whole PCG loop as ONE persistent cooperative kernel (pcg.hpp:59-85).
// Every iteration is four phases separated by grid barriers:
//   S  SpMV Ap = A p with the p.Ap partials (TMA-staged tiles, as k_spmv_tma)
//   U  x += alpha p, r -= alpha Ap, restriction to every coarse level
//   P  every MAS level's dense solves (warp pairs, TMA ring, as k_precond_so)
//   F  prolongation, convergence test, p = z + beta p, Ap cleared
// (+ the restart iterations' x update and A x SpMV, pcg.hpp:69-74). The dots
// are per-CTA partials that every CTA sums in the same fixed order after the
// barrier, so alpha, beta and the stop decision are identical in every CTA
// and never leave the device; the kernel-boundary ramp-up/drain of the four
// kernels per iteration (and their CTA launches) are gone. Shared memory is
// one union region that each phase lays out for itself (the phases are
// separated by grid barriers and every TMA copy a phase issues is consumed
// inside it).
namespace cg = cooperative_groups;

constexpr int kPT = 256;     // threads per CTA (8 warps, 4 warp pairs)
constexpr int kPWarps = kPT / 32;
constexpr int kPPairs = kPT / 64;

struct __align__(16) SpmvStage {
    double blk[288];
    std::uint32_t rows[32];
    std::uint32_t cols[32];
};

struct Persist {
    const std::uint32_t* rows;
    const std::uint32_t* cols;
    const double* blocks;
    std::int64_t U;
    std::int32_t n;
    double* x;
    double* r;
    double* p;
    double* ap;
    double* z;
    double* tmp;
    const double* b;
    SoRestrict so;
    PrecondTable pt;
    FinalSo fa;
    double* partials;  // 2 x gridDim.x
    double* scal;
    int* flags;
    unsigned long long* phase_ns;  // optional: S, U, P, F (summed by CTA 0)
    int restart, max_iters;
    int slot_doubles;              // preconditioner ring slot (packed_doubles(kK))
    int union_bytes;               // bytes of the shared union region
};

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// grid barrier; generic shared accesses of this phase are ordered before the
// next phase's TMA writes into the same bytes
__device__ __forceinline__ void phase_sync(cg::grid_group& grid) {
    fence_proxy_async();
    grid.sync();
}

// fixed-order sum of the per-CTA partials (identical in every CTA)
__device__ __forceinline__ double sum_partials(const double* part, double* red) {
    __syncthreads();
    if (threadIdx.x < 32) {
        double v = 0;
        for (unsigned i = threadIdx.x; i < gridDim.x; i += 32) v += __ldcg(part + i);
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (threadIdx.x == 0) red[0] = v;
    }
    __syncthreads();
    const double v = red[0];
    __syncthreads();
    return v;
}

__device__ __forceinline__ void store_partial(double v, double* part, double* red) {
    const double bs = block_sum(v, red);
    if (threadIdx.x == 0) part[blockIdx.x] = bs;
}

// ---- S: y (+)= A x over the solve-order matrix, p.Ap partial (kDot) ----------
template <bool kDot, int kSS>
__device__ double spmv_phase(const Persist& P, const double* __restrict__ xin, double* __restrict__ y,
                             unsigned char* smem, std::uint64_t* sbar, std::uint32_t& cnt) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    SpmvStage* stage = reinterpret_cast<SpmvStage*>(smem) + w * kSS;
    std::uint64_t* bar = sbar + w * kSS;
    const std::int64_t warp0 = static_cast<std::int64_t>(blockIdx.x) * kPWarps + w;
    const std::int64_t nwarps = static_cast<std::int64_t>(gridDim.x) * kPWarps;
    const std::int64_t n_chunks = (P.U + 31) >> 5;
    const std::int64_t ch0 = warp0 * n_chunks / nwarps, ch1 = (warp0 + 1) * n_chunks / nwarps;
    auto issue = [&](std::int64_t ch, std::uint32_t c) {  // lane 0
        const int s = static_cast<int>(c % kSS);
        mbar_arrive_expect_tx(&bar[s], static_cast<std::uint32_t>(sizeof(SpmvStage)));
        bulk_g2s_evict_first(stage[s].blk, P.blocks + ch * 288, 288 * 8, &bar[s]);
        bulk_g2s_evict_first(stage[s].rows, P.rows + ch * 32, 128, &bar[s]);
        bulk_g2s_evict_first(stage[s].cols, P.cols + ch * 32, 128, &bar[s]);
    };
    if (lane == 0) {
        fence_proxy_async();
        for (int i = 0; i < kSS && ch0 + i < ch1; ++i) issue(ch0 + i, cnt + i);
    }
    __syncwarp();
    std::uint32_t r = 0xFFFFFFFFu, c = 0;
    double g[6];
    auto gather = [&](std::int64_t ch, std::uint32_t cc, std::uint32_t& rr, std::uint32_t& cl, double* gg) {
        const int s = static_cast<int>(cc % kSS);
        mbar_wait(&bar[s], (cc / kSS) & 1u);
        const bool valid = (ch << 5) + lane < P.U;
        rr = valid ? stage[s].rows[lane] : 0xFFFFFFFFu;
        cl = valid ? stage[s].cols[lane] : 0u;
        const std::uint32_t rx = valid ? rr : 0u;
        gg[0] = ldg_issue(xin + 3 * cl);
        gg[1] = ldg_issue(xin + 3 * cl + 1);
        gg[2] = ldg_issue(xin + 3 * cl + 2);
        gg[3] = ldg_issue(xin + 3 * rx);
        gg[4] = ldg_issue(xin + 3 * rx + 1);
        gg[5] = ldg_issue(xin + 3 * rx + 2);
    };
    if (ch0 < ch1) gather(ch0, cnt, r, c, g);
    double dsum = 0;
    for (std::int64_t ch = ch0; ch < ch1; ++ch, ++cnt) {
        const int s = static_cast<int>(cnt % kSS);
        double h[9];
#pragma unroll
        for (int k = 0; k < 9; ++k) h[k] = stage[s].blk[32 * k + lane];
        std::uint32_t rn = 0xFFFFFFFFu, cn = 0;
        double gn[6];
        if (ch + 1 < ch1) gather(ch + 1, cnt + 1, rn, cn, gn);
        __syncwarp();
        if (lane == 0 && ch + kSS < ch1) {
            fence_proxy_async();
            issue(ch + kSS, cnt + kSS);
        }
        const bool valid = r != 0xFFFFFFFFu;
        double yr0 = 0, yr1 = 0, yr2 = 0;
        if (valid) {
            yr0 = h[0] * g[0] + h[3] * g[1] + h[6] * g[2];
            yr1 = h[1] * g[0] + h[4] * g[1] + h[7] * g[2];
            yr2 = h[2] * g[0] + h[5] * g[1] + h[8] * g[2];
            if (r != c) {
                red_add(y + 3 * c, h[0] * g[3] + h[1] * g[4] + h[2] * g[5]);
                red_add(y + 3 * c + 1, h[3] * g[3] + h[4] * g[4] + h[5] * g[5]);
                red_add(y + 3 * c + 2, h[6] * g[3] + h[7] * g[4] + h[8] * g[5]);
            }
            if (kDot) dsum += (r != c ? 2.0 : 1.0) * (g[3] * yr0 + g[4] * yr1 + g[5] * yr2);
        }
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
        r = rn;
        c = cn;
#pragma unroll
        for (int k = 0; k < 6; ++k) g[k] = gn[k];
    }
    return dsum;
}

// ---- U: vector update + restriction to every coarse level --------------------
template <int kMode>
__device__ void update_phase(const Persist& P, double alpha, const double* __restrict__ apv, double* sm) {
    PcgArgs a{};
    a.x = P.x;
    a.r = P.r;
    a.p = P.p;
    a.b = P.b;
    const std::int32_t ntiles = static_cast<std::int32_t>(ceil_div(P.so.n0_parts, P.so.subs));
    for (std::int32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x)
        update_tile<kMode, kPT>(P.so, a, alpha, apv, tile, sm);
}

// ---- P: every level's dense solves, z / y_l, partial r.z ----------------------
template <int kK, int kSP>
__device__ double precond_phase(const Persist& P, unsigned char* smem, std::uint64_t* pbar, std::uint32_t& cnt) {
    constexpr int RB = (kK + 31) / 32;
    const PrecondTable& pt = P.pt;
    const int slot = P.slot_doubles;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, pair = w >> 1, half = w & 1;
    double* ring = reinterpret_cast<double*>(smem) + static_cast<std::size_t>(pair) * kSP * slot;
    double* bs = reinterpret_cast<double*>(smem) + static_cast<std::size_t>(kPPairs) * kSP * slot +
                 static_cast<std::size_t>(w) * kK;
    std::uint64_t* bar = pbar + pair * kSP;
    // every pair takes an even share of EACH level (a contiguous run per
    // level, level 0 first): the coarse items, cheap in bytes but with a
    // longer gather chain, are spread over all pairs instead of piling up at
    // the end of the work list
    const std::int64_t gp = static_cast<std::int64_t>(blockIdx.x) * kPPairs + pair;
    const std::int64_t np = static_cast<std::int64_t>(gridDim.x) * kPPairs;
    std::int32_t lv_lo[kMaxLevels], lv_n[kMaxLevels];
    int nloc = 0;
#pragma unroll
    for (int l = 0; l < kMaxLevels; ++l) {
        lv_lo[l] = lv_n[l] = 0;
        if (l < pt.n) {
            std::int32_t a, b;
            if (pt.split && pt.np == np) {
                a = pt.split[l * (np + 1) + gp];
                b = pt.split[l * (np + 1) + gp + 1];
            } else {
                const std::int64_t nl = pt.base[l + 1] - pt.base[l];
                a = static_cast<std::int32_t>(gp * nl / np);
                b = static_cast<std::int32_t>((gp + 1) * nl / np);
            }
            lv_lo[l] = pt.base[l] + a;
            lv_n[l] = b - a;
            nloc += lv_n[l];
        }
    }
    auto item = [&](int i) -> std::int32_t {
#pragma unroll
        for (int l = 0; l < kMaxLevels; ++l) {
            if (i < lv_n[l]) return lv_lo[l] + i;
            i -= lv_n[l];
        }
        return 0;
    };
    auto level_of = [&](std::int32_t q) {
        int l = 0;
        while (l + 1 < pt.n && q >= pt.base[l + 1]) ++l;
        return l;
    };
    // warp 0 of the pair: zero the slot tail past this item's inverse (the
    // unrolled mat-vec reads up to packed_doubles(kK) with b_k = 0), then
    // lane 0 issues the bulk copy
    auto issue = [&](std::int32_t q, std::uint32_t c) {
        const int st = static_cast<int>(c % kSP);
        const int l = level_of(q);
        const std::int32_t s = q - pt.base[l];
        const std::int64_t o = pt.inv_off[l][s];
        const int nd = static_cast<int>(pt.inv_off[l][s + 1] - o);
        double* dst = ring + static_cast<std::size_t>(st) * slot;
        for (int i = nd + lane; i < slot; i += 32) dst[i] = 0.0;
        __syncwarp();
        if (lane == 0) {
            fence_proxy_async();
            mbar_arrive_expect_tx(&bar[st], static_cast<std::uint32_t>(nd * 8));
            if (l == 0)
                bulk_g2s_evict_first(dst, pt.inv[0] + o, static_cast<std::uint32_t>(nd * 8), &bar[st]);
            else
                bulk_g2s_evict_last(dst, pt.inv[l] + o, static_cast<std::uint32_t>(nd * 8), &bar[st]);
        }
    };
    if (half == 0)
        for (int i = 0; i < kSP && i < nloc; ++i) issue(item(i), cnt + i);
    struct Item {
        int l;
        std::int32_t s0, dim;
    };
    auto row_index = [&](const Item& it, int j) -> std::int64_t {
        if (it.l == 0) return 3 * static_cast<std::int64_t>(it.s0) + j;
        return 3 * static_cast<std::int64_t>(pt.sub_nodes[it.l][it.s0 + j / 3]) + (j % 3);
    };
    auto load_b = [&](std::int32_t q, Item& it, double* bb) {
        it.l = level_of(q);
        const std::int32_t s = q - pt.base[it.l];
        it.s0 = pt.sub_ptr[it.l][s];
        it.dim = 3 * (pt.sub_ptr[it.l][s + 1] - it.s0);
#pragma unroll
        for (int t = 0; t < RB; ++t) {
            const int j = lane + 32 * t;
            bb[t] = j < it.dim ? ldg_issue(pt.rin[it.l] + row_index(it, j)) : 0.0;
        }
    };
    Item cur{0, 0, 0};
    double b[RB];
    if (nloc > 0) load_b(item(0), cur, b);
    double dsum = 0;
    for (int i = 0; i < nloc; ++i, ++cnt) {
        const int st = static_cast<int>(cnt % kSP);
#pragma unroll
        for (int t = 0; t < RB; ++t)
            if (lane + 32 * t < kK) bs[lane + 32 * t] = b[t];
        Item nxt{0, 0, 0};
        double bn[RB];
        if (i + 1 < nloc) load_b(item(i + 1), nxt, bn);
        __syncwarp();
        mbar_wait(&bar[st], (cnt / kSP) & 1u);
        const double* M = ring + static_cast<std::size_t>(st) * slot;
        double* out = pt.out[cur.l];
        dsum += pair_solve<kK>(M, bs, lane, half, cur.dim,
                               [&](int j, double v) { out[row_index(cur, j)] = v; });
        pair_sync(pair);
        if (half == 0 && i + kSP < nloc) issue(item(i + kSP), cnt + kSP);
        cur = nxt;
#pragma unroll
        for (int t = 0; t < RB; ++t) b[t] = bn[t];
    }
    return dsum;
}

// ---- F: prolongation + p update (+ clears) ------------------------------------
__device__ void final_phase(const Persist& P, double beta, bool zero_tmp) {
    const FinalSo& fa = P.fa;
    const std::int64_t stride = static_cast<std::int64_t>(gridDim.x) * kPT;
    for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(kPT) + threadIdx.x; i < P.n; i += stride) {
        const std::int64_t g = 3 * i;
        std::int32_t nd[kMaxLevels];
#pragma unroll
        for (int l = 0; l < kMaxLevels; ++l)
            if (l < fa.n_coarse) nd[l] = fa.agg[l][i];
        double z0 = P.z[g], z1 = P.z[g + 1], z2 = P.z[g + 2];
        const double p0 = P.p[g], p1 = P.p[g + 1], p2 = P.p[g + 2];
#pragma unroll
        for (int l = 0; l < kMaxLevels; ++l)
            if (l < fa.n_coarse) {
                const double* yl = fa.y[l] + 3 * static_cast<std::int64_t>(nd[l]);
                z0 += yl[0];
                z1 += yl[1];
                z2 += yl[2];
            }
        P.p[g] = z0 + beta * p0;
        P.p[g + 1] = z1 + beta * p1;
        P.p[g + 2] = z2 + beta * p2;
        P.ap[g] = 0.0;
        P.ap[g + 1] = 0.0;
        P.ap[g + 2] = 0.0;
        if (zero_tmp) {
            P.tmp[g] = 0.0;
            P.tmp[g + 1] = 0.0;
            P.tmp[g + 2] = 0.0;
        }
    }
    const std::int64_t tid = blockIdx.x * static_cast<std::int64_t>(kPT) + threadIdx.x;
    for (int l = 0; l < fa.n_clear; ++l)
        for (std::int64_t i = tid; i < fa.clear_n[l]; i += stride) fa.clear[l][i] = 0.0;
}

template <int kK, int kSP, int kSS>
__global__ void __launch_bounds__(kPT, 2) k_pcg_persistent(Persist P) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ double red[32];
    if (P.flags[F_DONE]) return;  // !(rho0 > 0) in the init sequence (pcg.hpp:56)
    cg::grid_group grid = cg::this_grid();
    std::uint64_t* sbar = reinterpret_cast<std::uint64_t*>(smem + P.union_bytes);
    std::uint64_t* pbar = sbar + kPWarps * kSS;
    if (threadIdx.x == 0) {
        for (int i = 0; i < kPWarps * kSS + kPPairs * kSP; ++i) mbar_init(&sbar[i], 1);
        fence_mbar_init();
    }
    __syncthreads();
    std::uint32_t sp_cnt = 0, pc_cnt = 0;  // ring positions (per warp / per pair)
    double* part_a = P.partials;
    double* part_b = P.partials + gridDim.x;
    double rho = P.scal[S_RHO0];
    const double rho0 = P.scal[S_RHO_INIT];
    const double stop = P.scal[S_STOP];
    const bool lead = blockIdx.x == 0 && threadIdx.x == 0;
    const bool timed = P.phase_ns != nullptr && lead;
    unsigned long long t_s = 0, t_u = 0, t_p = 0, t_f = 0, t0 = timed ? gtimer() : 0;
    int k = 1;
    bool done = false;
    for (; k <= P.max_iters; ++k) {
        // S
        store_partial(spmv_phase<true, kSS>(P, P.p, P.ap, smem, sbar, sp_cnt), part_a, red);
        phase_sync(grid);
        const double pap = sum_partials(part_a, red);
        if (timed) { const unsigned long long t = gtimer(); t_s += t - t0; t0 = t; }
        if (!(pap > 0)) {  // pcg.hpp:61-66
            if (lead) {
                P.flags[F_DONE] = 1;
                P.flags[F_ITERS] = k - 1;
                P.scal[S_REL] = sqrt(fabs(rho) / rho0);
            }
            done = true;
            break;
        }
        const double alpha = rho / pap;
        // U
        if (P.restart > 0 && k % P.restart == 0) {  // pcg.hpp:69-72: x += alpha p; r = b - A x
            const std::int64_t n3 = 3 * static_cast<std::int64_t>(P.n);
            for (std::int64_t g = blockIdx.x * static_cast<std::int64_t>(kPT) + threadIdx.x; g < n3;
                 g += static_cast<std::int64_t>(gridDim.x) * kPT)
                P.x[g] += alpha * P.p[g];
            phase_sync(grid);
            spmv_phase<false, kSS>(P, P.x, P.tmp, smem, sbar, sp_cnt);
            phase_sync(grid);
            update_phase<M_RESTART>(P, alpha, P.tmp, reinterpret_cast<double*>(smem));
        } else {
            update_phase<M_UPDATE>(P, alpha, P.ap, reinterpret_cast<double*>(smem));
        }
        phase_sync(grid);
        if (timed) { const unsigned long long t = gtimer(); t_u += t - t0; t0 = t; }
        // P
        store_partial(precond_phase<kK, kSP>(P, smem, pbar, pc_cnt), part_b, red);
        phase_sync(grid);
        const double rz = sum_partials(part_b, red);
        if (timed) { const unsigned long long t = gtimer(); t_p += t - t0; t0 = t; }
        if (lead) {
            P.flags[F_ITERS] = k;
            P.scal[S_REL] = sqrt(fabs(rz) / rho0);
        }
        if (rz <= stop) {  // pcg.hpp:76-82
            if (lead) {
                P.flags[F_DONE] = 1;
                P.flags[F_CONVERGED] = 1;
            }
            done = true;
            break;
        }
        const double beta = rz / rho;
        rho = rz;
        // F
        final_phase(P, beta, P.restart > 0 && (k + 1) % P.restart == 0);
        phase_sync(grid);
        if (timed) { const unsigned long long t = gtimer(); t_f += t - t0; t0 = t; }
    }
    if (lead) {
        if (!done) P.scal[S_RHO0 + (P.max_iters & 1)] = rho;  // ran out (pcg.hpp:86-87)
        if (P.phase_ns) {
            P.phase_ns[0] += t_s;
            P.phase_ns[1] += t_u;
            P.phase_ns[2] += t_p;
            P.phase_ns[3] += t_f;
        }
    }
}

}  // namespace

// The solve-order kernels apply when the levels were built in solve order,
// there are >= 2 levels and every subdomain fits the unrolled mat-vec (fill <= 32).
bool so_supported(const Ctx& c) {
    if (!(c.pkind == kMas && c.perm_active) || c.levels.size() < 2 || c.levels.size() > kMaxLevels) return false;
    for (const auto& L : c.levels)
        if (L->max_fill > 32) return false;
    return true;
}

template <int kMode>
void launch_update_so(Ctx& c, const PcgArgs& a) {
    SoRestrict so{};
    const DeviceLevel& L0 = *c.levels[0];
    so.n_levels = static_cast<int>(c.levels.size());
    so.n0_parts = L0.n_parts;
    so.sub_ptr0 = L0.sub_ptr.p;
    so.up_first0 = L0.up_first.p;
    so.upc_ptr0 = L0.upc_ptr.p;
    so.upc_node0 = L0.upc_node.p;
    for (int l = 1; l < so.n_levels; ++l) {
        so.rr[l] = c.levels[l]->rr.p;
        so.up_node[l] = c.levels[l]->up_node.p;
        if (l >= 2) so.anc[l] = c.levels[l]->anc.p;
    }
    so.max_fill0 = L0.max_fill;
    so.subs = c.upd_subs;
    const int grid = static_cast<int>(std::max<std::int64_t>(1, ceil_div(L0.n_parts, so.subs)));
    const std::size_t smem = update_tile_smem(L0.max_fill, so.subs);
    static bool attr = false;
    if (!attr) {
        ADIPC_CUDA(cudaFuncSetAttribute(k_update_so<kMode>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024));
        attr = true;
    }
    ADIPC_CUDA(launch_pdl(k_update_so<kMode>, dim3(grid), dim3(kUpdThreads), smem, c.stream, c.pdl, so, a));
    ADIPC_LAUNCH_CHECK();
}
template void launch_update_so<M_UPDATE>(Ctx&, const PcgArgs&);
template void launch_update_so<M_RESTART>(Ctx&, const PcgArgs&);

// Byte-balanced split points of every level over np work units, cached on
// the context per (levels, np). Computed outside stream capture
// (prepare_work_splits, from pcg.cu before the iteration graphs are captured).
const std::int32_t* work_split(Ctx& c, int np) {
    for (auto& e : c.splits)
        if (e.np == np && e.version == c.levels_version) return e.buf.p;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    ADIPC_CUDA(cudaStreamIsCapturing(c.stream, &cs));
    if (cs != cudaStreamCaptureStatusNone) return nullptr;  // equal-count split inside an unprepared capture
    const int L = static_cast<int>(c.levels.size());
    std::vector<std::int32_t> h(static_cast<std::size_t>(L) * (np + 1));
    for (int l = 0; l < L; ++l) {
        // cost of a subdomain ~ a fixed per-item latency (kItemCost, in units
        // of one packed double streamed) + its packed-inverse doubles
        constexpr std::int64_t kItemCost = 700;
        const std::vector<std::int64_t>& off = c.levels[l]->inv_off_host;  // n_parts + 1 cumulative
        const std::int32_t n = c.levels[l]->n_parts;
        auto cost = [&](std::int32_t i) { return off[i] + kItemCost * i; };
        const std::int64_t total = cost(n);
        std::int32_t s = 0;
        for (int p = 0; p <= np; ++p) {
            const std::int64_t target = total * p / np;
            while (s < n && cost(s) < target) ++s;  // first subdomain starting at or after the cut
            h[static_cast<std::size_t>(l) * (np + 1) + p] = p == np ? n : s;
        }
    }
    if (c.splits.size() >= 4) {
        c.splits.front().buf.free();
        c.splits.erase(c.splits.begin());
    }
    c.splits.emplace_back();
    Ctx::Split& e = c.splits.back();
    e.np = np;
    e.version = c.levels_version;
    e.buf.reserve(h.size());
    ADIPC_CUDA(cudaMemcpyAsync(e.buf.p, h.data(), h.size() * sizeof(std::int32_t), cudaMemcpyHostToDevice, c.stream));
    ADIPC_CUDA(cudaStreamSynchronize(c.stream));  // h goes out of scope
    return e.buf.p;
}

struct PcLaunch {
    void* fn = nullptr;
    int slot = 0, pairs = 1, grid = 1;
    std::size_t smem = 0;
};

// launch configuration of k_precond_so (warp pairs, TMA ring per pair)
PcLaunch precond_launch(Ctx& c) {
    PcLaunch L;
    int fill = 1;
    for (const auto& lv : c.levels) fill = std::max(fill, lv->max_fill);
    const int kk = matvec_cols(fill);
    L.slot = static_cast<int>(packed_doubles(kk));
    const int stages = c.l0_stages;
    const std::size_t per_pair = (sizeof(double) * L.slot + sizeof(std::uint64_t)) * stages + sizeof(double) * kk;
    L.pairs = static_cast<int>(std::max<std::size_t>(1, std::min<std::size_t>(c.pc_pairs, (113u * 1024u) / per_pair)));
    L.smem = per_pair * L.pairs;
    if (kk == 24)
        L.fn = stages == 2 ? reinterpret_cast<void*>(k_precond_so<24, 2>) : reinterpret_cast<void*>(k_precond_so<24, 3>);
    else if (kk == 48)
        L.fn = stages == 2 ? reinterpret_cast<void*>(k_precond_so<48, 2>) : reinterpret_cast<void*>(k_precond_so<48, 3>);
    else
        L.fn = stages == 2 ? reinterpret_cast<void*>(k_precond_so<96, 2>) : reinterpret_cast<void*>(k_precond_so<96, 3>);
    ADIPC_CUDA(cudaFuncSetAttribute(L.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(L.smem)));
    int occ = 0;
    ADIPC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, L.fn, 64 * L.pairs, L.smem));
    if (occ < 1) throw StatusError(kInvalidArgument, "preconditioner ring does not fit in shared memory");
    int sms = kSMs;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c.device);
    std::int64_t items = 0;
    for (const auto& lv : c.levels) items += lv->n_parts;
    L.grid = static_cast<int>(std::max<std::int64_t>(1, std::min<std::int64_t>(static_cast<std::int64_t>(sms) * occ,
                                                                                  ceil_div(items, L.pairs))));
    return L;
}

// z = M r: every level in one persistent launch (k_precond_so); r.z -> *dot
void launch_precond_so(Ctx& c, const double* r, double* z, const int* flags, double* partials, unsigned* ticket,
                       double* dot) {
    PrecondTable pt{};
    pt.n = static_cast<int>(c.levels.size());
    if (const char* e = std::getenv("ADIPC_DEBUG_PC_LEVELS")) pt.n = std::min(pt.n, std::max(1, std::atoi(e)));  // timing experiments only
    if (const char* e = std::getenv("ADIPC_DEBUG_PC_NOMATH")) pt.dbg_nomath = std::atoi(e);
    pt.l0_keep = static_cast<std::int64_t>(c.levels[0]->inv_doubles * static_cast<double>(c.l0_keep_1024) / 1024.0);

    int fill = 1;
    for (int l = 0; l < pt.n; ++l) {
        const DeviceLevel& L = *c.levels[l];
        pt.base[l + 1] = pt.base[l] + L.n_parts;
        pt.sub_ptr[l] = L.sub_ptr.p;
        pt.sub_nodes[l] = l == 0 ? nullptr : L.sub_nodes.p;
        pt.inv_off[l] = L.inv_off.p;
        pt.inv[l] = L.inv.p;
        pt.rin[l] = l == 0 ? r : L.rr.p;
        pt.out[l] = l == 0 ? z : L.y.p;
        fill = std::max(fill, L.max_fill);
    }
    const int kk = matvec_cols(fill);
    const int slot = static_cast<int>(packed_doubles(kk));
    const int stages = c.l0_stages;
    int sms = kSMs;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c.device);
    if (c.pc_variant == 3 && kk <= 48) {  // warp-specialised: producer + consumers, CTA-wide ring
        int sms = kSMs;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c.device);
#define ADIPC_WS(K, NS, NC)                                                                                   \
    do {                                                                                                      \
        const std::size_t smw = sizeof(double) * (static_cast<std::size_t>(NS) * slot + static_cast<std::size_t>(NC) * 2 * (K + 2)) + \
                                sizeof(std::uint64_t) * 2 * NS;                                               \
        ADIPC_CUDA(cudaFuncSetAttribute(k_precond_ws<K, NS, NC>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                        static_cast<int>(smw)));                                              \
        k_precond_ws<K, NS, NC><<<sms, 32 * (NC + 1), smw, c.stream>>>(pt, partials, ticket, dot, flags, slot); \
    } while (0)
        if (kk == 24)
            ADIPC_WS(24, 22, 8);
        else if (c.ws_cons == 4)
            ADIPC_WS(48, 22, 4);
        else if (c.ws_cons == 6)
            ADIPC_WS(48, 22, 6);
        else if (c.ws_cons == 10)
            ADIPC_WS(48, 22, 10);
        else
            ADIPC_WS(48, 22, 8);
#undef ADIPC_WS
    } else if (c.pc_variant == 2 && kk <= 48) {  // two items per warp (half-warps), one warp per CTA
        constexpr int wpc = 1;
        const std::size_t per_warp = (sizeof(double) * 2 * slot + sizeof(std::uint64_t)) * stages +
                                     sizeof(double) * 2 * (kk + 2);
        const std::size_t sm2 = per_warp * wpc;
#define ADIPC_PC2(K, S)                                                                                       \
    do {                                                                                                      \
        ADIPC_CUDA(cudaFuncSetAttribute(k_precond_so2<K, S>, cudaFuncAttributeMaxDynamicSharedMemorySize,     \
                                        static_cast<int>(sm2)));                                              \
        int occ = 0;                                                                                          \
        ADIPC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_precond_so2<K, S>, 32 * wpc, sm2));  \
        if (occ < 1) throw StatusError(kInvalidArgument, "preconditioner ring does not fit in shared memory"); \
        const int grid = static_cast<int>(std::min<std::int64_t>(static_cast<std::int64_t>(sms) * occ,          \
                                                                 ceil_div(pt.base[pt.n], 2 * wpc)));          \
        k_precond_so2<K, S><<<std::max(grid, 1), 32 * wpc, sm2, c.stream>>>(pt, partials, ticket, dot, flags,   \
                                                                            slot);                            \
    } while (0)
        if (kk == 24) {
            if (stages == 2) ADIPC_PC2(24, 2); else ADIPC_PC2(24, 3);
        } else {
            if (stages == 2) ADIPC_PC2(48, 2); else ADIPC_PC2(48, 3);
        }
#undef ADIPC_PC2
    } else if (c.pc_variant == 1 && kk <= 48) {  // one warp per item, 4 warps per CTA
        const std::size_t per_warp = (sizeof(double) * slot + sizeof(std::uint64_t)) * stages + sizeof(double) * kk;
        const int wpc = 4;
        const std::size_t sm1 = per_warp * wpc;
#define ADIPC_PC1(K, S)                                                                                       \
    do {                                                                                                      \
        ADIPC_CUDA(cudaFuncSetAttribute(k_precond_so1<K, S>, cudaFuncAttributeMaxDynamicSharedMemorySize,     \
                                        static_cast<int>(sm1)));                                              \
        int occ = 0;                                                                                          \
        ADIPC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_precond_so1<K, S>, 32 * wpc, sm1));  \
        if (occ < 1) throw StatusError(kInvalidArgument, "preconditioner ring does not fit in shared memory"); \
        const int grid = static_cast<int>(std::min<std::int64_t>(static_cast<std::int64_t>(sms) * occ,          \
                                                                 ceil_div(pt.base[pt.n], wpc)));              \
        k_precond_so1<K, S><<<std::max(grid, 1), 32 * wpc, sm1, c.stream>>>(pt, partials, ticket, dot, flags,   \
                                                                            slot);                            \
    } while (0)
        if (kk == 24) {
            if (stages == 2) ADIPC_PC1(24, 2); else ADIPC_PC1(24, 3);
        } else {
            if (stages == 2) ADIPC_PC1(48, 2); else ADIPC_PC1(48, 3);
        }
#undef ADIPC_PC1
    } else {
        const PcLaunch L = precond_launch(c);
        pt.np = L.grid * L.pairs;
        pt.split = c.pc_split ? work_split(c, pt.np) : nullptr;
        int slot_arg = L.slot;
        void* args[] = {&pt, &partials, &ticket, &dot, const_cast<int**>(&flags), &slot_arg};
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(L.grid);
        cfg.blockDim = dim3(64 * L.pairs);
        cfg.dynamicSmemBytes = L.smem;
        cfg.stream = c.stream;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = c.pdl ? 1 : 0;
        ADIPC_CUDA(cudaLaunchKernelExC(&cfg, L.fn, args));
    }
    ADIPC_LAUNCH_CHECK();
}

// grid upper bound of the solve-order kernels (sizes the per-CTA partials)
int so_partials(const Ctx& c) {
    (void)c;
    return kSMs * 8;
}

namespace {
__global__ void k_pad4(std::int32_t n, const double* __restrict__ p, double* __restrict__ p4) {
    for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        p4[4 * i] = p[3 * i];
        p4[4 * i + 1] = p[3 * i + 1];
        p4[4 * i + 2] = p[3 * i + 2];
        p4[4 * i + 3] = 0.0;
    }
}
}  // namespace

void pad4(Ctx& c, const double* p, double* p4) {
    if (c.A.n == 0) return;
    k_pad4<<<grid_for(c.A.n, 256, 8), 256, 0, c.stream>>>(c.A.n, p, p4);
    ADIPC_LAUNCH_CHECK();
}

template <int kFinal>
void launch_final_so(Ctx& c, double* z, double* p, double* ap, const PcgArgs& a) {
    FinalSo fa{};
    fa.p4 = c.p4_active;
    const int L = static_cast<int>(c.levels.size());
    fa.n_coarse = L - 1;
    for (int l = 1; l < L; ++l) {
        fa.agg[l - 1] = c.levels[l]->agg.p;
        fa.y[l - 1] = c.levels[l]->y.p;
    }
    for (int l = 2; l < L; ++l) {
        fa.clear[fa.n_clear] = c.levels[l]->rr.p;
        fa.clear_n[fa.n_clear] = 3 * static_cast<std::int64_t>(c.levels[l]->n_nodes);
        ++fa.n_clear;
    }
    const int per = c.final_per, block = c.final_block;
    const int grid = static_cast<int>(
        std::max<std::int64_t>(1, ceil_div(ceil_div(c.A.n, 2), static_cast<std::int64_t>(block) * per)));
    if (per == 1)
        ADIPC_CUDA(launch_pdl(k_final_so<kFinal, 1>, dim3(grid), dim3(block), 0, c.stream, c.pdl, c.A.n, fa, z, p, ap, a));
    else if (per == 2)
        k_final_so<kFinal, 2><<<grid, block, 0, c.stream>>>(c.A.n, fa, z, p, ap, a);
    else
        k_final_so<kFinal, 4><<<grid, block, 0, c.stream>>>(c.A.n, fa, z, p, ap, a);
    ADIPC_LAUNCH_CHECK();
}
template void launch_final_so<F_PCG_INIT>(Ctx&, double*, double*, double*, const PcgArgs&);
template void launch_final_so<F_PCG_STEP>(Ctx&, double*, double*, double*, const PcgArgs&);

// zero the RED targets (levels >= 2) before the first update pass
void clear_restrict_so(Ctx& c) {
    for (std::size_t l = 2; l < c.levels.size(); ++l)
        ADIPC_CUDA(cudaMemsetAsync(c.levels[l]->rr.p, 0, sizeof(double) * 3 * c.levels[l]->n_nodes, c.stream));
}

}  // namespace adipc_gpu

namespace adipc_gpu {

// The PCG iterations (after the init sequence of pcg.cu) as one persistent
// cooperative launch. Returns false when the configuration is not covered
// (the caller then runs the per-kernel CUDA-graph iterations).
bool pcg_persistent(Ctx& c, const PcgArgs& a, double* partials, int restart, int max_iters) {
    if (!c.persistent || !so_supported(c) || c.levels.size() > kMaxLevels) return false;
    const DeviceMatrix& M = c.S();
    Persist P{};
    P.rows = M.rows.p;
    P.cols = M.cols.p;
    P.blocks = M.blocks.p;
    P.U = M.U;
    P.n = M.n;
    P.x = a.x;
    P.r = a.r;
    P.p = const_cast<double*>(a.p);
    P.ap = const_cast<double*>(a.ap);
    P.z = c.w.z.p;
    P.tmp = c.w.tmp.p;
    P.b = a.b;
    // restriction
    const DeviceLevel& L0 = *c.levels[0];
    SoRestrict& so = P.so;
    so.n_levels = static_cast<int>(c.levels.size());
    so.n0_parts = L0.n_parts;
    so.sub_ptr0 = L0.sub_ptr.p;
    so.up_first0 = L0.up_first.p;
    so.upc_ptr0 = L0.upc_ptr.p;
    so.upc_node0 = L0.upc_node.p;
    for (int l = 1; l < so.n_levels; ++l) {
        so.rr[l] = c.levels[l]->rr.p;
        so.up_node[l] = c.levels[l]->up_node.p;
        if (l >= 2) so.anc[l] = c.levels[l]->anc.p;
    }
    so.max_fill0 = L0.max_fill;
    // preconditioner table
    PrecondTable& pt = P.pt;
    pt.n = so.n_levels;
    int fill = 1;
    for (int l = 0; l < pt.n; ++l) {
        const DeviceLevel& L = *c.levels[l];
        pt.base[l + 1] = pt.base[l] + L.n_parts;
        pt.sub_ptr[l] = L.sub_ptr.p;
        pt.sub_nodes[l] = l == 0 ? nullptr : L.sub_nodes.p;
        pt.inv_off[l] = L.inv_off.p;
        pt.inv[l] = L.inv.p;
        pt.rin[l] = l == 0 ? a.r : L.rr.p;
        pt.out[l] = l == 0 ? c.w.z.p : L.y.p;
        fill = std::max(fill, L.max_fill);
    }
    // prolongation
    FinalSo& fa = P.fa;
    fa.n_coarse = pt.n - 1;
    for (int l = 1; l < pt.n; ++l) {
        fa.agg[l - 1] = c.levels[l]->agg.p;
        fa.y[l - 1] = c.levels[l]->y.p;
    }
    for (int l = 2; l < pt.n; ++l) {
        fa.clear[fa.n_clear] = c.levels[l]->rr.p;
        fa.clear_n[fa.n_clear] = 3 * static_cast<std::int64_t>(c.levels[l]->n_nodes);
        ++fa.n_clear;
    }
    P.partials = partials;
    P.scal = a.scal;
    P.flags = a.flags;
    P.restart = restart;
    P.max_iters = max_iters;
    if (c.profile) {
        c.phase_ns.reserve(4);
        ADIPC_CUDA(cudaMemsetAsync(c.phase_ns.p, 0, 4 * sizeof(unsigned long long), c.stream));
        P.phase_ns = c.phase_ns.p;
    }
    const int kk = matvec_cols(fill);
    if (kk == 0) return false;
    P.slot_doubles = static_cast<int>(packed_doubles(kk));
    constexpr int kSP = 2, kSS = 4;
    std::size_t ub = std::max<std::size_t>(sizeof(SpmvStage) * kPWarps * kSS,
                                           sizeof(double) * (static_cast<std::size_t>(kPPairs) * kSP * P.slot_doubles +
                                                             static_cast<std::size_t>(kPWarps) * kk));
    P.so.subs = kUpdSubs;
    ub = std::max<std::size_t>(ub, update_tile_smem(L0.max_fill, kUpdSubs));
    ub = (ub + 127) & ~static_cast<std::size_t>(127);
    P.union_bytes = static_cast<int>(ub);
    const std::size_t smem = ub + sizeof(std::uint64_t) * (kPWarps * kSS + kPPairs * kSP);
    ADIPC_CUDA(cudaMemsetAsync(c.w.tmp.p, 0, sizeof(double) * 3 * static_cast<std::size_t>(M.n), c.stream));
    int sms = kSMs;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c.device);
    void* args[] = {&P};
    void* fn = nullptr;
    if (kk == 24)
        fn = reinterpret_cast<void*>(k_pcg_persistent<24, kSP, kSS>);
    else if (kk == 48)
        fn = reinterpret_cast<void*>(k_pcg_persistent<48, kSP, kSS>);
    else
        fn = reinterpret_cast<void*>(k_pcg_persistent<96, kSP, kSS>);
    ADIPC_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    int occ = 0;
    ADIPC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, kPT, smem));
    if (occ < 1) return false;
    const int grid = sms * std::min(occ, 2);
    ADIPC_CUDA(cudaLaunchCooperativeKernel(fn, grid, kPT, args, smem, c.stream));
    ADIPC_LAUNCH_CHECK();
    return true;
}

}  // namespace adipc_gpu

namespace adipc_gpu {

// One PCG iteration after the SpMV: update + every MAS level + prolongation
// (k_iter_so), cooperative launch (the in-kernel arrival counters need every
// CTA resident). Returns false when not applicable.
bool iter_so_supported(const Ctx& c) {
    if (!c.fused || !so_supported(c)) return false;
    int fill = 1;
    for (const auto& L : c.levels) fill = std::max(fill, L->max_fill);
    return matvec_cols(fill) != 0;
}

struct IterLaunch {
    void* fn = nullptr;
    int kk = 0, slot = 0, pairs = 1, grid = 1;
    std::size_t smem = 0;
};

IterLaunch iter_launch(Ctx& c) {
    IterLaunch L;
    int fill = 1;
    for (const auto& lv : c.levels) fill = std::max(fill, lv->max_fill);
    L.kk = matvec_cols(fill);
    L.slot = static_cast<int>(packed_doubles(L.kk));
    const int stages = c.l0_stages;
    const std::size_t per_pair = (sizeof(double) * L.slot + sizeof(std::uint64_t)) * stages +
                                 sizeof(double) * L.kk + sizeof(double) * 40;
    L.pairs = static_cast<int>(std::max<std::size_t>(1, std::min<std::size_t>(4, (113u * 1024u) / per_pair)));
    L.smem = per_pair * L.pairs;
    int sms = kSMs;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c.device);
    if (L.kk == 24)
        L.fn = stages == 2 ? reinterpret_cast<void*>(k_iter_so<24, 2>) : reinterpret_cast<void*>(k_iter_so<24, 3>);
    else if (L.kk == 48)
        L.fn = stages == 2 ? reinterpret_cast<void*>(k_iter_so<48, 2>) : reinterpret_cast<void*>(k_iter_so<48, 3>);
    else
        L.fn = stages == 2 ? reinterpret_cast<void*>(k_iter_so<96, 2>) : reinterpret_cast<void*>(k_iter_so<96, 3>);
    ADIPC_CUDA(cudaFuncSetAttribute(L.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(L.smem)));
    int occ = 0;
    ADIPC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, L.fn, 64 * L.pairs, L.smem));
    if (occ < 1) throw StatusError(kInvalidArgument, "fused iteration kernel does not fit on an SM");
    L.grid = sms * occ;
    return L;
}

void launch_iter_so(Ctx& c, const PcgArgs& a, bool restart, unsigned* counters, double* partials) {
    IterArgs ia{};
    PrecondTable& pt = ia.pt;
    pt.n = static_cast<int>(c.levels.size());
    int fill = 1;
    for (int l = 0; l < pt.n; ++l) {
        const DeviceLevel& L = *c.levels[l];
        pt.base[l + 1] = pt.base[l] + L.n_parts;
        pt.sub_ptr[l] = L.sub_ptr.p;
        pt.sub_nodes[l] = l == 0 ? nullptr : L.sub_nodes.p;
        pt.inv_off[l] = L.inv_off.p;
        pt.inv[l] = L.inv.p;
        pt.rin[l] = l == 0 ? a.r : L.rr.p;
        pt.out[l] = l == 0 ? c.w.z.p : L.y.p;
        fill = std::max(fill, L.max_fill);
    }
    FinalSo& fa = ia.fa;
    fa.n_coarse = pt.n - 1;
    for (int l = 1; l < pt.n; ++l) {
        fa.agg[l - 1] = c.levels[l]->agg.p;
        fa.y[l - 1] = c.levels[l]->y.p;
    }
    for (int l = 2; l < pt.n; ++l) {
        fa.clear[fa.n_clear] = c.levels[l]->rr.p;
        fa.clear_n[fa.n_clear] = 3 * static_cast<std::int64_t>(c.levels[l]->n_nodes);
        ++fa.n_clear;
    }
    const DeviceLevel& L0 = *c.levels[0];
    ia.x = a.x;
    ia.r = a.r;
    ia.p = a.p;
    ia.ap = a.ap;
    ia.b = a.b;
    ia.z = c.w.z.p;
    ia.pout = c.w.p.p;
    ia.apclear = c.w.ap.p;
    ia.tmpclear = nullptr;
    ia.up_first0 = L0.up_first.p;
    ia.upc_ptr0 = L0.upc_ptr.p;
    ia.upc_node0 = L0.upc_node.p;
    ia.rr1 = c.levels[1]->rr.p;
    ia.n_levels = pt.n;
    for (int l = 2; l < pt.n; ++l) {
        ia.rr[l] = c.levels[l]->rr.p;
        ia.anc[l] = c.levels[l]->anc.p;
    }
    ia.n_slots = c.A.n;
    ia.scal = a.scal;
    ia.flags = a.flags;
    ia.counters = counters;
    ia.partials = partials;
    ia.restart_mode = restart ? 1 : 0;
    const IterLaunch L = iter_launch(c);
    const int slot = L.slot, pairs = L.pairs, grid = L.grid;
    const std::size_t smem = L.smem;
    void* fn = L.fn;
    pt.np = grid * pairs;
    pt.split = c.pc_split ? work_split(c, pt.np) : nullptr;
    int slot_arg = slot;
    void* args[] = {&ia, &slot_arg};
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(64 * pairs);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = c.stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    ADIPC_CUDA(cudaLaunchKernelExC(&cfg, fn, args));
    ADIPC_LAUNCH_CHECK();
}

}  // namespace adipc_gpu

namespace adipc_gpu {
IterLaunch iter_launch(Ctx& c);
PcLaunch precond_launch(Ctx& c);
// byte-balanced splits for the launch configurations the PCG iteration graph
// will capture (no allocation may happen while capturing)
void prepare_work_splits(Ctx& c) {
    if (!so_supported(c) || !c.pc_split) return;
    if (iter_so_supported(c)) {
        const IterLaunch L = iter_launch(c);
        work_split(c, L.grid * L.pairs);
    }
    const PcLaunch P = precond_launch(c);
    work_split(c, P.grid * P.pairs);
}
}  // namespace adipc_gpu
