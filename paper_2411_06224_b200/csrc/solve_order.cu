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
    int red_levels;                           // levels >= 2 restricted by RED here (deterministic mode: none)
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
__device__ __forceinline__ void update_tile(const SoRestrict& so, const PcgArgs& a, const double* __restrict__ apv,
                                            std::int32_t tile, double* smem) {
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
    // before the dependency wait: the restriction metadata and the first
    // pass of r, p, x (written two or more kernels back, all complete once
    // the SpMV passed its own wait) — only Ap and alpha come from the SpMV
    for (int i = threadIdx.x; i <= v1 - v0; i += kThreads) uptr[i] = so.upc_ptr0[v0 + i] - slot0;
    for (int i = threadIdx.x; i < slot1 - slot0; i += kThreads) child[i] = so.upc_node0[slot0 + i] - slot0;
    constexpr int kU = 4;
    double rv[kU], pv[kU], xv[kU];
    auto load_pass = [&](std::int64_t gb) {
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const std::int64_t g = gb + u * kThreads;
            if (g < g1) {
                if (kMode == M_UPDATE) {
                    rv[u] = a.r[g];
                    pv[u] = a.p[g];
                    xv[u] = a.x[g];
                } else {
                    rv[u] = a.b[g];
                }
            }
        }
    };
    load_pass(g0 + threadIdx.x);
    double alpha = 0;
    pdl_wait();
    if (a.flags[F_DONE]) return;
    if (!pcg_alpha(a, alpha)) return;  // also the restart pass's breakdown check, as before
    pdl_launch();
    for (std::int64_t gb = g0 + threadIdx.x; gb < g1; gb += kU * kThreads) {
        if (gb != g0 + threadIdx.x) load_pass(gb);
        double av[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const std::int64_t g = gb + u * kThreads;
            if (g < g1) av[u] = apv[g];
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
            if (l < so.red_levels) w[l] = so.anc[l][v];
        double acc = 0;
        for (int q = uptr[i]; q < uptr[i + 1]; ++q) acc += sr[3 * child[q] + comp];
        so.rr[1][3 * static_cast<std::int64_t>(v) + comp] = acc;
#pragma unroll
        for (int l = 2; l < kMaxLevels; ++l)
            if (l < so.red_levels) red_add(so.rr[l] + 3 * static_cast<std::int64_t>(w[l]) + comp, acc);
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
    update_tile<kMode, kUpdThreads>(so, a, a.ap, blockIdx.x, sr);
}

// Deterministic mode: level l >= 2 restricted from level l - 1 in a fixed
// order, r_l[w] = sum of r_{l-1} over w's children in ascending id
// (hierarchy.hpp:53-72 nesting), one thread per (node, component).
__global__ void k_restrict_up(std::int32_t n_nodes, const std::int32_t* __restrict__ upc_ptr,
                              const std::int32_t* __restrict__ upc_node, const double* __restrict__ r_prev,
                              double* __restrict__ r_next, const int* __restrict__ flags) {
    pdl_wait();
    if (flags[F_DONE]) return;
    pdl_launch();
    for (std::int64_t t = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; t < 3 * std::int64_t(n_nodes);
         t += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        const std::int32_t w = static_cast<std::int32_t>(t / 3);
        const int comp = static_cast<int>(t - 3 * std::int64_t(w));
        double acc = 0;
        for (std::int32_t q = upc_ptr[w]; q < upc_ptr[w + 1]; ++q)
            acc += r_prev[3 * static_cast<std::int64_t>(upc_node[q]) + comp];
        r_next[t] = acc;
    }
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
    // b of the current item, one copy per warp: each warp writes its own
    // after the pair barrier that ends the previous item and reads it after
    // its __syncwarp (a copy shared by the pair had both warps store the same
    // values concurrently with the other's reads: compute-sanitizer racecheck)
    double* bs = reinterpret_cast<double*>(smem) + static_cast<std::size_t>(npc) * kStages * slot_doubles +
                 static_cast<std::size_t>(2 * pair + half) * kK;
    std::uint64_t* bar = reinterpret_cast<std::uint64_t*>(
                             reinterpret_cast<double*>(smem) + static_cast<std::size_t>(npc) * kStages * slot_doubles +
                             static_cast<std::size_t>(2 * npc) * kK) +
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
    // finite slot contents beyond each inverse (packed_matvec reads them x 0)
    for (int i = half * 32 + lane; i < kStages * slot_doubles; i += 64) ring[i] = 0.0;
    fence_proxy_async();
    pair_sync(pair);
    // one thread of the pair: the inverse of packed offset range [o, o1) of level l
    auto issue_at = [&](int l, std::int64_t o, std::int64_t o1, int st) {
        const std::uint32_t bytes = static_cast<std::uint32_t>((o1 - o) * 8);
        mbar_arrive_expect_tx(&bar[st], bytes);
        if (l == 0)  // streamed once per application
            bulk_g2s_evict_first(ring + static_cast<std::size_t>(st) * slot_doubles, pt.inv[0] + o, bytes, &bar[st]);
        else  // coarse inverses (~26 MB at cfg5) stay L2-resident across iterations
            bulk_g2s_evict_last(ring + static_cast<std::size_t>(st) * slot_doubles, pt.inv[l] + o, bytes, &bar[st]);
    };
    auto issue = [&](std::int32_t q, int st) {
        const int l = level_of(q);
        const std::int32_t s = q - pt.base[l];
        issue_at(l, pt.inv_off[l][s], pt.inv_off[l][s + 1], st);
    };
    const bool leader = half == 0 && lane == 0;
    if (leader) {
        for (int st = 0; st < kStages; ++st) mbar_init(&bar[st], 1);
        fence_mbar_init();
        for (int st = 0; st < kStages && st < nloc; ++st) issue(item(st), st);
    }
    pair_sync(pair);
    // the inverses are constant during the solve: the ring above fills while
    // the predecessor (update pass) drains; its outputs are read from here on
    pdl_wait();
    if (flags && flags[F_DONE]) {  // PCG already finished: drain the issued copies, leave
        if (leader)
            for (int st = 0; st < kStages && st < nloc; ++st) mbar_wait(&bar[st], 0);
        return;
    }
    pdl_launch();
    // Every global load on an item's critical path is issued one item ahead
    // of its use: the subdomain range (sub_ptr) two items ahead, the residual
    // gathers of the next item, and (leader) the packed-inverse offsets of
    // the refill — so the pair never waits on a dependent load round trip
    // between the ring slot landing and its refill being issued.
    struct Item {
        int l;
        std::int32_t s0, dim;
    };
    struct Meta {  // sub_ptr[s], sub_ptr[s + 1] of an item (loads in flight)
        int l;
        std::int32_t lo, hi;
    };
    auto meta_load = [&](int idx, Meta& m) {
        m.l = 0;
        m.lo = m.hi = 0;
        if (idx < nloc) {
            const std::int32_t q = item(idx);
            m.l = level_of(q);
            const std::int32_t s = q - pt.base[m.l];
            m.lo = ldg_issue(pt.sub_ptr[m.l] + s);
            m.hi = ldg_issue(pt.sub_ptr[m.l] + s + 1);
        }
    };
    auto row_index = [&](const Item& it, int j) -> std::int64_t {
        if (it.l == 0) return 3 * static_cast<std::int64_t>(it.s0) + j;
        return 3 * static_cast<std::int64_t>(pt.sub_nodes[it.l][it.s0 + j / 3]) + (j % 3);
    };
    auto load_b = [&](const Meta& m, Item& it, double* bb) {
        it.l = m.l;
        it.s0 = m.lo;
        it.dim = 3 * (m.hi - m.lo);
#pragma unroll
        for (int t = 0; t < RB; ++t) {
            const int j = lane + 32 * t;
            bb[t] = j < it.dim ? ldg_issue(pt.rin[it.l] + row_index(it, j)) : 0.0;
        }
    };
    Item cur{0, 0, 0};
    double b[RB];
    Meta mn;  // item i + 1
    {
        Meta m0;
        meta_load(0, m0);
        meta_load(1, mn);
        load_b(m0, cur, b);
    }
    double dsum = 0;
    int st = 0;
    std::uint32_t par = 0;
    for (int i = 0; i < nloc; ++i) {
#pragma unroll
        for (int t = 0; t < RB; ++t)
            if (lane + 32 * t < kK) bs[lane + 32 * t] = b[t];
        // refill target (leader): offsets of item i + kStages
        int rl = 0;
        std::int64_t ro = 0, ro1 = 0;
        if (leader && i + kStages < nloc) {
            const std::int32_t q = item(i + kStages);
            rl = level_of(q);
            const std::int32_t s = q - pt.base[rl];
            ro = ldg_issue(pt.inv_off[rl] + s);
            ro1 = ldg_issue(pt.inv_off[rl] + s + 1);
        }
        Item nxt{0, 0, 0};
        double bn[RB];
        if (i + 1 < nloc) load_b(mn, nxt, bn);
        Meta mnn;
        meta_load(i + 2, mnn);
        __syncwarp();
        mbar_wait(&bar[st], par);
        const double* M = ring + static_cast<std::size_t>(st) * slot_doubles;
        double* out = pt.out[cur.l];
        dsum += pair_solve<kK>(M, bs, lane, half, cur.dim,
                                   [&](int j, double v) { out[row_index(cur, j)] = v; });
        pair_sync(pair);  // both warps are done with the slot (and with bs before its next write)
        if (leader && i + kStages < nloc) {
            fence_proxy_async();
            issue_at(rl, ro, ro1, st);
        }
        if (++st == kStages) {
            st = 0;
            par ^= 1u;
        }
        cur = nxt;
        mn = mnn;
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
};

template <int kFinal>
__global__ void __launch_bounds__(512) k_final_so(std::int32_t n, FinalSo fa, const double* __restrict__ z,
                                                 double* __restrict__ p, double* __restrict__ ap, PcgArgs a) {
    // one slot pair (6 doubles, three 128-bit accesses per vector) per thread
    // (the grid covers n). Everything this pass reads that the preconditioner
    // does not write — the aggregation maps and p — is loaded, and Ap (read
    // by the update pass, which completed before the preconditioner passed
    // its own dependency wait) is cleared, BEFORE the dependency wait.
    const std::int64_t nthreads = static_cast<std::int64_t>(gridDim.x) * blockDim.x;
    const std::int64_t tid = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x;
    const std::int64_t pr = tid, sl0 = 2 * pr;
    const bool have = sl0 < n, two = sl0 + 1 < n;
    std::int32_t nd[kMaxLevels][2];
    double pp[6];
    if (have) {
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
        if (two) {
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                if (kFinal != F_PCG_INIT) {
                    const double2 pv = reinterpret_cast<const double2*>(p)[3 * pr + q];
                    pp[2 * q] = pv.x;
                    pp[2 * q + 1] = pv.y;
                } else {
                    pp[2 * q] = pp[2 * q + 1] = 0.0;
                }
                reinterpret_cast<double2*>(ap)[3 * pr + q] = make_double2(0.0, 0.0);
            }
        } else {
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                pp[q] = kFinal != F_PCG_INIT ? p[3 * sl0 + q] : 0.0;
                pp[3 + q] = 0.0;
                ap[3 * sl0 + q] = 0.0;
            }
        }
    }
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
    if (have) {
        double zz[6];
        if (two) {
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                const double2 zv = reinterpret_cast<const double2*>(z)[3 * pr + q];
                zz[2 * q] = zv.x;
                zz[2 * q + 1] = zv.y;
            }
        } else {
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                zz[q] = z[3 * sl0 + q];
                zz[3 + q] = 0.0;
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
            for (int q = 0; q < 3; ++q)
                reinterpret_cast<double2*>(p)[3 * pr + q] = make_double2(pn[2 * q], pn[2 * q + 1]);
        } else {
#pragma unroll
            for (int q = 0; q < 3; ++q) p[3 * sl0 + q] = pn[q];
        }
    }
    // clear the RED targets of the next update pass
    for (int l = 0; l < fa.n_clear; ++l)
        for (std::int64_t i = tid; i < fa.clear_n[l]; i += nthreads) fa.clear[l][i] = 0.0;
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
    so.red_levels = c.deterministic ? 2 : so.n_levels;
    // tiles sized so the grid is ONE wave of resident CTAs (at least kUpdSubs
    // subdomains per tile): a second, mostly empty wave costs a whole CTA
    // latency chain (cfg5: 687 tiles of 32 on 592 resident CTAs)
    int sms = kSMs, occ = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c.device);
    so.subs = kUpdSubs;
    for (int it = 0; it < 2; ++it) {  // smem depends on subs; occupancy on smem
        const std::size_t sm = update_tile_smem(L0.max_fill, so.subs);
        ADIPC_CUDA(cudaFuncSetAttribute(k_update_so<kMode>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(sm)));
        ADIPC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_update_so<kMode>, kUpdThreads, sm));
        const std::int64_t slots = static_cast<std::int64_t>(sms) * std::max(occ, 1);
        so.subs = static_cast<int>(std::max<std::int64_t>(kUpdSubs, ceil_div(L0.n_parts, slots)));
    }

    const int grid = static_cast<int>(std::max<std::int64_t>(1, ceil_div(L0.n_parts, so.subs)));
    const std::size_t smem = update_tile_smem(L0.max_fill, so.subs);
    // a per-device function attribute: set on every launch (cheap, legal while
    // capturing), so contexts on different devices each get it
    ADIPC_CUDA(cudaFuncSetAttribute(k_update_so<kMode>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(smem)));
    ADIPC_CUDA(launch_pdl(k_update_so<kMode>, dim3(grid), dim3(kUpdThreads), smem, c.stream, true, so, a));
    ADIPC_LAUNCH_CHECK();
    if (c.deterministic)
        for (int l = 2; l < so.n_levels; ++l) {
            const DeviceLevel& P = *c.levels[l - 1];
            const DeviceLevel& N = *c.levels[l];
            ADIPC_CUDA(launch_pdl(k_restrict_up, dim3(grid_for(3 * std::int64_t(N.n_nodes), 256, 8)), dim3(256), 0,
                                  c.stream, true, N.n_nodes, P.upc_ptr.p, P.upc_node.p, P.rr.p, N.rr.p, a.flags));
            ADIPC_LAUNCH_CHECK();
        }
}
template void launch_update_so<M_UPDATE>(Ctx&, const PcgArgs&);
template void launch_update_so<M_RESTART>(Ctx&, const PcgArgs&);

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
    const std::size_t per_pair = (sizeof(double) * L.slot + sizeof(std::uint64_t)) * stages + 2 * sizeof(double) * kk;
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
    ADIPC_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c.device));
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
    for (int l = 0; l < pt.n; ++l) {
        const DeviceLevel& L = *c.levels[l];
        pt.base[l + 1] = pt.base[l] + L.n_parts;
        pt.sub_ptr[l] = L.sub_ptr.p;
        pt.sub_nodes[l] = l == 0 ? nullptr : L.sub_nodes.p;
        pt.inv_off[l] = L.inv_off.p;
        pt.inv[l] = L.inv.p;
        pt.rin[l] = l == 0 ? r : L.rr.p;
        pt.out[l] = l == 0 ? z : L.y.p;
    }
    const PcLaunch L = precond_launch(c);
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
    cfg.numAttrs = 1;
    ADIPC_CUDA(cudaLaunchKernelExC(&cfg, L.fn, args));
    ADIPC_LAUNCH_CHECK();
}

template <int kFinal>
void launch_final_so(Ctx& c, double* z, double* p, double* ap, const PcgArgs& a) {
    FinalSo fa{};
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
    constexpr int block = 256;
    // one CTA per 512 slots (a one-wave grid-stride variant measured slower
    // in the PDL-chained graph: 137.0 vs 135.1 us per cfg5 iteration)
    const int grid = static_cast<int>(std::max<std::int64_t>(1, ceil_div(ceil_div(c.A.n, 2), block)));
    ADIPC_CUDA(launch_pdl(k_final_so<kFinal>, dim3(grid), dim3(block), 0, c.stream, true, c.A.n, fa, z, p, ap, a));
    ADIPC_LAUNCH_CHECK();
}
// grid upper bound of the solve-order kernels (sizes the per-CTA partials)
int so_partials(const Ctx& c) { return kSMs * 8; }

template void launch_final_so<F_PCG_INIT>(Ctx&, double*, double*, double*, const PcgArgs&);
template void launch_final_so<F_PCG_STEP>(Ctx&, double*, double*, double*, const PcgArgs&);

// zero the RED targets (levels >= 2) before the first update pass
void clear_restrict_so(Ctx& c) {
    for (std::size_t l = 2; l < c.levels.size(); ++l)
        ADIPC_CUDA(cudaMemsetAsync(c.levels[l]->rr.p, 0, sizeof(double) * 3 * c.levels[l]->n_nodes, c.stream));
}

}  // namespace adipc_gpu
