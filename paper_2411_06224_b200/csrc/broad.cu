// Device broad phase (contact/broad_phase.hpp:143-211):
// vertex-triangle and edge-edge candidates of the contact surface whose
// inflated (optionally swept) AABBs overlap, stencils sharing a node dropped,
// sorted and duplicate free — the same set and order as the reference's hash
// grid (its result is exactly the overlapping pairs; tests/test_contact.cpp:
// 341-409 pins that against brute force).
//
// Uniform grid with the reference's cell size (mean triangle extent +
// inflation), exact integer cell coordinates, an open hash table of (cell,
// primitive) entries: count -> scan -> fill. Every query enumerates the cells
// of its box and keeps a pair only in the FIRST cell the two cell ranges
// share (componentwise max of the two low cells), so each pair is found once
// without a global sort; each query's pairs are then sorted in place (short
// lists) — query order x partner order = the reference's lexicographic order.
#include <cmath>

#include "context.hpp"
#include "scan.cuh"

namespace adipc_gpu {

namespace {

using Box = BpBox;
using Entry = BpEntry;
struct Cell {
    int x, y, z;
};

__device__ __forceinline__ void grow(Box& b, const double* p) {
    for (int a = 0; a < 3; ++a) {
        b.lo[a] = fmin(b.lo[a], p[a]);
        b.hi[a] = fmax(b.hi[a], p[a]);
    }
}
__device__ __forceinline__ Box empty_box() {
    Box b;
    for (int a = 0; a < 3; ++a) {
        b.lo[a] = 1.7976931348623157e308;
        b.hi[a] = -1.7976931348623157e308;
    }
    return b;
}
// swept_point (broad_phase.hpp:125-131): the node, and node + disp
__device__ __forceinline__ void grow_node(Box& b, const double* pos, const double* disp, int v) {
    const double* p = pos + 3 * static_cast<std::int64_t>(v);
    grow(b, p);
    if (disp) {
        const double* d = disp + 3 * static_cast<std::int64_t>(v);
        const double e[3] = {p[0] + d[0], p[1] + d[1], p[2] + d[2]};
        grow(b, e);
    }
}
__device__ __forceinline__ void inflate(Box& b, double r) {
    for (int a = 0; a < 3; ++a) {
        b.lo[a] -= r;
        b.hi[a] += r;
    }
}
__device__ __forceinline__ bool overlaps(const Box& a, const Box& b) {
    for (int k = 0; k < 3; ++k)
        if (!(a.lo[k] <= b.hi[k] && b.lo[k] <= a.hi[k])) return false;
    return true;
}
__device__ __forceinline__ Cell cell_of(const double* p, double h) {
    return {static_cast<int>(floor(p[0] / h)), static_cast<int>(floor(p[1] / h)), static_cast<int>(floor(p[2] / h))};
}
__device__ __forceinline__ std::uint32_t bucket_of(int x, int y, int z, std::uint32_t mask) {
    std::uint64_t k = (static_cast<std::uint64_t>(static_cast<std::uint32_t>(x)) * 0x9E3779B97F4A7C15ull) ^
                      (static_cast<std::uint64_t>(static_cast<std::uint32_t>(y)) * 0xC2B2AE3D27D4EB4Full) ^
                      (static_cast<std::uint64_t>(static_cast<std::uint32_t>(z)) * 0x165667B19E3779F9ull);
    k ^= k >> 29;
    return static_cast<std::uint32_t>(k) & mask;
}

struct Surface {
    const double* pos;
    const double* disp;
    std::int32_t n_verts, n_edges, n_tris;
    const int* verts;
    const int* edges;
    const int* tris;
    double half;
};

// primitive boxes: kind 0 triangles (also their un-inflated max extent), 1 edges
__global__ void k_boxes(Surface s, Box* __restrict__ tri_box, Box* __restrict__ edge_box, double* __restrict__ extent) {
    double ext = 0;
    for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < s.n_tris + s.n_edges;
         i += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        Box b = empty_box();
        if (i < s.n_tris) {
            for (int k = 0; k < 3; ++k) grow_node(b, s.pos, s.disp, s.tris[3 * i + k]);
            ext += fmax(fmax(b.hi[0] - b.lo[0], b.hi[1] - b.lo[1]), b.hi[2] - b.lo[2]);
            inflate(b, s.half);
            tri_box[i] = b;
        } else {
            const std::int64_t e = i - s.n_tris;
            for (int k = 0; k < 2; ++k) grow_node(b, s.pos, s.disp, s.edges[2 * e + k]);
            inflate(b, s.half);
            edge_box[e] = b;
        }
    }
    for (int o = 16; o > 0; o >>= 1) ext += __shfl_xor_sync(0xffffffffu, ext, o);
    if ((threadIdx.x & 31) == 0 && ext != 0) atomicAdd(extent, ext);
}

__device__ __forceinline__ std::int64_t cells_in(const Box& b, double h) {
    const Cell lo = cell_of(b.lo, h), hi = cell_of(b.hi, h);
    return static_cast<std::int64_t>(hi.x - lo.x + 1) * (hi.y - lo.y + 1) * (hi.z - lo.z + 1);
}

__global__ void k_grid_count(const Box* __restrict__ box, std::int32_t n, double h, std::int32_t* __restrict__ cnt) {
    for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<std::int64_t>(gridDim.x) * blockDim.x)
        cnt[i] = static_cast<std::int32_t>(cells_in(box[i], h));
}
// (cell, id) entries, bucket histogram
__global__ void k_grid_fill(const Box* __restrict__ box, std::int32_t n, double h, const std::int64_t* __restrict__ off,
                            Entry* __restrict__ ent, std::uint32_t mask, std::int32_t* __restrict__ bcnt) {
    for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        const Cell lo = cell_of(box[i].lo, h), hi = cell_of(box[i].hi, h);
        std::int64_t o = off[i];
        for (int x = lo.x; x <= hi.x; ++x)
            for (int y = lo.y; y <= hi.y; ++y)
                for (int z = lo.z; z <= hi.z; ++z) {
                    ent[o++] = {x, y, z, static_cast<int>(i)};
                    atomicAdd(bcnt + bucket_of(x, y, z, mask), 1);
                }
    }
}
__global__ void k_grid_scatter(const Entry* __restrict__ ent, std::int64_t m, std::uint32_t mask,
                               const std::int64_t* __restrict__ bstart, std::int32_t* __restrict__ bcur,
                               Entry* __restrict__ table) {
    for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < m;
         i += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        const Entry e = ent[i];
        const std::uint32_t b = bucket_of(e.x, e.y, e.z, mask);
        table[bstart[b] + atomicAdd(bcur + b, 1)] = e;
    }
}

struct Grid {
    const Entry* table;
    const std::int64_t* bstart;
    std::uint32_t mask;
    double h;
};

// kind 0: surface vertex vi against triangles; kind 1: edge i against edges j > i.
// count (out == null) or write the accepted partners of query q at out + off[q]
template <int kKind>
__global__ void k_query(Surface s, Grid g, const Box* __restrict__ part_box, const Box* __restrict__ self_box,
                        std::int32_t n_query, const std::int64_t* __restrict__ off, std::int32_t* __restrict__ cnt,
                        int* __restrict__ out) {
    for (std::int64_t q = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; q < n_query;
         q += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        Box b;
        int n0 = -1, e0 = -1, e1 = -1;
        if (kKind == 0) {
            n0 = s.verts[q];
            b = empty_box();
            grow_node(b, s.pos, s.disp, n0);
            inflate(b, s.half);
        } else {
            b = self_box[q];
            e0 = s.edges[2 * q];
            e1 = s.edges[2 * q + 1];
        }
        const Cell lo = cell_of(b.lo, g.h), hi = cell_of(b.hi, g.h);
        std::int32_t found = 0;
        const std::int64_t o = out ? off[q] : 0;
        for (int x = lo.x; x <= hi.x; ++x)
            for (int y = lo.y; y <= hi.y; ++y)
                for (int z = lo.z; z <= hi.z; ++z) {
                    const std::uint32_t bk = bucket_of(x, y, z, g.mask);
                    for (std::int64_t k = g.bstart[bk]; k < g.bstart[bk + 1]; ++k) {
                        const Entry e = g.table[k];
                        if (e.x != x || e.y != y || e.z != z) continue;
                        const int p = e.id;
                        if (kKind == 0) {
                            const int* t = s.tris + 3 * static_cast<std::int64_t>(p);
                            if (t[0] == n0 || t[1] == n0 || t[2] == n0) continue;
                        } else {
                            if (p <= q) continue;
                            const int* f = s.edges + 2 * static_cast<std::int64_t>(p);
                            if (e0 == f[0] || e0 == f[1] || e1 == f[0] || e1 == f[1]) continue;
                        }
                        const Box& pb = part_box[p];
                        if (!overlaps(b, pb)) continue;
                        // once per pair: the first cell both ranges share
                        const Cell plo = cell_of(pb.lo, g.h);
                        if (x != max(lo.x, plo.x) || y != max(lo.y, plo.y) || z != max(lo.z, plo.z)) continue;
                        if (out) out[o + found] = p;
                        ++found;
                    }
                }
        if (!out) {
            cnt[q] = found;
        } else {  // partners ascending (insertion sort: short lists)
            for (int i = 1; i < found; ++i) {
                const int v = out[o + i];
                int j = i - 1;
                for (; j >= 0 && out[o + j] > v; --j) out[o + j + 1] = out[o + j];
                out[o + j + 1] = v;
            }
        }
    }
}

// (query, partner) pairs and their node stencils
__global__ void k_pairs(Surface s, int kind, std::int32_t n_query, const std::int64_t* __restrict__ off,
                        const int* __restrict__ partner, int* __restrict__ pairs, int* __restrict__ stencils) {
    for (std::int64_t q = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; q < n_query;
         q += static_cast<std::int64_t>(gridDim.x) * blockDim.x)
        for (std::int64_t k = off[q]; k < off[q + 1]; ++k) {
            const int p = partner[k];
            pairs[2 * k] = static_cast<int>(q);
            pairs[2 * k + 1] = p;
            int* st = stencils + 4 * k;
            if (kind == 0) {
                st[0] = s.verts[q];
                st[1] = s.tris[3 * static_cast<std::int64_t>(p)];
                st[2] = s.tris[3 * static_cast<std::int64_t>(p) + 1];
                st[3] = s.tris[3 * static_cast<std::int64_t>(p) + 2];
            } else {
                st[0] = s.edges[2 * q];
                st[1] = s.edges[2 * q + 1];
                st[2] = s.edges[2 * static_cast<std::int64_t>(p)];
                st[3] = s.edges[2 * static_cast<std::int64_t>(p) + 1];
            }
        }
}

}  // namespace

void broad_phase(Ctx& c, const BroadDesc& d, std::int64_t* n_pt, std::int64_t* n_ee) {
    cudaStream_t st = c.stream;
    BroadState& B = c.bp;
    Surface s{d.pos, d.disp, d.n_verts, d.n_edges, d.n_tris, d.verts, d.edges, d.tris, d.inflate / 2};
    *n_pt = *n_ee = 0;
    B.n_pt = B.n_ee = 0;
    if (d.n_tris == 0 && d.n_edges == 0) return;
    B.tri_box.reserve(static_cast<std::size_t>(std::max(d.n_tris, 1)));
    B.edge_box.reserve(static_cast<std::size_t>(std::max(d.n_edges, 1)));
    B.scal.reserve(1);
    ADIPC_CUDA(cudaMemsetAsync(B.scal.p, 0, sizeof(double), st));
    k_boxes<<<grid_for(static_cast<std::int64_t>(d.n_tris) + d.n_edges, 256, 16), 256, 0, st>>>(
        s, B.tri_box.p, B.edge_box.p, B.scal.p);
    ADIPC_LAUNCH_CHECK();
    double ext = 0;
    ADIPC_CUDA(cudaMemcpyAsync(&ext, B.scal.p, sizeof(double), cudaMemcpyDeviceToHost, st));
    ADIPC_CUDA(cudaStreamSynchronize(st));
    // broad_phase.hpp:178-179 (the set does not depend on the cell size)
    const double mean = d.n_tris == 0 ? d.inflate : ext / d.n_tris;
    const double h = std::max(mean + d.inflate, 1e-12);

    auto build_grid = [&](const Box* box, std::int32_t n, DBuf<Entry>& table, DBuf<std::int64_t>& bstart) -> Grid {
        B.cnt.reserve(static_cast<std::size_t>(std::max(n, 1)));
        B.off.reserve(static_cast<std::size_t>(n) + 1);
        if (n > 0) {
            k_grid_count<<<grid_for(n, 256, 16), 256, 0, st>>>(box, n, h, B.cnt.p);
            ADIPC_LAUNCH_CHECK();
        }
        exclusive_scan(B.cnt.p, n, B.off.p, c.scan_scratch, st);
        std::int64_t m = 0;
        ADIPC_CUDA(cudaMemcpyAsync(&m, B.off.p + n, sizeof(m), cudaMemcpyDeviceToHost, st));
        ADIPC_CUDA(cudaStreamSynchronize(st));
        std::uint32_t nb = 1024;
        while (nb < 2 * m && nb < (1u << 30)) nb <<= 1;
        B.entries.reserve(static_cast<std::size_t>(std::max<std::int64_t>(m, 1)));
        table.reserve(static_cast<std::size_t>(std::max<std::int64_t>(m, 1)));
        B.bcnt.reserve(nb + 1);
        bstart.reserve(static_cast<std::size_t>(nb) + 1);
        ADIPC_CUDA(cudaMemsetAsync(B.bcnt.p, 0, sizeof(std::int32_t) * (nb + 1), st));
        if (n > 0) {
            k_grid_fill<<<grid_for(n, 256, 16), 256, 0, st>>>(box, n, h, B.off.p, B.entries.p, nb - 1, B.bcnt.p);
            ADIPC_LAUNCH_CHECK();
        }
        exclusive_scan(B.bcnt.p, nb, bstart.p, c.scan_scratch, st);
        ADIPC_CUDA(cudaMemsetAsync(B.bcnt.p, 0, sizeof(std::int32_t) * (nb + 1), st));
        if (m > 0) {
            k_grid_scatter<<<grid_for(m, 256, 16), 256, 0, st>>>(B.entries.p, m, nb - 1, bstart.p, B.bcnt.p, table.p);
            ADIPC_LAUNCH_CHECK();
        }
        return Grid{table.p, bstart.p, nb - 1, h};
    };

    auto run = [&](auto kern, const Grid& g, const Box* part, const Box* self, std::int32_t nq, int kind,
                   DBuf<int>& partner, DBuf<int>& pairs, DBuf<int>& stencils) -> std::int64_t {
        B.qcnt.reserve(static_cast<std::size_t>(std::max(nq, 1)));
        B.qoff.reserve(static_cast<std::size_t>(nq) + 1);
        if (nq > 0) {
            kern<<<grid_for(nq, 128, 16), 128, 0, st>>>(s, g, part, self, nq, nullptr, B.qcnt.p, nullptr);
            ADIPC_LAUNCH_CHECK();
        }
        exclusive_scan(B.qcnt.p, nq, B.qoff.p, c.scan_scratch, st);
        std::int64_t total = 0;
        ADIPC_CUDA(cudaMemcpyAsync(&total, B.qoff.p + nq, sizeof(total), cudaMemcpyDeviceToHost, st));
        ADIPC_CUDA(cudaStreamSynchronize(st));
        partner.reserve(static_cast<std::size_t>(std::max<std::int64_t>(total, 1)));
        pairs.reserve(static_cast<std::size_t>(std::max<std::int64_t>(2 * total, 1)));
        stencils.reserve(static_cast<std::size_t>(std::max<std::int64_t>(4 * total, 1)));
        if (total > 0) {
            kern<<<grid_for(nq, 128, 16), 128, 0, st>>>(s, g, part, self, nq, B.qoff.p, nullptr, partner.p);
            ADIPC_LAUNCH_CHECK();
            k_pairs<<<grid_for(nq, 128, 16), 128, 0, st>>>(s, kind, nq, B.qoff.p, partner.p, pairs.p, stencils.p);
            ADIPC_LAUNCH_CHECK();
        }
        return total;
    };

    if (d.n_tris > 0 && d.n_verts > 0) {
        const Grid g = build_grid(B.tri_box.p, d.n_tris, B.tri_table, B.tri_bstart);
        B.n_pt = run(k_query<0>, g, B.tri_box.p, nullptr, d.n_verts, 0, B.pt_partner, B.pt_pairs, B.pt_stencils);
    }
    if (d.n_edges > 0) {
        const Grid g = build_grid(B.edge_box.p, d.n_edges, B.edge_table, B.edge_bstart);
        B.n_ee = run(k_query<1>, g, B.edge_box.p, B.edge_box.p, d.n_edges, 1, B.ee_partner, B.ee_pairs, B.ee_stencils);
    }
    *n_pt = B.n_pt;
    *n_ee = B.n_ee;
}

}  // namespace adipc_gpu
