// See host_precond.hpp. Integer-exact with the reference; the parity tests
// compare every output array against the oracle restatement.
#include "host_precond.hpp"

#include <chrono>
#include <cstdio>
#include <cstdlib>

#include <algorithm>
#include <cstring>

#include <omp.h>

namespace adipc_gpu::host {

Index subdomain_count(Index v, Index n, Index n_o) {  // partition.hpp:12-15
    const Index eff = n - n_o;
    return (v + eff - 1) / eff;
}

Partition chunk_partition(Index v, Index capacity) {  // partition.hpp:25-32
    Partition p;
    p.capacity = capacity;
    p.part_of.resize(v);
    for (Index i = 0; i < v; ++i) p.part_of[i] = i / capacity;
    p.n_parts = v == 0 ? 0 : (v - 1) / capacity + 1;
    return p;
}

namespace {

// Adjacency lists of the undirected graph over v nodes whose edges are
// edge(e, a, b) for e < n_edges (false = no edge, e.g. a diagonal block):
// every list sorted ascending and duplicate-free, which is the
// std::set-per-node result of partition.hpp:37-50 independent of the edge
// order, so counting and scattering run in parallel (relaxed atomics) and
// each list is sorted after the scatter.
template <class Edge>
Graph build_graph_impl(Index v, std::int64_t n_edges, Edge edge) {
    Graph g;
    std::vector<std::int64_t> deg(static_cast<std::size_t>(v) + 1, 0);
#pragma omp parallel for schedule(static, 65536)
    for (std::int64_t e = 0; e < n_edges; ++e) {
        Index a, b;
        if (!edge(e, a, b) || a == b) continue;
        __atomic_fetch_add(&deg[a + 1], 1, __ATOMIC_RELAXED);
        __atomic_fetch_add(&deg[b + 1], 1, __ATOMIC_RELAXED);
    }
    for (Index i = 0; i < v; ++i) deg[i + 1] += deg[i];
    std::vector<Index> adj(static_cast<std::size_t>(deg[v]));
    std::vector<std::int64_t> cur(deg.begin(), deg.end() - 1);
#pragma omp parallel for schedule(static, 65536)
    for (std::int64_t e = 0; e < n_edges; ++e) {
        Index a, b;
        if (!edge(e, a, b) || a == b) continue;
        adj[__atomic_fetch_add(&cur[a], 1, __ATOMIC_RELAXED)] = b;
        adj[__atomic_fetch_add(&cur[b], 1, __ATOMIC_RELAXED)] = a;
    }
    // sort + unique each list, then compact into the final arrays
    std::vector<std::int64_t> ulen(static_cast<std::size_t>(v) + 1, 0);
#pragma omp parallel for schedule(static, 4096)
    for (Index i = 0; i < v; ++i) {
        Index* beg = adj.data() + deg[i];
        Index* end = adj.data() + deg[i + 1];
        std::sort(beg, end);
        ulen[i + 1] = std::unique(beg, end) - beg;
    }
    for (Index i = 0; i < v; ++i) ulen[i + 1] += ulen[i];
    if (ulen[v] == deg[v]) {  // already duplicate-free (e.g. a symmetric matrix's pattern)
        g.ptr = std::move(deg);
        g.adj = std::move(adj);
        return g;
    }
    g.ptr = std::move(ulen);
    g.adj.resize(static_cast<std::size_t>(g.ptr[v]));
#pragma omp parallel for schedule(static, 4096)
    for (Index i = 0; i < v; ++i)
        std::memcpy(g.adj.data() + g.ptr[i], adj.data() + deg[i], sizeof(Index) * (g.ptr[i + 1] - g.ptr[i]));
    return g;
}

}  // namespace

Graph build_graph(Index v, const Index* pairs, std::size_t n_edges) {  // partition.hpp:37-50
    return build_graph_impl(v, static_cast<std::int64_t>(n_edges), [pairs](std::int64_t e, Index& a, Index& b) {
        a = pairs[2 * e];
        b = pairs[2 * e + 1];
        return true;
    });
}

// partition.hpp:54-77 BFS components + partition.hpp:88-159 packing/carving.
Partition partition_block_graph(Index v, const Graph& g, Index capacity) {
    Partition p;
    p.capacity = capacity;
    p.part_of.assign(v, 0);
    // components in discovery order, flattened
    std::vector<Index> order;
    order.reserve(v);
    std::vector<std::int64_t> comp_ptr;
    comp_ptr.reserve(64);
    {
        std::vector<char> seen(v, 0);
        for (Index start = 0; start < v; ++start) {
            if (seen[start]) continue;
            comp_ptr.push_back(static_cast<std::int64_t>(order.size()));
            seen[start] = 1;
            std::size_t head = order.size();
            order.push_back(start);
            for (; head < order.size(); ++head) {
                const Index cur = order[head];
                for (std::int64_t k = g.ptr[cur]; k < g.ptr[cur + 1]; ++k) {
                    const Index nb = g.adj[k];
                    if (!seen[nb]) {
                        seen[nb] = 1;
                        order.push_back(nb);
                    }
                }
            }
        }
        comp_ptr.push_back(static_cast<std::int64_t>(order.size()));
    }
    // the carving frontier as a bucket queue with lazy deletion: a
    // candidate whose connection count into the open cluster rises to k is
    // appended to bucket k and its older entries go stale (valid iff the
    // node's conn still equals the bucket index); the pick — most
    // connections, ties to the lowest id — compacts the top bucket while it
    // takes the minimum. conn: -1 = assigned, 0 = not a candidate.
    std::vector<Index> conn(v, 0);
    std::vector<std::vector<Index>> bucket(1);
    int top = 0;
    Index next_part = 0, open_part = kInvalid, open_fill = 0;
    const std::size_t n_comps = comp_ptr.size() - 1;
    for (std::size_t ci = 0; ci < n_comps; ++ci) {
        const Index* comp = order.data() + comp_ptr[ci];
        const Index size = static_cast<Index>(comp_ptr[ci + 1] - comp_ptr[ci]);
        if (size <= capacity) {  // next fit (partition.hpp:105-112)
            if (open_part == kInvalid || open_fill + size > capacity) {
                open_part = next_part++;
                open_fill = 0;
            }
            for (Index k = 0; k < size; ++k) p.part_of[comp[k]] = open_part;
            open_fill += size;
            continue;
        }
        const Index chunks = subdomain_count(size, capacity, 0);
        const Index base = size / chunks, extra = size % chunks;
        Index seed_at = 0, chunk = 0, left = size;
        while (left > 0) {
            const Index target = chunk < chunks ? base + (chunk < extra ? 1 : 0) : capacity;
            ++chunk;
            while (conn[comp[seed_at]] < 0) ++seed_at;
            Index pick = comp[seed_at];
            const Index part = next_part++;
            for (Index fill = 0; pick != kInvalid;) {
                p.part_of[pick] = part;
                conn[pick] = -1;
                ++fill;
                --left;
                if (fill == target || left == 0) break;
                const Index* nb_end = g.adj.data() + g.ptr[pick + 1];
                for (const Index* it = g.adj.data() + g.ptr[pick]; it != nb_end; ++it) {
                    const Index nb = *it;
                    if (conn[nb] < 0) continue;
                    const Index c = ++conn[nb];
                    if (c >= static_cast<Index>(bucket.size())) bucket.resize(static_cast<std::size_t>(c) + 1);
                    bucket[c].push_back(nb);
                    if (c > top) top = c;
                }
                pick = kInvalid;
                for (; top > 0; --top) {
                    std::vector<Index>& bk = bucket[top];
                    std::size_t w = 0;
                    for (std::size_t k = 0; k < bk.size(); ++k) {
                        const Index x = bk[k];
                        if (conn[x] != top) continue;
                        bk[w++] = x;
                        pick = (pick == kInvalid || x < pick) ? x : pick;
                    }
                    bk.resize(w);
                    if (w) break;
                }
                if (pick == kInvalid) break;
                conn[pick] = 0;  // its entry goes stale
            }
            for (int k = 1; k <= top; ++k) {
                for (Index x : bucket[k])
                    if (conn[x] > 0) conn[x] = 0;
                bucket[k].clear();
            }
            top = 0;
        }
    }
    p.n_parts = next_part;
    return p;
}

Partition partition_block_graph(Index v, const Index* pairs, std::size_t n_edges, Index capacity) {
    const auto t0 = std::chrono::steady_clock::now();
    Graph g = build_graph(v, pairs, n_edges);
    const auto t1 = std::chrono::steady_clock::now();
    Partition p = partition_block_graph(v, g, capacity);
    if (std::getenv("ADIPC_DEBUG_HIER"))
        std::fprintf(stderr, "  partition v=%d e=%zu: graph %.1f ms, carve %.1f ms\n", v, n_edges,
                     std::chrono::duration<double, std::milli>(t1 - t0).count(),
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t1).count());
    return p;
}

// hierarchy.hpp:30-100
MasHierarchy build_hierarchy(const Partition& l0, const Index* pairs, std::size_t n_edges, int max_levels) {
    return build_hierarchy(l0, build_graph(static_cast<Index>(l0.part_of.size()), pairs, n_edges), max_levels);
}

namespace {

MasHierarchy base_hierarchy(const Partition& l0) {
    MasHierarchy h;
    h.capacity = l0.capacity;
    h.n_slots = static_cast<Index>(l0.part_of.size());
    Level base;
    base.n_nodes = h.n_slots;
    base.n_parts = l0.n_parts;
    base.part_of = l0.part_of;
    base.agg.resize(h.n_slots);
    for (Index i = 0; i < h.n_slots; ++i) base.agg[i] = i;
    h.levels.push_back(std::move(base));
    return h;
}

// the aggregation loop of hierarchy.hpp:46-99 from the current last level,
// whose node graph is g
void extend_hierarchy(MasHierarchy& h, Graph g, int max_levels);

}  // namespace

MasHierarchy hierarchy_base(const Partition& l0) { return base_hierarchy(l0); }

void extend_from(MasHierarchy& h, Graph g, int max_levels) { extend_hierarchy(h, std::move(g), max_levels); }

void append_level(MasHierarchy& h, std::vector<Index> up, Index n_next, const Graph& g_next) {
    Level next;
    next.n_nodes = n_next;
    Partition grouped = partition_block_graph(n_next, g_next, h.capacity);
    next.n_parts = grouped.n_parts;
    next.part_of = std::move(grouped.part_of);
    if (h.n_levels() == 1) {
        next.agg = std::move(up);  // level 0's agg is the identity
    } else {
        Level& cur = h.levels.back();
        next.agg.resize(h.n_slots);
#pragma omp parallel for schedule(static)
        for (Index slot = 0; slot < h.n_slots; ++slot) next.agg[slot] = up[cur.agg[slot]];
        cur.up = std::move(up);
    }
    h.levels.push_back(std::move(next));
}

MasHierarchy build_hierarchy(const Partition& l0, Graph g0, int max_levels) {
    MasHierarchy h = base_hierarchy(l0);
    extend_hierarchy(h, std::move(g0), max_levels);
    return h;
}

MasHierarchy build_hierarchy_l1(const Partition& l0, std::vector<Index> up1, Index n1, Graph g1, int max_levels) {
    const auto t0 = std::chrono::steady_clock::now();
    MasHierarchy h = base_hierarchy(l0);
    const auto t1 = std::chrono::steady_clock::now();
    // the first pass of the loop (hierarchy.hpp:46-99) with its super nodes
    // and their graph given
    if (h.n_levels() >= max_levels || l0.n_parts <= 1 || n1 == h.n_slots) return h;
    Level next;
    next.n_nodes = n1;
    Partition grouped = partition_block_graph(n1, g1, h.capacity);
    const auto t2 = std::chrono::steady_clock::now();
    next.n_parts = grouped.n_parts;
    next.part_of = std::move(grouped.part_of);
    next.agg = std::move(up1);  // level 0's agg is the identity
    h.levels.push_back(std::move(next));
    const long long e1 = static_cast<long long>(g1.adj.size());
    extend_hierarchy(h, std::move(g1), max_levels);
    if (std::getenv("ADIPC_DEBUG_HIER")) {
        auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
        std::fprintf(stderr, "hierarchy from level 1: base %.1f ms, level-1 partition (v=%d, e=%lld) %.1f ms, "
                             "levels >= 2 %.1f ms\n", ms(t0, t1), n1, e1, ms(t1, t2),
                     ms(t2, std::chrono::steady_clock::now()));
    }
    return h;
}

namespace {

void extend_hierarchy(MasHierarchy& h, Graph g, int max_levels) {
    std::vector<Index> up, queue, members, mem_ptr;
    while (h.n_levels() < max_levels) {
        const Level& cur = h.levels.back();
        if (cur.n_parts <= 1) break;
        const bool dbg = std::getenv("ADIPC_DEBUG_HIER") != nullptr;
        auto tnow = [] { return std::chrono::steady_clock::now(); };
        auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
        const auto t1 = tnow();
        // members of each subdomain in ascending node order (counting sort)
        mem_ptr.assign(static_cast<std::size_t>(cur.n_parts) + 1, 0);
        for (Index i = 0; i < cur.n_nodes; ++i) ++mem_ptr[cur.part_of[i] + 1];
        for (Index s = 0; s < cur.n_parts; ++s) mem_ptr[s + 1] += mem_ptr[s];
        members.resize(cur.n_nodes);
        {
            std::vector<Index> fill(mem_ptr.begin(), mem_ptr.end() - 1);
            for (Index i = 0; i < cur.n_nodes; ++i) members[fill[cur.part_of[i]]++] = i;
        }
        // connected components inside each subdomain (hierarchy.hpp:53-72:
        // seeds in ascending node order, neighbours in adjacency order),
        // subdomains in parallel with local ids, then offset by a scan over
        // the subdomains so the super-node ids are exactly the sequential ones
        up.assign(cur.n_nodes, kInvalid);
        std::vector<Index> ncomp(static_cast<std::size_t>(cur.n_parts) + 1, 0);
#pragma omp parallel
        {
            std::vector<Index> q;
#pragma omp for schedule(dynamic, 256)
            for (Index s = 0; s < cur.n_parts; ++s) {
                Index local = 0;
                for (Index k = mem_ptr[s]; k < mem_ptr[s + 1]; ++k) {
                    const Index seed = members[k];
                    if (up[seed] != kInvalid) continue;
                    const Index super = local++;
                    up[seed] = super;
                    q.assign(1, seed);
                    for (std::size_t head = 0; head < q.size(); ++head) {
                        const Index qq = q[head];
                        for (std::int64_t e = g.ptr[qq]; e < g.ptr[qq + 1]; ++e) {
                            const Index nb = g.adj[e];
                            if (cur.part_of[nb] == s && up[nb] == kInvalid) {
                                up[nb] = super;
                                q.push_back(nb);
                            }
                        }
                    }
                }
                ncomp[s + 1] = local;
            }
        }
        for (Index s = 0; s < cur.n_parts; ++s) ncomp[s + 1] += ncomp[s];
        const Index n_next = ncomp[cur.n_parts];
#pragma omp parallel for schedule(static, 4096)
        for (Index i = 0; i < cur.n_nodes; ++i) up[i] += ncomp[cur.part_of[i]];
        const auto t2 = tnow();
        if (n_next == cur.n_nodes) break;
        // coarse edges (hierarchy.hpp:75-85: mapped, deduplicated, sorted)
        // and the graph partition.hpp:37-50 builds from them, in one step:
        // node U's adjacency list is the sorted set of super nodes V != U
        // adjacent to any member of U. Threads own contiguous U ranges and
        // dedupe with a stamp array; their lists are concatenated in U order.
        std::vector<Index> sptr(static_cast<std::size_t>(n_next) + 1, 0), smem(cur.n_nodes);
        for (Index i = 0; i < cur.n_nodes; ++i) ++sptr[up[i] + 1];
        for (Index u = 0; u < n_next; ++u) sptr[u + 1] += sptr[u];
        {
            std::vector<Index> fill(sptr.begin(), sptr.end() - 1);
            for (Index i = 0; i < cur.n_nodes; ++i) smem[fill[up[i]]++] = i;
        }
        Graph cg;
        cg.ptr.assign(static_cast<std::size_t>(n_next) + 1, 0);
        std::vector<std::vector<Index>> part_adj;
#pragma omp parallel
        {
            const int nt = omp_get_num_threads(), t = omp_get_thread_num();
#pragma omp single
            part_adj.resize(nt);
            const Index u0 = static_cast<Index>(static_cast<std::int64_t>(n_next) * t / nt);
            const Index u1 = static_cast<Index>(static_cast<std::int64_t>(n_next) * (t + 1) / nt);
            std::vector<Index>& out = part_adj[t];
            std::vector<Index> stamp(static_cast<std::size_t>(n_next), kInvalid);
            for (Index u = u0; u < u1; ++u) {
                const std::size_t o = out.size();
                for (Index k = sptr[u]; k < sptr[u + 1]; ++k) {
                    const Index m = smem[k];
                    for (std::int64_t e = g.ptr[m]; e < g.ptr[m + 1]; ++e) {
                        const Index v = up[g.adj[e]];
                        if (v != u && stamp[v] != u) {
                            stamp[v] = u;
                            out.push_back(v);
                        }
                    }
                }
                std::sort(out.begin() + o, out.end());
                cg.ptr[u + 1] = static_cast<std::int64_t>(out.size() - o);
            }
#pragma omp barrier
#pragma omp single
            {
                for (Index u = 0; u < n_next; ++u) cg.ptr[u + 1] += cg.ptr[u];
                cg.adj.resize(static_cast<std::size_t>(cg.ptr[n_next]));
            }
            if (!out.empty()) std::memcpy(cg.adj.data() + cg.ptr[u0], out.data(), sizeof(Index) * out.size());
        }
        const auto t3 = tnow();
        Level next;
        next.n_nodes = n_next;
        Partition grouped = partition_block_graph(n_next, cg, h.capacity);
        next.n_parts = grouped.n_parts;
        next.part_of = std::move(grouped.part_of);
        next.agg.resize(h.n_slots);
        for (Index slot = 0; slot < h.n_slots; ++slot) next.agg[slot] = up[cur.agg[slot]];
        if (h.n_levels() > 1) h.levels.back().up = up;  // coarse node maps (level 0's is agg of level 1)
        h.levels.push_back(std::move(next));
        g = std::move(cg);
        if (dbg)
            std::fprintf(stderr, "hierarchy level %d: bfs %.1f ms, coarse graph %.1f ms, partition %.1f ms\n",
                         h.n_levels() - 1, ms(t1, t2), ms(t2, t3), ms(t3, tnow()));
    }
}

}  // namespace

}  // namespace adipc_gpu::host
