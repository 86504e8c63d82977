// Host-side (C++) partition and aggregation-hierarchy construction of the MAS
// preconditioner: integer-exact re-implementations of
//   precond/partition.hpp:12-159  (subdomain_count, chunk_partition,
//                                  partition_block_graph)
//   precond/hierarchy.hpp:30-100  (build_hierarchy)
// over CSR adjacency instead of vector<vector>. These are sequential greedy
// algorithms on graphs that are small after level 0, so they stay on the host;
// their outputs (part_of / agg per level) feed the device restriction and
// inversion kernels in mas.cu.
#pragma once

#include <cstdint>
#include <utility>
#include <vector>

namespace adipc_gpu::host {

using Index = std::int32_t;
constexpr Index kInvalid = -1;

struct Partition {
    std::vector<Index> part_of;
    Index n_parts = 0;
    Index capacity = 0;
};

struct Level {
    Index n_nodes = 0;
    Index n_parts = 0;
    std::vector<Index> part_of;  // node -> subdomain
    std::vector<Index> agg;      // slot -> node
    std::vector<Index> up;       // node -> the next level's node (levels >= 1 with a next level)
};

struct MasHierarchy {
    Index capacity = 0;
    Index n_slots = 0;
    std::vector<Level> levels;
    int n_levels() const { return static_cast<int>(levels.size()); }
};

// Undirected simple graph in CSR form: neighbours sorted ascending, unique,
// self loops dropped (partition.hpp:37-50 semantics).
struct Graph {
    std::vector<std::int64_t> ptr;
    std::vector<Index> adj;
    Index n() const { return static_cast<Index>(ptr.size()) - 1; }
};

Index subdomain_count(Index v, Index n, Index n_o);
Partition chunk_partition(Index v, Index capacity);
Graph build_graph(Index v, const Index* pairs, std::size_t n_edges);  // pairs: (a,b) interleaved
Partition partition_block_graph(Index v, const Graph& g, Index capacity);
Partition partition_block_graph(Index v, const Index* pairs, std::size_t n_edges, Index capacity);
MasHierarchy build_hierarchy(const Partition& l0, const Index* pairs, std::size_t n_edges, int max_levels);
// same, with the level-0 graph already built (the device build, mas.cu level0_graph)
MasHierarchy build_hierarchy(const Partition& l0, Graph g0, int max_levels);
// same, with the first aggregation pass done elsewhere (the device, mas.cu): up1 = level-0 node ->
// level-1 node (n1 nodes) and g1 = the level-1 node graph
MasHierarchy build_hierarchy_l1(const Partition& l0, std::vector<Index> up1, Index n1, Graph g1, int max_levels);
// the pieces for a loop driven elsewhere (the device aggregation passes,
// mas.cu): the level-0 base, and one more level from the current last
// level's node map `up` (node -> next node, n_next nodes) and the next
// level's graph, partitioned here (partition.hpp:88-159; hierarchy.hpp:86-99)
MasHierarchy hierarchy_base(const Partition& l0);
void append_level(MasHierarchy& h, std::vector<Index> up, Index n_next, const Graph& g_next);
// the rest of the aggregation loop on the host from the last level, whose graph is g
void extend_from(MasHierarchy& h, Graph g, int max_levels);

}  // namespace adipc_gpu::host
