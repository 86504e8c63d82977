// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// CPU restatement of the reference `adipc` hot path (StiffGIPC, arXiv
// 2411.06224): Hessian assembly (sort + hash/segment reduction + two-level
// affine-body reduction), MAS preconditioner construction/apply, block Jacobi
// and PCG. Every function cites the reference file:line it follows; paths are
// relative to /root/reference/proj/include/adipc/.
//
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference leg may load this code, and only as the checker or as the
// timed CPU baseline. The product path (paper_2411_06224_b200/) never links
// or calls it.
//
// Eigen is absent here, so the arithmetic Eigen performs (3x3 products, LLT,
// dots) is restated with plain loops, following Eigen 3.4's evaluation order
// where that order decides bits (fixed-size products, the 3x3 inverse).
// Everything integer (keys, sort order, partitions, hierarchies), the
// deterministic reductions and the two-level tiles are bit-exact with the
// reference's own code compiled in place (oracle/_ref, see ref_capi.cpp and
// tests/test_oracle_vs_reference.py); LLT solves and dots agree to rounding.
// Compiled like the reference: -O2 -fopenmp, no FMA contraction.
#pragma once

#include <algorithm>
#include <array>
#include <limits>
#include <unordered_map>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <stdexcept>
#include <thread>
#include <utility>
#include <vector>

#ifdef _OPENMP
#include <omp.h>

#include "sym_eig.hpp"
#endif

namespace oracle {

using Real = double;  // core/types.hpp:9
using Index = std::int32_t;  // core/types.hpp:10
constexpr Index kInvalid = -1;  // core/types.hpp:31

// Eigen::Matrix3d / Vector3d stand-ins, column-major storage like Eigen
// (Mat3::data()[k] walks columns).
struct Vec3 {
    Real v[3] = {0, 0, 0};
    Real& operator[](int i) { return v[i]; }
    Real operator[](int i) const { return v[i]; }
    Vec3& operator+=(const Vec3& o) {
        for (int i = 0; i < 3; ++i) v[i] += o.v[i];
        return *this;
    }
    bool operator==(const Vec3& o) const {
        return v[0] == o.v[0] && v[1] == o.v[1] && v[2] == o.v[2];
    }
};

struct Mat3 {
    Real m[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};  // column-major
    Real& operator()(int r, int c) { return m[3 * c + r]; }
    Real operator()(int r, int c) const { return m[3 * c + r]; }
    Real* data() { return m; }
    const Real* data() const { return m; }
    static Mat3 identity() {
        Mat3 a;
        a.m[0] = a.m[4] = a.m[8] = 1;
        return a;
    }
    Mat3 transpose() const {
        Mat3 t;
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) t(r, c) = (*this)(c, r);
        return t;
    }
    Mat3& operator+=(const Mat3& o) {
        for (int k = 0; k < 9; ++k) m[k] += o.m[k];
        return *this;
    }
    bool operator==(const Mat3& o) const {
        for (int k = 0; k < 9; ++k)
            if (m[k] != o.m[k]) return false;
        return true;
    }
    // Eigen's lazy fixed-size product: ((a0 b0 + a1 b1) + a2 b2).
    Vec3 operator*(const Vec3& x) const {
        Vec3 y;
        for (int r = 0; r < 3; ++r)
            y[r] = (*this)(r, 0) * x[0] + (*this)(r, 1) * x[1] + (*this)(r, 2) * x[2];
        return y;
    }
    // Mat3::inverse as Eigen 3.4 computes a fixed 3x3 inverse
    // (block_jacobi.hpp:13 -> Eigen/src/LU/InverseImpl.h compute_inverse<3,3>):
    // cyclic cofactors, det by expansion down column 0, times 1/det.
    static Real cofactor(const Mat3& a, int i, int j) {
        const int i1 = (i + 1) % 3, i2 = (i + 2) % 3, j1 = (j + 1) % 3, j2 = (j + 2) % 3;
        return a(i1, j1) * a(i2, j2) - a(i1, j2) * a(i2, j1);
    }
    Mat3 inverse() const {
        const Mat3& a = *this;
        const Real c0 = cofactor(a, 0, 0), c1 = cofactor(a, 1, 0), c2 = cofactor(a, 2, 0);
        const Real det = c0 * a(0, 0) + c1 * a(1, 0) + c2 * a(2, 0);
        const Real invdet = Real(1) / det;
        Mat3 inv;
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) inv(i, j) = cofactor(a, j, i) * invdet;
        return inv;
    }
};

// ---------------------------------------------------------------------------
// core/parallel.hpp:18-70
struct ExecPolicy {
    bool deterministic = false;
    int threads = 0;
    int lane_width = 32;
};

inline int& process_thread_default() {  // parallel.hpp:24-34
    static int n = [] {
        if (const char* env = std::getenv("ADIPC_THREADS")) {
            int v = std::atoi(env);
            if (v > 0) return v;
        }
        unsigned hw = std::thread::hardware_concurrency();
        return hw > 0 ? static_cast<int>(hw) : 1;
    }();
    return n;
}

inline int effective_threads(const ExecPolicy& pol) {  // parallel.hpp:40-43
    if (pol.deterministic) return 1;
    return pol.threads > 0 ? pol.threads : process_thread_default();
}

template <class F>
void parallel_for(std::int64_t n, const ExecPolicy& pol, F&& fn) {  // parallel.hpp:46-58
    const int nt = effective_threads(pol);
    if (nt <= 1 || n < 2) {
        for (std::int64_t i = 0; i < n; ++i) fn(i);
        return;
    }
#ifdef _OPENMP
#pragma omp parallel for schedule(static) num_threads(nt)
    for (std::int64_t i = 0; i < n; ++i) fn(i);
#else
    for (std::int64_t i = 0; i < n; ++i) fn(i);
#endif
}

inline void atomic_add(Real& slot, Real v) {  // parallel.hpp:60-62
    std::atomic_ref<Real>(slot).fetch_add(v, std::memory_order_relaxed);
}
inline void atomic_add(Vec3& slot, const Vec3& v) {
    for (int k = 0; k < 3; ++k) atomic_add(slot.v[k], v.v[k]);
}
inline void atomic_add(Mat3& slot, const Mat3& v) {
    for (int k = 0; k < 9; ++k) atomic_add(slot.m[k], v.m[k]);
}

// ---------------------------------------------------------------------------
// sparse/block_coo.hpp:13-21
inline std::uint64_t make_block_key(std::uint32_t row, std::uint32_t col) {
    return (static_cast<std::uint64_t>(row) << 32) | col;
}
inline std::uint32_t block_key_row(std::uint64_t k) { return static_cast<std::uint32_t>(k >> 32); }
inline std::uint32_t block_key_col(std::uint64_t k) {
    return static_cast<std::uint32_t>(k & 0xFFFFFFFFu);
}

// sparse/block_coo.hpp:25-51
struct BlockTripletStream {
    std::vector<std::uint64_t> keys;
    std::vector<Mat3> values;
    std::size_t size() const { return keys.size(); }
    void emit(Index r, Index c, const Mat3& m) {
        if (r <= c) {
            keys.push_back(make_block_key(r, c));
            values.push_back(m);
        } else {
            keys.push_back(make_block_key(c, r));
            values.push_back(m.transpose());
        }
    }
    void append(const BlockTripletStream& o) {
        keys.insert(keys.end(), o.keys.begin(), o.keys.end());
        values.insert(values.end(), o.values.begin(), o.values.end());
    }
};

// sparse/block_coo.hpp:54-61
struct SortedSymBlockCoo {
    Index n_block_rows = 0;
    std::vector<std::uint32_t> rows, cols;
    std::vector<Mat3> blocks;
    std::size_t size() const { return blocks.size(); }
};

// sparse/block_coo.hpp:67-101 — serial stable LSD radix sort, 4 x 16 bits,
// always four passes (the "skip" comment at :82 is not implemented).
inline void radix_sort_keys(std::vector<std::uint64_t>& keys, std::vector<std::uint32_t>& perm) {
    const std::size_t n = keys.size();
    perm.resize(n);
    for (std::size_t i = 0; i < n; ++i) perm[i] = static_cast<std::uint32_t>(i);
    if (n < 2) return;
    std::vector<std::uint64_t> kbuf(n);
    std::vector<std::uint32_t> pbuf(n);
    constexpr int kBits = 16;
    constexpr std::size_t kBuckets = std::size_t(1) << kBits;
    std::vector<std::size_t> count(kBuckets);
    for (int pass = 0; pass < 4; ++pass) {
        const int shift = pass * kBits;
        std::fill(count.begin(), count.end(), 0);
        for (std::size_t i = 0; i < n; ++i) ++count[(keys[i] >> shift) & (kBuckets - 1)];
        std::size_t sum = 0;
        for (std::size_t b = 0; b < kBuckets; ++b) {
            std::size_t c = count[b];
            count[b] = sum;
            sum += c;
        }
        for (std::size_t i = 0; i < n; ++i) {
            const std::size_t b = (keys[i] >> shift) & (kBuckets - 1);
            kbuf[count[b]] = keys[i];
            pbuf[count[b]] = perm[i];
            ++count[b];
        }
        keys.swap(kbuf);
        perm.swap(pbuf);
    }
}

// sparse/block_coo.hpp:106-113
inline void sort_stream(BlockTripletStream& s, const ExecPolicy& pol) {
    std::vector<std::uint32_t> perm;
    radix_sort_keys(s.keys, perm);
    std::vector<Mat3> sorted(s.values.size());
    parallel_for(static_cast<std::int64_t>(perm.size()), pol,
                 [&](std::int64_t i) { sorted[i] = s.values[perm[i]]; });
    s.values.swap(sorted);
}

// ---------------------------------------------------------------------------
// sparse/reduction.hpp:30-79. V is Real, Vec3 or Mat3 (tests use all three).
inline void zero_value(Real& v) { v = 0; }
inline void zero_value(Vec3& v) { v = Vec3(); }
inline void zero_value(Mat3& v) { v = Mat3(); }

template <class V>
std::vector<V> fast_segment_reduction(const std::vector<Index>& O, const std::vector<V>& values,
                                      Index n_segments, const ExecPolicy& pol) {
    const std::size_t n = values.size();
    if (O.size() != n) throw std::invalid_argument("segment map size mismatch");
    std::vector<V> R(n_segments);
    for (auto& r : R) zero_value(r);
    if (n == 0) return R;
    if (pol.deterministic) {  // reduction.hpp:39-53
        Index seg = O[0];
        V sum = values[0];
        for (std::size_t i = 1; i < n; ++i) {
            if (O[i] == seg) {
                sum += values[i];
            } else {
                R[seg] = sum;
                seg = O[i];
                sum = values[i];
            }
        }
        R[seg] = sum;
        return R;
    }
    const std::size_t w = static_cast<std::size_t>(pol.lane_width);  // reduction.hpp:55-77
    const std::int64_t n_groups = static_cast<std::int64_t>((n + w - 1) / w);
    parallel_for(n_groups, pol, [&](std::int64_t gi) {
        const std::size_t begin = static_cast<std::size_t>(gi) * w;
        const std::size_t end = std::min(begin + w, n);
        std::size_t i = begin;
        while (i < end) {
            const Index seg = O[i];
            V sum = values[i];
            std::size_t j = i + 1;
            while (j < end && O[j] == seg) {
                sum += values[j];
                ++j;
            }
            const bool cl = (i == begin && begin > 0 && O[begin - 1] == seg);
            const bool cr = (j == end && end < n && O[end] == seg);
            if (cl || cr)
                atomic_add(R[seg], sum);
            else
                R[seg] = sum;
            i = j;
        }
    });
    return R;
}

// sparse/reduction.hpp:83-107 (serial O scan + head rows/cols)
inline SortedSymBlockCoo fast_hash_reduction(const BlockTripletStream& sorted, Index n_block_rows,
                                             const ExecPolicy& pol) {
    SortedSymBlockCoo out;
    out.n_block_rows = n_block_rows;
    const std::size_t n = sorted.size();
    if (n == 0) return out;
    std::vector<Index> O(n);
    O[0] = 0;
    for (std::size_t i = 1; i < n; ++i)
        O[i] = O[i - 1] + (sorted.keys[i - 1] != sorted.keys[i] ? 1 : 0);
    const Index n_unique = O[n - 1] + 1;
    out.rows.resize(n_unique);
    out.cols.resize(n_unique);
    for (std::size_t i = 0; i < n; ++i)
        if (i == 0 || O[i] != O[i - 1]) {
            out.rows[O[i]] = block_key_row(sorted.keys[i]);
            out.cols[O[i]] = block_key_col(sorted.keys[i]);
        }
    out.blocks = fast_segment_reduction(O, sorted.values, n_unique, pol);
    return out;
}

// ---------------------------------------------------------------------------
// sparse/srbk_spmv.hpp:13-49
inline std::vector<Vec3> srbk_spmv(const SortedSymBlockCoo& A, const std::vector<Vec3>& x,
                                   const ExecPolicy& pol) {
    std::vector<Vec3> y(x.size());
    const std::size_t n = A.size();
    if (n == 0) return y;
    if (effective_threads(pol) <= 1) {
        for (std::size_t e = 0; e < n; ++e) {
            const Index r = A.rows[e], c = A.cols[e];
            y[r] += A.blocks[e] * x[c];
            if (r != c) y[c] += A.blocks[e].transpose() * x[r];
        }
        return y;
    }
    const std::size_t w = static_cast<std::size_t>(pol.lane_width);
    const std::int64_t n_groups = static_cast<std::int64_t>((n + w - 1) / w);
    parallel_for(n_groups, pol, [&](std::int64_t gi) {
        const std::size_t begin = static_cast<std::size_t>(gi) * w;
        const std::size_t end = std::min(begin + w, n);
        std::size_t i = begin;
        while (i < end) {
            const std::uint32_t row = A.rows[i];
            Vec3 run;
            std::size_t j = i;
            for (; j < end && A.rows[j] == row; ++j) {
                run += A.blocks[j] * x[A.cols[j]];
                if (A.cols[j] != row) atomic_add(y[A.cols[j]], A.blocks[j].transpose() * x[row]);
            }
            atomic_add(y[row], run);
            i = j;
        }
    });
    return y;
}

// ---------------------------------------------------------------------------
// sparse/block_split.hpp:10-33. Large blocks are dense column-major arrays.
struct MatRC {  // small dense column-major matrix (Mat12, Mat12x3, Mat3x12)
    int rows = 0, cols = 0;
    std::vector<Real> a;
    MatRC() = default;
    MatRC(int r, int c) : rows(r), cols(c), a(static_cast<std::size_t>(r) * c, 0.0) {}
    Real& operator()(int r, int c) { return a[static_cast<std::size_t>(c) * rows + r]; }
    Real operator()(int r, int c) const { return a[static_cast<std::size_t>(c) * rows + r]; }
    Mat3 block3(int r0, int c0) const {
        Mat3 b;
        for (int c = 0; c < 3; ++c)
            for (int r = 0; r < 3; ++r) b(r, c) = (*this)(r0 + r, c0 + c);
        return b;
    }
    MatRC transpose() const {
        MatRC t(cols, rows);
        for (int r = 0; r < rows; ++r)
            for (int c = 0; c < cols; ++c) t(c, r) = (*this)(r, c);
        return t;
    }
};

// Eigen's dynamic-free product for small fixed matrices: inner-product order k=0..K-1.
// Eigen product evaluation for the shapes on this path: coefficient-based
// (3x3*3x12, 12x3*3x3) sums from the first term; the 12x3*3x12 product is a
// GEMM (GeneralProduct.h product_type_selector<Large,Large,Small>, 27 >=
// EIGEN_GEMM_TO_COEFFBASED_THRESHOLD) whose accumulators start at zero, so
// its -0.0 entries come out +0.0 (gemm = true). Inner index ascending, no FMA.
inline MatRC matmul(const MatRC& A, const MatRC& B, bool gemm = false) {
    MatRC C(A.rows, B.cols);
    for (int c = 0; c < B.cols; ++c)
        for (int r = 0; r < A.rows; ++r) {
            Real s = A(r, 0) * B(0, c);
            for (int k = 1; k < A.cols; ++k) s += A(r, k) * B(k, c);
            C(r, c) = gemm ? 0.0 + s : s;
        }
    return C;
}

inline MatRC from_mat3(const Mat3& m) {
    MatRC a(3, 3);
    for (int k = 0; k < 9; ++k) a.a[k] = m.m[k];
    return a;
}

inline void split_12x12(Index row_base, Index col_base, const MatRC& H, BlockTripletStream& out) {
    for (int ti = 0; ti < 4; ++ti)
        for (int tj = 0; tj < 4; ++tj) out.emit(row_base + ti, col_base + tj, H.block3(3 * ti, 3 * tj));
}
inline void split_sym_12x12(Index base, const MatRC& H, BlockTripletStream& out) {
    for (int ti = 0; ti < 4; ++ti)
        for (int tj = ti; tj < 4; ++tj) out.emit(base + ti, base + tj, H.block3(3 * ti, 3 * tj));
}
inline void split_12x3(Index row_base, Index col, const MatRC& H, BlockTripletStream& out) {
    for (int t = 0; t < 4; ++t) out.emit(row_base + t, col, H.block3(3 * t, 0));
}
inline void split_3x12(Index row, Index col_base, const MatRC& H, BlockTripletStream& out) {
    for (int t = 0; t < 4; ++t) out.emit(row, col_base + t, H.block3(0, 3 * t));
}

// sparse/abd_reduce.hpp:11-27
struct DofMap {
    Index n_fem_nodes = 0;
    Index n_bodies = 0;
    std::vector<Index> abd_node_body;
    std::vector<MatRC> abd_node_jacobian;  // 3x12 each
    Index n_nodes() const { return n_fem_nodes + static_cast<Index>(abd_node_body.size()); }
    Index n_blocks() const { return n_fem_nodes + 4 * n_bodies; }
    bool is_fem(Index node) const { return node < n_fem_nodes; }
    Index body_of(Index node) const { return abd_node_body[node - n_fem_nodes]; }
    Index body_block_base(Index body) const { return n_fem_nodes + 4 * body; }
    const MatRC& jacobian(Index node) const { return abd_node_jacobian[node - n_fem_nodes]; }
};

// sparse/abd_reduce.hpp:32-74
inline BlockTripletStream two_level_abd_reduce(const BlockTripletStream& node_pairs, const DofMap& map,
                                               const ExecPolicy& pol) {
    BlockTripletStream sorted = node_pairs;
    sort_stream(sorted, pol);
    SortedSymBlockCoo merged = fast_hash_reduction(sorted, map.n_nodes(), pol);
    BlockTripletStream out;
    for (std::size_t e = 0; e < merged.size(); ++e) {
        const Index i = static_cast<Index>(merged.rows[e]);
        const Index j = static_cast<Index>(merged.cols[e]);
        const MatRC C = from_mat3(merged.blocks[e]);
        const bool fi = map.is_fem(i), fj = map.is_fem(j);
        if (fi && fj) {
            out.emit(i, j, merged.blocks[e]);
        } else if (fi && !fj) {
            split_3x12(i, map.body_block_base(map.body_of(j)), matmul(C, map.jacobian(j)), out);
        } else if (!fi && fj) {  // unreachable for canonical keys (abd_reduce.hpp:52-54)
            split_12x3(map.body_block_base(map.body_of(i)), j, matmul(map.jacobian(i).transpose(), C),
                       out);
        } else {
            const Index bi = map.body_of(i), bj = map.body_of(j);
            const MatRC JiT = map.jacobian(i).transpose();
            if (bi != bj) {
                split_12x12(map.body_block_base(bi), map.body_block_base(bj),
                            matmul(matmul(JiT, C), map.jacobian(j), true), out);
            } else if (i == j) {
                split_sym_12x12(map.body_block_base(bi), matmul(matmul(JiT, C), map.jacobian(i), true), out);
            } else {
                const MatRC K = matmul(matmul(JiT, C), map.jacobian(j), true);
                MatRC S(12, 12);
                for (int r = 0; r < 12; ++r)
                    for (int c = 0; c < 12; ++c) S(r, c) = K(r, c) + K(c, r);
                split_sym_12x12(map.body_block_base(bi), S, out);
            }
        }
    }
    return out;
}

// solver/incremental_potential.hpp:410-425
inline void filter_pinned(BlockTripletStream& s, const std::vector<char>& slot_pinned) {
    std::size_t w = 0;
    for (std::size_t i = 0; i < s.size(); ++i) {
        const Index r = block_key_row(s.keys[i]);
        const Index c = block_key_col(s.keys[i]);
        if (slot_pinned[r] || slot_pinned[c]) continue;
        s.keys[w] = s.keys[i];
        s.values[w] = s.values[i];
        ++w;
    }
    s.keys.resize(w);
    s.values.resize(w);
    for (Index slot = 0; slot < static_cast<Index>(slot_pinned.size()); ++slot)
        if (slot_pinned[slot]) s.emit(slot, slot, Mat3::identity());
}

// ---------------------------------------------------------------------------
// precond/partition.hpp:12-32
inline Index subdomain_count(Index v, Index n, Index n_o) {
    const Index eff = n - n_o;
    return (v + eff - 1) / eff;
}

struct Partition {
    std::vector<Index> part_of;
    Index n_parts = 0;
    Index capacity = 0;
};

inline Partition chunk_partition(Index v, Index capacity) {
    Partition p;
    p.capacity = capacity;
    p.part_of.resize(v);
    for (Index i = 0; i < v; ++i) p.part_of[i] = i / capacity;
    p.n_parts = v == 0 ? 0 : (v - 1) / capacity + 1;
    return p;
}

using Edge = std::pair<Index, Index>;

// partition.hpp:37-50
inline std::vector<std::vector<Index>> adjacency_lists(Index v, const std::vector<Edge>& edges) {
    std::vector<std::vector<Index>> adj(v);
    for (const auto& [a, b] : edges) {
        if (a == b) continue;
        adj[a].push_back(b);
        adj[b].push_back(a);
    }
    for (auto& n : adj) {
        std::sort(n.begin(), n.end());
        n.erase(std::unique(n.begin(), n.end()), n.end());
    }
    return adj;
}

// partition.hpp:54-77
inline std::vector<std::vector<Index>> connected_components(const std::vector<std::vector<Index>>& adj) {
    const Index v = static_cast<Index>(adj.size());
    std::vector<std::vector<Index>> comps;
    std::vector<char> seen(v, 0);
    std::vector<Index> queue;
    for (Index start = 0; start < v; ++start) {
        if (seen[start]) continue;
        comps.emplace_back();
        auto& comp = comps.back();
        seen[start] = 1;
        queue.assign(1, start);
        for (std::size_t head = 0; head < queue.size(); ++head) {
            const Index cur = queue[head];
            comp.push_back(cur);
            for (Index nb : adj[cur])
                if (!seen[nb]) {
                    seen[nb] = 1;
                    queue.push_back(nb);
                }
        }
    }
    return comps;
}

// partition.hpp:88-159 — next-fit packing (only the single open part is
// tried, :106-111) + greedy max-connectivity cluster growth.
inline Partition partition_block_graph(Index v, const std::vector<Edge>& edges, Index capacity) {
    Partition p;
    p.capacity = capacity;
    p.part_of.assign(v, 0);
    const auto adj = adjacency_lists(v, edges);
    const auto comps = connected_components(adj);
    std::vector<char> assigned(v, 0);
    std::vector<Index> conn(v, 0);
    std::vector<Index> cand, touched;
    Index next_part = 0;
    Index open_part = kInvalid;
    Index open_fill = 0;
    for (const auto& comp : comps) {
        const Index size = static_cast<Index>(comp.size());
        if (size <= capacity) {
            if (open_part == kInvalid || open_fill + size > capacity) {
                open_part = next_part++;
                open_fill = 0;
            }
            for (Index slot : comp) p.part_of[slot] = open_part;
            open_fill += size;
            continue;
        }
        const Index chunks = subdomain_count(size, capacity, 0);
        const Index base = size / chunks, extra = size % chunks;
        std::size_t seed_at = 0;
        Index chunk = 0, left = size;
        while (left > 0) {
            const Index target = chunk < chunks ? base + (chunk < extra ? 1 : 0) : capacity;
            ++chunk;
            while (assigned[comp[seed_at]]) ++seed_at;
            Index pick = comp[seed_at];
            const Index part = next_part++;
            cand.clear();
            touched.clear();
            for (Index fill = 0; pick != kInvalid;) {
                p.part_of[pick] = part;
                assigned[pick] = 1;
                ++fill;
                --left;
                if (fill == target || left == 0) break;
                for (Index nb : adj[pick])
                    if (!assigned[nb]) {
                        if (conn[nb] == 0) {
                            cand.push_back(nb);
                            touched.push_back(nb);
                        }
                        ++conn[nb];
                    }
                pick = kInvalid;
                Index best = 0;
                for (Index c : cand)
                    if (!assigned[c] && (pick == kInvalid || conn[c] > best || (conn[c] == best && c < pick))) {
                        pick = c;
                        best = conn[c];
                    }
            }
            for (Index t : touched) conn[t] = 0;
        }
    }
    p.n_parts = next_part;
    return p;
}

// ---------------------------------------------------------------------------
// precond/hierarchy.hpp:15-28
struct MasHierarchy {
    Index capacity = 0;
    Index n_slots = 0;
    struct Level {
        Index n_nodes = 0;
        Index n_parts = 0;
        std::vector<Index> part_of;
        std::vector<Index> agg;
    };
    std::vector<Level> levels;
    int n_levels() const { return static_cast<int>(levels.size()); }
};

// hierarchy.hpp:30-100
inline MasHierarchy build_hierarchy(const Partition& l0, const std::vector<Edge>& edges, int max_levels) {
    MasHierarchy h;
    h.capacity = l0.capacity;
    h.n_slots = static_cast<Index>(l0.part_of.size());
    MasHierarchy::Level base;
    base.n_nodes = h.n_slots;
    base.n_parts = l0.n_parts;
    base.part_of = l0.part_of;
    base.agg.resize(h.n_slots);
    for (Index i = 0; i < h.n_slots; ++i) base.agg[i] = i;
    h.levels.push_back(std::move(base));
    std::vector<Edge> cur_edges = edges;
    while (h.n_levels() < max_levels) {
        const MasHierarchy::Level& cur = h.levels.back();
        if (cur.n_parts <= 1) break;
        auto adj = adjacency_lists(cur.n_nodes, cur_edges);
        std::vector<std::vector<Index>> members(cur.n_parts);
        for (Index i = 0; i < cur.n_nodes; ++i) members[cur.part_of[i]].push_back(i);
        std::vector<Index> up(cur.n_nodes, kInvalid);
        Index n_next = 0;
        std::vector<Index> queue;
        for (Index s = 0; s < cur.n_parts; ++s)
            for (Index seed : members[s]) {
                if (up[seed] != kInvalid) continue;
                const Index super = n_next++;
                up[seed] = super;
                queue.assign(1, seed);
                for (std::size_t head = 0; head < queue.size(); ++head)
                    for (Index nb : adj[queue[head]])
                        if (cur.part_of[nb] == s && up[nb] == kInvalid) {
                            up[nb] = super;
                            queue.push_back(nb);
                        }
            }
        if (n_next == cur.n_nodes) break;
        std::vector<Edge> next_edges;
        next_edges.reserve(cur_edges.size());
        for (const auto& [a, b] : cur_edges) {
            Index ua = up[a], ub = up[b];
            if (ua == ub) continue;
            if (ua > ub) std::swap(ua, ub);
            next_edges.emplace_back(ua, ub);
        }
        std::sort(next_edges.begin(), next_edges.end());
        next_edges.erase(std::unique(next_edges.begin(), next_edges.end()), next_edges.end());
        MasHierarchy::Level next;
        next.n_nodes = n_next;
        Partition grouped = partition_block_graph(n_next, next_edges, h.capacity);
        next.n_parts = grouped.n_parts;
        next.part_of = std::move(grouped.part_of);
        next.agg.resize(h.n_slots);
        for (Index slot = 0; slot < h.n_slots; ++slot) next.agg[slot] = up[cur.agg[slot]];
        h.levels.push_back(std::move(next));
        cur_edges = std::move(next_edges);
    }
    return h;
}

// ---------------------------------------------------------------------------
// precond/mas.hpp:19-25
inline std::vector<Edge> block_edges(const SortedSymBlockCoo& A) {
    std::vector<Edge> e;
    e.reserve(A.rows.size());
    for (std::size_t i = 0; i < A.rows.size(); ++i)
        if (A.rows[i] != A.cols[i]) e.emplace_back(A.rows[i], A.cols[i]);
    return e;
}

// Dense column-major square matrix + Eigen::LLT restatement (unblocked,
// lower, right-looking like Eigen's llt_inplace::unblocked: fail iff a pivot
// x <= 0; a NaN pivot does not fail, as in Eigen).
struct DenseLLT {
    int n = 0;
    std::vector<Real> L;  // column-major lower factor
    bool ok = false;
    bool compute(const std::vector<Real>& A, int dim) {
        n = dim;
        L = A;
        auto at = [&](int r, int c) -> Real& { return L[static_cast<std::size_t>(c) * n + r]; };
        for (int k = 0; k < n; ++k) {
            Real x = at(k, k);
            for (int j = 0; j < k; ++j) x -= at(k, j) * at(k, j);
            if (x <= 0) {
                ok = false;
                return false;
            }
            x = std::sqrt(x);
            at(k, k) = x;
            for (int i = k + 1; i < n; ++i) {
                Real s = at(i, k);
                for (int j = 0; j < k; ++j) s -= at(i, j) * at(k, j);
                at(i, k) = s / x;
            }
        }
        for (int c = 0; c < n; ++c)
            for (int r = 0; r < c; ++r) at(r, c) = 0;
        ok = true;
        return true;
    }
    std::vector<Real> solve(const std::vector<Real>& b) const {
        std::vector<Real> y = b;
        auto at = [&](int r, int c) { return L[static_cast<std::size_t>(c) * n + r]; };
        for (int i = 0; i < n; ++i) {
            Real s = y[i];
            for (int j = 0; j < i; ++j) s -= at(i, j) * y[j];
            y[i] = s / at(i, i);
        }
        for (int i = n - 1; i >= 0; --i) {
            Real s = y[i];
            for (int j = i + 1; j < n; ++j) s -= at(j, i) * y[j];
            y[i] = s / at(i, i);
        }
        return y;
    }
};

struct Preconditioner {  // mas.hpp:12-15
    virtual ~Preconditioner() = default;
    virtual void apply(const std::vector<Real>& r, std::vector<Real>& z) const = 0;
};

class MasPreconditioner : public Preconditioner {  // mas.hpp:32-115
public:
    struct LevelData {
        std::vector<Index> agg, part_of, pos_of;
        std::vector<std::vector<std::pair<Index, Index>>> sub_slots;
        std::vector<std::vector<Real>> dense;  // column-major 3f x 3f
        std::vector<int> dim;
        std::vector<DenseLLT> factor;
    };
    std::vector<LevelData> levels_;
    // counts regularisation shifts applied, for parity checks of the retry rule
    long shifts_applied = 0;

    // mas.hpp:34-83
    void build(const SortedSymBlockCoo& A, const MasHierarchy& h) {
        levels_.assign(h.n_levels(), LevelData{});
        shifts_applied = 0;
        const Index n_slots = h.n_slots;
        for (int l = 0; l < h.n_levels(); ++l) {
            const auto& hl = h.levels[l];
            LevelData& ld = levels_[l];
            ld.agg = hl.agg;
            ld.part_of = hl.part_of;
            ld.pos_of.assign(hl.n_nodes, 0);
            std::vector<Index> fill(hl.n_parts, 0);
            for (Index node = 0; node < hl.n_nodes; ++node) ld.pos_of[node] = fill[hl.part_of[node]]++;
            ld.dense.resize(hl.n_parts);
            ld.dim.resize(hl.n_parts);
            for (Index s = 0; s < hl.n_parts; ++s) {
                ld.dim[s] = 3 * fill[s];
                ld.dense[s].assign(static_cast<std::size_t>(ld.dim[s]) * ld.dim[s], 0.0);
            }
            ld.sub_slots.assign(hl.n_parts, {});
            for (Index slot = 0; slot < n_slots; ++slot) {
                const Index node = ld.agg[slot];
                ld.sub_slots[ld.part_of[node]].emplace_back(slot, ld.pos_of[node]);
            }
            for (std::size_t i = 0; i < A.rows.size(); ++i) {  // mas.hpp:56-64
                const Index r = A.rows[i], c = A.cols[i];
                const Index nr = ld.agg[r], nc = ld.agg[c];
                if (ld.part_of[nr] != ld.part_of[nc]) continue;
                const Index s = ld.part_of[nr];
                auto& D = ld.dense[s];
                const int d = ld.dim[s];
                const Index pr = ld.pos_of[nr], pc = ld.pos_of[nc];
                for (int cc = 0; cc < 3; ++cc)
                    for (int rr = 0; rr < 3; ++rr) {
                        D[static_cast<std::size_t>(3 * pc + cc) * d + 3 * pr + rr] += A.blocks[i](rr, cc);
                    }
                if (r != c)
                    for (int cc = 0; cc < 3; ++cc)
                        for (int rr = 0; rr < 3; ++rr)
                            D[static_cast<std::size_t>(3 * pr + cc) * d + 3 * pc + rr] += A.blocks[i](cc, rr);
            }
            ld.factor.resize(hl.n_parts);
            for (Index s = 0; s < hl.n_parts; ++s) {  // mas.hpp:66-81
                std::vector<Real> D = ld.dense[s];
                const int d = ld.dim[s];
                Real tr = 0;
                for (int k = 0; k < d; ++k) tr += D[static_cast<std::size_t>(k) * d + k];
                Real eps = 1e-8 * tr / d;
                if (!(eps > 0)) eps = 1e-12;
                for (int attempt = 0;; ++attempt) {
                    if (ld.factor[s].compute(D, d)) break;
                    if (attempt >= 3)
                        throw std::runtime_error("subdomain matrix stayed indefinite after regularization");
                    for (int k = 0; k < d; ++k) D[static_cast<std::size_t>(k) * d + k] += eps;
                    eps *= 100;
                    ++shifts_applied;
                }
            }
        }
    }

    // mas.hpp:85-99
    void apply(const std::vector<Real>& r, std::vector<Real>& z) const override {
        z.assign(r.size(), 0.0);
        ExecPolicy pol;
        for (const LevelData& ld : levels_) {
            parallel_for(static_cast<Index>(ld.sub_slots.size()), pol, [&](std::int64_t s) {
                const auto& slots = ld.sub_slots[s];
                std::vector<Real> b(ld.dim[s], 0.0);
                for (const auto& [slot, pos] : slots)
                    for (int k = 0; k < 3; ++k) b[3 * pos + k] += r[3 * slot + k];
                const std::vector<Real> y = ld.factor[s].solve(b);
                for (const auto& [slot, pos] : slots)
                    for (int k = 0; k < 3; ++k) z[3 * slot + k] += y[3 * pos + k];
            });
        }
    }
};

// precond/block_jacobi.hpp:8-26
class BlockJacobiPreconditioner : public Preconditioner {
public:
    std::vector<Mat3> inv_;
    void build(const SortedSymBlockCoo& A) {
        inv_.assign(A.n_block_rows, Mat3::identity());
        for (std::size_t i = 0; i < A.rows.size(); ++i)
            if (A.rows[i] == A.cols[i]) inv_[A.rows[i]] = A.blocks[i].inverse();
    }
    void apply(const std::vector<Real>& r, std::vector<Real>& z) const override {
        z.resize(r.size());
        ExecPolicy pol;
        parallel_for(static_cast<Index>(inv_.size()), pol, [&](std::int64_t i) {
            Vec3 ri;
            for (int k = 0; k < 3; ++k) ri[k] = r[3 * i + k];
            const Vec3 zi = inv_[i] * ri;
            for (int k = 0; k < 3; ++k) z[3 * i + k] = zi[k];
        });
    }
};

// ---------------------------------------------------------------------------
// solver/pcg.hpp:10-88. Dot products and axpys are single-threaded loops
// (Eigen VecX ops in the reference run on one thread).
struct PcgResult {
    int iters = 0;
    Real rel_residual = 0;
    bool converged = false;
};

inline Real dot(const std::vector<Real>& a, const std::vector<Real>& b) {
    Real s = 0;
    for (std::size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
    return s;
}

inline PcgResult pcg_solve(const SortedSymBlockCoo& A, const std::vector<Real>& b, const Preconditioner& M,
                           Real rel_tol, int restart, int max_iters, const ExecPolicy& pol,
                           std::vector<Real>& x) {
    PcgResult out;
    const std::size_t n = b.size();
    x.assign(n, 0.0);
    if (dot(b, b) == 0) {
        out.converged = true;
        return out;
    }
    std::vector<Vec3> sin, sout;
    auto apply_a = [&](const std::vector<Real>& v, std::vector<Real>& av) {  // pcg.hpp:45-49
        sin.resize(n / 3);
        for (std::size_t i = 0; i < sin.size(); ++i)
            for (int k = 0; k < 3; ++k) sin[i][k] = v[3 * i + k];
        sout = srbk_spmv(A, sin, pol);
        av.resize(3 * sout.size());
        for (std::size_t i = 0; i < sout.size(); ++i)
            for (int k = 0; k < 3; ++k) av[3 * i + k] = sout[i][k];
    };
    std::vector<Real> r = b, z, p, ap;
    M.apply(r, z);
    p = z;
    Real rho = dot(r, z);
    const Real rho0 = rho;
    if (!(rho0 > 0)) return out;
    const Real stop = rel_tol * rel_tol * rho0;
    for (int k = 1; k <= max_iters; ++k) {
        apply_a(p, ap);
        const Real p_ap = dot(p, ap);
        if (!(p_ap > 0)) {
            out.iters = k - 1;
            out.rel_residual = std::sqrt(std::abs(rho) / rho0);
            return out;
        }
        const Real alpha = rho / p_ap;
        for (std::size_t i = 0; i < n; ++i) x[i] += alpha * p[i];
        if (restart > 0 && k % restart == 0) {
            apply_a(x, ap);
            for (std::size_t i = 0; i < n; ++i) r[i] = b[i] - ap[i];
        } else {
            for (std::size_t i = 0; i < n; ++i) r[i] -= alpha * ap[i];
        }
        M.apply(r, z);
        const Real rho_next = dot(r, z);
        out.iters = k;
        if (rho_next <= stop) {
            out.rel_residual = std::sqrt(std::abs(rho_next) / rho0);
            out.converged = true;
            return out;
        }
        const Real beta = rho_next / rho;
        for (std::size_t i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
        rho = rho_next;
    }
    out.rel_residual = std::sqrt(std::abs(rho) / rho0);
    return out;
}


// ---------------------------------------------------------------------------
// Element-Hessian producer: the stable Neo-Hookean stencil
// (energy/neo_hookean.hpp:13-104), its PSD projection (energy/psd.hpp:8-14;
// Eigen's SelfAdjointEigenSolver restated in sym_eig.hpp) and the
// deformable-solid part of IncrementalPotential::assemble
// (solver/incremental_potential.hpp:170-180 inertia, :222-239 tets,
// scatter12 :310-318, pinned gradient :253-254). 12-vectors and 12x12
// matrices are plain column-major arrays.

// Eigen 3.4 determinant of a fixed 3x3 (Determinant.h bruteforce_det3_helper)
inline Real det3(const Mat3& m) {
    return m(0, 0) * (m(1, 1) * m(2, 2) - m(1, 2) * m(2, 1)) - m(0, 1) * (m(1, 0) * m(2, 2) - m(1, 2) * m(2, 0)) +
           m(0, 2) * (m(1, 0) * m(2, 1) - m(1, 1) * m(2, 0));
}

inline Vec3 cross(const Vec3& a, const Vec3& b) {  // Eigen cross order
    Vec3 c;
    c[0] = a[1] * b[2] - a[2] * b[1];
    c[1] = a[2] * b[0] - a[0] * b[2];
    c[2] = a[0] * b[1] - a[1] * b[0];
    return c;
}

// neo_hookean.hpp:8-27
struct TetRest {
    Mat3 inv_rest_edges;
    Real volume = 0;
};
inline TetRest tet_rest(const Vec3& p0, const Vec3& p1, const Vec3& p2, const Vec3& p3) {
    Mat3 Dm;
    for (int k = 0; k < 3; ++k) {
        Dm(k, 0) = p1[k] - p0[k];
        Dm(k, 1) = p2[k] - p0[k];
        Dm(k, 2) = p3[k] - p0[k];
    }
    const Real vol = det3(Dm) / 6.0;
    if (!(vol > 0)) throw std::invalid_argument("inverted or degenerate rest tet");
    return TetRest{Dm.inverse(), vol};
}

// neo_hookean.hpp:44-54: vec(F) vs (x0..x3), 9 x 12 column-major
inline void tet_dFdx(const Mat3& B, Real* J) {
    for (int k = 0; k < 108; ++k) J[k] = 0;
    for (int j = 0; j < 3; ++j)
        for (int c = 0; c < 3; ++c)
            for (int k = 0; k < 3; ++k) {
                J[9 * (3 * (c + 1) + k) + 3 * j + k] += B(c, j);
                J[9 * k + 3 * j + k] -= B(c, j);
            }
}

struct Stencil12 {  // neo_hookean.hpp:56-60
    Real value = 0;
    Real grad[12] = {};
    Real hess[144] = {};
};

// neo_hookean.hpp:64-104 (polynomial stable variant)
inline Stencil12 stable_neo_hookean(const Vec3& x0, const Vec3& x1, const Vec3& x2, const Vec3& x3,
                                    const TetRest& rest, Real mu, Real lam, bool project = true) {
    Mat3 Ds, F;
    for (int k = 0; k < 3; ++k) {
        Ds(k, 0) = x1[k] - x0[k];
        Ds(k, 1) = x2[k] - x0[k];
        Ds(k, 2) = x3[k] - x0[k];
    }
    const Mat3& B = rest.inv_rest_edges;
    for (int j = 0; j < 3; ++j)
        for (int i = 0; i < 3; ++i) F(i, j) = Ds(i, 0) * B(0, j) + Ds(i, 1) * B(1, j) + Ds(i, 2) * B(2, j);
    const Real J = det3(F);
    Real IC = 0;
    for (int k = 0; k < 9; ++k) IC += F.m[k] * F.m[k];
    Vec3 f[3];
    for (int c = 0; c < 3; ++c)
        for (int k = 0; k < 3; ++k) f[c][k] = F(k, c);
    const Vec3 cof_c[3] = {cross(f[1], f[2]), cross(f[2], f[0]), cross(f[0], f[1])};
    Real cof[9];
    for (int c = 0; c < 3; ++c)
        for (int k = 0; k < 3; ++k) cof[3 * c + k] = cof_c[c][k];
    const Real V = rest.volume;
    Stencil12 out;
    out.value = V * (0.5 * mu * (IC - 3) - mu * (J - 1) + 0.5 * lam * (J - 1) * (J - 1));
    const Real dJcoef = lam * (J - 1) - mu;
    Real P[9];
    for (int k = 0; k < 9; ++k) P[k] = mu * F.m[k] + dJcoef * cof[k];
    Real D[108];
    tet_dFdx(B, D);
    for (int i = 0; i < 12; ++i) {
        Real s = 0;
        for (int k = 0; k < 9; ++k) s += (V * D[9 * i + k]) * P[k];
        out.grad[i] = s;
    }
    // H9 = mu I + lam cof cof^T + dJcoef HJ (neo_hookean.hpp:90-99)
    Real H9[81];
    for (int j = 0; j < 9; ++j)
        for (int i = 0; i < 9; ++i) H9[9 * j + i] = (i == j ? mu : 0.0) + lam * cof[i] * cof[j];
    auto cross_mat = [](const Vec3& a, Real* M3) {  // neo_hookean.hpp:37-42, column-major
        M3[0] = 0, M3[3] = -a[2], M3[6] = a[1];
        M3[1] = a[2], M3[4] = 0, M3[7] = -a[0];
        M3[2] = -a[1], M3[5] = a[0], M3[8] = 0;
    };
    Real HJ[81] = {};
    auto put = [&](int bi, int bj, const Vec3& a, Real sgn) {
        Real M3[9];
        cross_mat(a, M3);
        for (int c = 0; c < 3; ++c)
            for (int r = 0; r < 3; ++r) HJ[9 * (3 * bj + c) + 3 * bi + r] = sgn * M3[3 * c + r];
    };
    put(0, 1, f[2], -1);
    put(0, 2, f[1], 1);
    put(1, 0, f[2], 1);
    put(1, 2, f[0], -1);
    put(2, 0, f[1], -1);
    put(2, 1, f[0], 1);
    for (int k = 0; k < 81; ++k) H9[k] += dJcoef * HJ[k];
    // hess = (V D^T) H9 D
    Real T[108];  // (V D^T) H9: 12 x 9
    for (int j = 0; j < 9; ++j)
        for (int i = 0; i < 12; ++i) {
            Real s = 0;
            for (int k = 0; k < 9; ++k) s += (V * D[9 * i + k]) * H9[9 * j + k];
            T[12 * j + i] = s;
        }
    for (int j = 0; j < 12; ++j)
        for (int i = 0; i < 12; ++i) {
            Real s = 0;
            for (int k = 0; k < 9; ++k) s += T[12 * k + i] * D[9 * j + k];
            out.hess[12 * j + i] = s;
        }
    if (project) {
        Real Pj[144];
        oracle_eig::project_psd(12, out.hess, Pj);
        for (int k = 0; k < 144; ++k) out.hess[k] = Pj[k];
    }
    return out;
}


// energy/abd_energy.hpp:9-42: rigidity penalty kappa V |A^T A - I|_F^2 on the
// affine part of q = [p, row0(A), row1(A), row2(A)]
inline Stencil12 abd_orthogonality(const Real* q, Real kappa, Real rest_volume, bool project = true) {
    Mat3 A;
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) A(r, c) = q[3 + 3 * r + c];
    Mat3 C;  // A^T A - I (Eigen lazy product: k ascending from the first term)
    for (int c = 0; c < 3; ++c)
        for (int r = 0; r < 3; ++r) C(r, c) = (A(0, r) * A(0, c) + A(1, r) * A(1, c) + A(2, r) * A(2, c)) - (r == c ? 1.0 : 0.0);
    const Real kv = kappa * rest_volume;
    Stencil12 out;
    Real cn = 0;
    for (int k = 0; k < 9; ++k) cn += C.m[k] * C.m[k];
    out.value = kv * cn;
    Mat3 G;  // 4 kv A C
    for (int c = 0; c < 3; ++c)
        for (int r = 0; r < 3; ++r) G(r, c) = (4 * kv * A(r, 0)) * C(0, c) + (4 * kv * A(r, 1)) * C(1, c) + (4 * kv * A(r, 2)) * C(2, c);
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) out.grad[3 + 3 * r + c] = G(r, c);
    Mat3 AAt;
    for (int c = 0; c < 3; ++c)
        for (int r = 0; r < 3; ++r) AAt(r, c) = A(r, 0) * A(c, 0) + A(r, 1) * A(c, 1) + A(r, 2) * A(c, 2);
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c)
            for (int s2 = 0; s2 < 3; ++s2)
                for (int t = 0; t < 3; ++t) {
                    const Real v = A(r, t) * A(s2, c) + (r == s2 ? C(t, c) : 0.0) + (t == c ? AAt(r, s2) : 0.0);
                    out.hess[12 * (3 + 3 * s2 + t) + 3 + 3 * r + c] = 4 * kv * v;
                }
    if (project) {
        Real P[144];
        oracle_eig::project_psd(12, out.hess, P);
        for (int k = 0; k < 144; ++k) out.hess[k] = P[k];
    }
    return out;
}


// ---------------------------------------------------------------------------
// Contact producers: closest-feature classification and
// per-feature squared distances with first and second derivatives
// (contact/distance.hpp:13-209, forward-mode AD of core/dual2.hpp restated),
// the log barrier (contact/barrier.hpp:14-91), lagged friction
// (contact/friction.hpp:12-91) and the contact-node part of
// IncrementalPotential::assemble_contact (solver/incremental_potential.hpp:
// 322-384); the line-search value (:61-159, contact terms) and the
// conservative-advancement CCD (contact/ccd.hpp:17-110).

// core/dual2.hpp:11-86 (N = 12; Hessian dense column-major as Eigen stores it)
struct Dual12 {
    Real v = 0;
    Real g[12] = {};
    Real h[144] = {};
    Dual12() = default;
    explicit Dual12(Real c) : v(c) {}
    static Dual12 variable(Real value, int k) {
        Dual12 d(value);
        d.g[k] = 1;
        return d;
    }
};
inline Dual12 operator+(const Dual12& a, const Dual12& b) {
    Dual12 r(a.v + b.v);
    for (int i = 0; i < 12; ++i) r.g[i] = a.g[i] + b.g[i];
    for (int i = 0; i < 144; ++i) r.h[i] = a.h[i] + b.h[i];
    return r;
}
inline Dual12 operator-(const Dual12& a, const Dual12& b) {
    Dual12 r(a.v - b.v);
    for (int i = 0; i < 12; ++i) r.g[i] = a.g[i] - b.g[i];
    for (int i = 0; i < 144; ++i) r.h[i] = a.h[i] - b.h[i];
    return r;
}
inline Dual12 operator*(const Dual12& a, const Dual12& b) {
    Dual12 r(a.v * b.v);
    for (int i = 0; i < 12; ++i) r.g[i] = a.g[i] * b.v + b.g[i] * a.v;
    for (int j = 0; j < 12; ++j)
        for (int i = 0; i < 12; ++i)
            r.h[12 * j + i] = a.h[12 * j + i] * b.v + b.h[12 * j + i] * a.v + a.g[i] * b.g[j] + b.g[i] * a.g[j];
    return r;
}
inline Dual12 inverse(const Dual12& b) {
    const Real iv = 1.0 / b.v;
    Dual12 r(iv);
    for (int i = 0; i < 12; ++i) r.g[i] = -b.g[i] * (iv * iv);
    const Real c = 2 * iv * iv * iv;
    for (int j = 0; j < 12; ++j)
        for (int i = 0; i < 12; ++i) r.h[12 * j + i] = -b.h[12 * j + i] * (iv * iv) + (c * b.g[i]) * b.g[j];
    return r;
}
inline Dual12 operator/(const Dual12& a, const Dual12& b) { return a * inverse(b); }
inline Dual12 operator*(const Dual12& a, Real s) {  // dual2.hpp:48-53
    Dual12 r(a.v * s);
    for (int i = 0; i < 12; ++i) r.g[i] = a.g[i] * s;
    for (int i = 0; i < 144; ++i) r.h[i] = a.h[i] * s;
    return r;
}
inline Dual12 operator*(Real s, const Dual12& a) { return a * s; }
inline Dual12 operator-(const Dual12& a, Real s) {  // a + (-s)
    Dual12 r = a;
    r.v += -s;
    return r;
}
inline Dual12 sqrt(const Dual12& a) {  // dual2.hpp:80-86
    const Real s = std::sqrt(a.v);
    Dual12 r(s);
    for (int i = 0; i < 12; ++i) r.g[i] = a.g[i] / (2 * s);
    for (int j = 0; j < 12; ++j)
        for (int i = 0; i < 12; ++i) r.h[12 * j + i] = a.h[12 * j + i] / (2 * s) - a.g[i] * a.g[j] / (4 * a.v * s);
    return r;
}
inline Dual12 atan2(const Dual12& y, const Dual12& x) {  // dual2.hpp:89-101
    const Real r2 = x.v * x.v + y.v * y.v;
    Dual12 r(std::atan2(y.v, x.v));
    for (int i = 0; i < 12; ++i) r.g[i] = (x.v * y.g[i] - y.v * x.g[i]) / r2;
    const Real c1 = y.v * y.v - x.v * x.v, c2 = 2 * x.v * y.v;
    for (int j = 0; j < 12; ++j)
        for (int i = 0; i < 12; ++i) {
            const Real gxgy = x.g[i] * y.g[j] + x.g[j] * y.g[i];
            const Real dd = x.g[i] * x.g[j] - y.g[i] * y.g[j];
            r.h[12 * j + i] = (c1 * gxgy + c2 * dd) / (r2 * r2) + (x.v * y.h[12 * j + i] - y.v * x.h[12 * j + i]) / r2;
        }
    return r;
}

template <class T>
using G3 = std::array<T, 3>;
template <class T>
G3<T> gsub(const G3<T>& a, const G3<T>& b) {
    return {a[0] - b[0], a[1] - b[1], a[2] - b[2]};
}
template <class T>
T gdot(const G3<T>& a, const G3<T>& b) {
    return a[0] * b[0] + a[1] * b[1] + a[2] * b[2];
}
template <class T>
G3<T> gcross(const G3<T>& a, const G3<T>& b) {
    return {a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]};
}
template <class T>
T gnorm2(const G3<T>& a) {
    return gdot(a, a);
}
using std::atan2;
using std::sqrt;

// distance.hpp:111-140
template <class T>
T pp_dist2_g(const G3<T>& a, const G3<T>& b) {
    return gnorm2(gsub(a, b));
}
template <class T>
T pe_dist2_g(const G3<T>& p, const G3<T>& e0, const G3<T>& e1) {
    const G3<T> d = gsub(e1, e0);
    const G3<T> w = gsub(p, e0);
    return gnorm2(gcross(w, d)) / gnorm2(d);
}
template <class T>
T pt_plane_dist2_g(const G3<T>& p, const G3<T>& t0, const G3<T>& t1, const G3<T>& t2) {
    const G3<T> n = gcross(gsub(t1, t0), gsub(t2, t0));
    const T h = gdot(gsub(p, t0), n);
    return h * h / gnorm2(n);
}
template <class T>
T ee_line_dist2_g(const G3<T>& a0, const G3<T>& a1, const G3<T>& b0, const G3<T>& b1) {
    const G3<T> n = gcross(gsub(a1, a0), gsub(b1, b0));
    const T h = gdot(gsub(b0, a0), n);
    return h * h / gnorm2(n);
}

inline Real dot3(const Vec3& a, const Vec3& b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }
inline Vec3 sub3(const Vec3& a, const Vec3& b) {
    Vec3 c;
    for (int k = 0; k < 3; ++k) c[k] = a[k] - b[k];
    return c;
}

// distance.hpp:13-108
enum class PtRegion { V0, V1, V2, E01, E12, E20, Interior };
enum class EeRegion { A0B0, A0B1, A1B0, A1B1, A0Int, A1Int, IntB0, IntB1, Interior };
struct PtClass {
    PtRegion region;
    Real beta[3];
};
struct EeClass {
    EeRegion region;
    Real s = 0, t = 0;
};
inline PtClass classify_pt(const Vec3& p, const Vec3& t0, const Vec3& t1, const Vec3& t2) {
    const Vec3 ab = sub3(t1, t0), ac = sub3(t2, t0), ap = sub3(p, t0);
    const Real d1 = dot3(ab, ap), d2 = dot3(ac, ap);
    if (d1 <= 0 && d2 <= 0) return {PtRegion::V0, {1, 0, 0}};
    const Vec3 bp = sub3(p, t1);
    const Real d3 = dot3(ab, bp), d4 = dot3(ac, bp);
    if (d3 >= 0 && d4 <= d3) return {PtRegion::V1, {0, 1, 0}};
    const Real vc = d1 * d4 - d3 * d2;
    if (vc <= 0 && d1 >= 0 && d3 <= 0) {
        const Real v = d1 / (d1 - d3);
        return {PtRegion::E01, {1 - v, v, 0}};
    }
    const Vec3 cp = sub3(p, t2);
    const Real d5 = dot3(ab, cp), d6 = dot3(ac, cp);
    if (d6 >= 0 && d5 <= d6) return {PtRegion::V2, {0, 0, 1}};
    const Real vb = d5 * d2 - d1 * d6;
    if (vb <= 0 && d2 >= 0 && d6 <= 0) {
        const Real w = d2 / (d2 - d6);
        return {PtRegion::E20, {1 - w, 0, w}};
    }
    const Real va = d3 * d6 - d5 * d4;
    if (va <= 0 && d4 - d3 >= 0 && d5 - d6 >= 0) {
        const Real w = (d4 - d3) / ((d4 - d3) + (d5 - d6));
        return {PtRegion::E12, {0, 1 - w, w}};
    }
    const Real denom = 1.0 / (va + vb + vc);
    const Real v = vb * denom, w = vc * denom;
    return {PtRegion::Interior, {1 - v - w, v, w}};
}
inline EeClass classify_ee(const Vec3& a0, const Vec3& a1, const Vec3& b0, const Vec3& b1) {
    const Vec3 da = sub3(a1, a0), db = sub3(b1, b0), r = sub3(a0, b0);
    const Real a = dot3(da, da), e = dot3(db, db);
    const Real f = dot3(db, r), c = dot3(da, r), b = dot3(da, db);
    const Real denom = a * e - b * b;
    Real s = 0;
    bool s_interior_formula = false;
    if (denom > 1e-12 * a * e) {
        s = (b * f - c * e) / denom;
        if (s <= 0)
            s = 0;
        else if (s >= 1)
            s = 1;
        else
            s_interior_formula = true;
    }
    Real t = e > 0 ? (b * s + f) / e : 0;
    bool t_clamped = false;
    if (t <= 0) {
        t = 0;
        t_clamped = true;
    } else if (t >= 1) {
        t = 1;
        t_clamped = true;
    }
    if (t_clamped) {
        s = a > 0 ? (b * t - c) / a : 0;
        s_interior_formula = s > 0 && s < 1;
        if (s <= 0)
            s = 0;
        else if (s >= 1)
            s = 1;
    }
    const bool s_end = !s_interior_formula;
    const bool t_end = t == 0 || t == 1;
    EeClass out;
    out.s = s;
    out.t = t;
    if (s_end && t_end)
        out.region = s == 0 ? (t == 0 ? EeRegion::A0B0 : EeRegion::A0B1) : (t == 0 ? EeRegion::A1B0 : EeRegion::A1B1);
    else if (s_end)
        out.region = s == 0 ? EeRegion::A0Int : EeRegion::A1Int;
    else if (t_end)
        out.region = t == 0 ? EeRegion::IntB0 : EeRegion::IntB1;
    else
        out.region = EeRegion::Interior;
    return out;
}
// distance.hpp:144-155 (value paths for ccd and the line-search value)
inline Real pt_dist2(const Vec3& p, const Vec3& t0, const Vec3& t1, const Vec3& t2) {
    const PtClass c = classify_pt(p, t0, t1, t2);
    Vec3 cl, d;
    for (int k = 0; k < 3; ++k) cl[k] = c.beta[0] * t0[k] + c.beta[1] * t1[k] + c.beta[2] * t2[k];
    d = sub3(p, cl);
    return dot3(d, d);
}
inline Real ee_dist2(const Vec3& a0, const Vec3& a1, const Vec3& b0, const Vec3& b1) {
    const EeClass c = classify_ee(a0, a1, b0, b1);
    Vec3 pa, pb;
    for (int k = 0; k < 3; ++k) {
        pa[k] = a0[k] + c.s * (a1[k] - a0[k]);
        pb[k] = b0[k] + c.t * (b1[k] - b0[k]);
    }
    const Vec3 d = sub3(pa, pb);
    return dot3(d, d);
}

// distance.hpp:159-223: squared distance of the active feature with its
// derivatives over the stacked stencil (12 dofs)
struct PairDerivs {
    Real dist2 = 0;
    Real grad[12] = {};
    Real hess[144] = {};
};
inline G3<Dual12> dual_point(const Vec3& p, int k0) {
    return {Dual12::variable(p[0], k0), Dual12::variable(p[1], k0 + 1), Dual12::variable(p[2], k0 + 2)};
}
inline PairDerivs pack_pair(const Dual12& d) {
    PairDerivs o;
    o.dist2 = d.v;
    for (int i = 0; i < 12; ++i) o.grad[i] = d.g[i];
    for (int i = 0; i < 144; ++i) o.hess[i] = d.h[i];
    return o;
}
inline PairDerivs pt_dist2_derivs(const Vec3& p, const Vec3& t0, const Vec3& t1, const Vec3& t2) {
    const PtClass c = classify_pt(p, t0, t1, t2);
    const auto P = dual_point(p, 0), T0 = dual_point(t0, 3), T1 = dual_point(t1, 6), T2 = dual_point(t2, 9);
    Dual12 d2;
    switch (c.region) {
        case PtRegion::V0: d2 = pp_dist2_g(P, T0); break;
        case PtRegion::V1: d2 = pp_dist2_g(P, T1); break;
        case PtRegion::V2: d2 = pp_dist2_g(P, T2); break;
        case PtRegion::E01: d2 = pe_dist2_g(P, T0, T1); break;
        case PtRegion::E12: d2 = pe_dist2_g(P, T1, T2); break;
        case PtRegion::E20: d2 = pe_dist2_g(P, T2, T0); break;
        case PtRegion::Interior: d2 = pt_plane_dist2_g(P, T0, T1, T2); break;
    }
    return pack_pair(d2);
}
inline PairDerivs ee_dist2_derivs(const Vec3& a0, const Vec3& a1, const Vec3& b0, const Vec3& b1) {
    const EeClass c = classify_ee(a0, a1, b0, b1);
    const auto A0 = dual_point(a0, 0), A1 = dual_point(a1, 3), B0 = dual_point(b0, 6), B1 = dual_point(b1, 9);
    Dual12 d2;
    switch (c.region) {
        case EeRegion::A0B0: d2 = pp_dist2_g(A0, B0); break;
        case EeRegion::A0B1: d2 = pp_dist2_g(A0, B1); break;
        case EeRegion::A1B0: d2 = pp_dist2_g(A1, B0); break;
        case EeRegion::A1B1: d2 = pp_dist2_g(A1, B1); break;
        case EeRegion::A0Int: d2 = pe_dist2_g(A0, B0, B1); break;
        case EeRegion::A1Int: d2 = pe_dist2_g(A1, B0, B1); break;
        case EeRegion::IntB0: d2 = pe_dist2_g(B0, A0, A1); break;
        case EeRegion::IntB1: d2 = pe_dist2_g(B1, A0, A1); break;
        case EeRegion::Interior: d2 = ee_line_dist2_g(A0, A1, B0, B1); break;
    }
    return pack_pair(d2);
}

// barrier.hpp:14-31
inline Real barrier_value(Real s, Real shat, Real kappa) {
    if (s >= shat) return 0;
    const Real r = s - shat;
    return -kappa * r * r * std::log(s / shat);
}
inline Real barrier_d1(Real s, Real shat, Real kappa) {
    if (s >= shat) return 0;
    const Real r = s - shat;
    return -kappa * (2 * r * std::log(s / shat) + r * r / s);
}
inline Real barrier_d2(Real s, Real shat, Real kappa) {
    if (s >= shat) return 0;
    const Real r = s - shat;
    return -kappa * (2 * std::log(s / shat) + 4 * r / s - r * r / (s * s));
}
inline Real barrier_curvature_in_d(Real d, Real dhat, Real kappa) {  // barrier.hpp:35-39
    const Real s = d * d;
    return 4 * s * barrier_d2(s, dhat * dhat, kappa) + 2 * barrier_d1(s, dhat * dhat, kappa);
}
// barrier.hpp:50-66
struct BarrierDerivs {
    Real value = 0;
    Real grad[12] = {};
    Real hess[144] = {};
};
inline BarrierDerivs barrier_pair_derivs(const PairDerivs& d, Real shat, Real kappa, bool project = true) {
    BarrierDerivs out;
    if (d.dist2 >= shat) return out;
    const Real b1 = barrier_d1(d.dist2, shat, kappa);
    const Real b2 = barrier_d2(d.dist2, shat, kappa);
    out.value = barrier_value(d.dist2, shat, kappa);
    for (int i = 0; i < 12; ++i) out.grad[i] = b1 * d.grad[i];
    for (int j = 0; j < 12; ++j)
        for (int i = 0; i < 12; ++i) out.hess[12 * j + i] = b2 * (d.grad[i] * d.grad[j]) + b1 * d.hess[12 * j + i];
    if (project) {
        Real P[144];
        oracle_eig::project_psd(12, out.hess, P);
        for (int k = 0; k < 144; ++k) out.hess[k] = P[k];
    }
    return out;
}
// barrier.hpp:70-91
struct GroundDerivs {
    Real value = 0;
    Vec3 grad;
    Mat3 hess;
    Real dist = 0;
};
inline GroundDerivs ground_barrier_derivs(const Vec3& x, const Vec3& normal, Real height, Real dhat, Real kappa,
                                          bool project = true) {
    GroundDerivs out;
    out.dist = dot3(normal, x) - height;
    const Real s = out.dist * out.dist;
    const Real shat = dhat * dhat;
    if (out.dist <= 0 || s >= shat) return out;
    out.value = barrier_value(s, shat, kappa);
    const Real gs = barrier_d1(s, shat, kappa) * 2 * out.dist;
    for (int k = 0; k < 3; ++k) out.grad[k] = gs * normal[k];
    Real c = barrier_curvature_in_d(out.dist, dhat, kappa);
    if (project && c < 0) c = 0;
    for (int j = 0; j < 3; ++j)
        for (int i = 0; i < 3; ++i) out.hess(i, j) = (c * normal[i]) * normal[j];
    return out;
}

// friction.hpp:12-36
inline Real friction_f0(Real y, Real eps) {
    if (y >= eps) return y;
    return -y * y * y / (3 * eps * eps) + y * y / eps + eps / 3;
}
inline Real friction_f1(Real y, Real eps) {
    if (y >= eps) return 1;
    return y * (2 * eps - y) / (eps * eps);
}
inline Real friction_f1_over_y(Real y, Real eps) {
    if (y >= eps) return 1 / y;
    return (2 * eps - y) / (eps * eps);
}
inline Real friction_f2(Real y, Real eps) {
    if (y >= eps) return 0;
    return 2 * (eps - y) / (eps * eps);
}
// friction.hpp:38-44
struct FrictionConstraint {
    Index nodes[4] = {kInvalid, kInvalid, kInvalid, kInvalid};
    int n_nodes = 0;
    Real coeff[4] = {0, 0, 0, 0};
    Vec3 t1, t2;
    Real lambda = 0;
};
// friction.hpp:58-91
struct FrictionDerivs {
    Real value = 0;
    Real grad[12] = {};
    Real hess[144] = {};
};
inline FrictionDerivs friction_derivs(const FrictionConstraint& c, const Vec3* dx, Real mu, Real eps) {
    FrictionDerivs out;
    Vec3 w;
    for (int k = 0; k < c.n_nodes; ++k)
        for (int a = 0; a < 3; ++a) w[a] += c.coeff[k] * dx[k][a];
    const Real u0 = dot3(c.t1, w), u1 = dot3(c.t2, w);
    const Real y = std::sqrt(u0 * u0 + u1 * u1);
    const Real scale = mu * c.lambda;
    out.value = scale * friction_f0(y, eps);
    Real inner[4];  // 2x2 column-major
    Vec3 gw;
    if (y > 1e-14 * eps) {
        const Real h0 = u0 / y, h1 = u1 / y;
        const Real f1 = scale * friction_f1(y, eps);
        for (int a = 0; a < 3; ++a) gw[a] = f1 * (c.t1[a] * h0 + c.t2[a] * h1);
        const Real f2 = friction_f2(y, eps), fy = friction_f1_over_y(y, eps);
        inner[0] = scale * (f2 * (h0 * h0) + fy * (1 - h0 * h0));
        inner[1] = scale * (f2 * (h1 * h0) + fy * (0 - h1 * h0));
        inner[2] = scale * (f2 * (h0 * h1) + fy * (0 - h0 * h1));
        inner[3] = scale * (f2 * (h1 * h1) + fy * (1 - h1 * h1));
    } else {
        const Real fy = scale * friction_f1_over_y(0, eps);
        inner[0] = fy, inner[1] = 0, inner[2] = 0, inner[3] = fy;
    }
    Mat3 hw;  // P inner P^T, P = [t1 t2]
    for (int j = 0; j < 3; ++j)
        for (int i = 0; i < 3; ++i) {
            const Real pi0 = c.t1[i], pi1 = c.t2[i];
            const Real q0 = inner[0] * c.t1[j] + inner[2] * c.t2[j];
            const Real q1 = inner[1] * c.t1[j] + inner[3] * c.t2[j];
            hw(i, j) = pi0 * q0 + pi1 * q1;
        }
    for (int k = 0; k < c.n_nodes; ++k) {
        for (int a = 0; a < 3; ++a) out.grad[3 * k + a] = c.coeff[k] * gw[a];
        for (int l = 0; l < c.n_nodes; ++l)
            for (int b = 0; b < 3; ++b)
                for (int a = 0; a < 3; ++a)
                    out.hess[12 * (3 * l + b) + 3 * k + a] = c.coeff[k] * c.coeff[l] * hw(a, b);
    }
    return out;
}

// The contact-node part of IncrementalPotential::assemble_contact
// (incremental_potential.hpp:322-384) for GIVEN candidates (pt / ee stencils
// as node ids; the broad phase of :330 is separate): node stream in emission
// order (active PT pairs, active EE pairs, ground contacts, friction
// constraints), node gradient, value. Returns the value.
struct ContactInput {
    std::vector<Vec3> pos;                       // contact-node positions
    std::vector<std::array<Index, 4>> pt, ee;    // stencils (v, t0, t1, t2) / (a0, a1, b0, b1)
    Real dhat = 0, kappa = 0;
    bool ground = false;
    Vec3 ground_normal;
    Real ground_height = 0;
    std::vector<Index> surf_verts;
    std::vector<FrictionConstraint> friction;
    std::vector<Vec3> fr_base;
    Real mu = 0, fr_eps = 1;
};
inline Real contact_assemble(const ContactInput& in, Real dt2, std::vector<Vec3>& node_grad,
                             BlockTripletStream& out, bool project = true) {
    const Real shat = in.dhat * in.dhat;
    node_grad.assign(in.pos.size(), Vec3());
    out.keys.clear();
    out.values.clear();
    Real val = 0;
    struct PS {
        BarrierDerivs bd;
        Index nodes[4];
        Real dist2;
    };
    std::vector<PS> ps(in.pt.size() + in.ee.size());
#pragma omp parallel for schedule(static)
    for (std::int64_t i = 0; i < static_cast<std::int64_t>(ps.size()); ++i) {
        const bool is_pt = i < static_cast<std::int64_t>(in.pt.size());
        const auto& st = is_pt ? in.pt[i] : in.ee[i - in.pt.size()];
        const PairDerivs pd = is_pt ? pt_dist2_derivs(in.pos[st[0]], in.pos[st[1]], in.pos[st[2]], in.pos[st[3]])
                                    : ee_dist2_derivs(in.pos[st[0]], in.pos[st[1]], in.pos[st[2]], in.pos[st[3]]);
        ps[i].bd = barrier_pair_derivs(pd, shat, in.kappa, project);
        for (int a = 0; a < 4; ++a) ps[i].nodes[a] = st[a];
        ps[i].dist2 = pd.dist2;
    }
    auto emit12 = [&](const Index* nodes, int n, const Real* hess) {
        for (int a = 0; a < n; ++a)
            for (int b = a; b < n; ++b) {
                Mat3 blk;
                for (int c = 0; c < 3; ++c)
                    for (int r = 0; r < 3; ++r) blk(r, c) = dt2 * hess[12 * (3 * b + c) + 3 * a + r];
                out.emit(nodes[a], nodes[b], blk);
            }
    };
    for (const auto& p : ps) {  // :350-359
        if (p.dist2 >= shat) continue;
        val += dt2 * p.bd.value;
        for (int a = 0; a < 4; ++a)
            for (int k = 0; k < 3; ++k) node_grad[p.nodes[a]][k] += dt2 * p.bd.grad[3 * a + k];
        emit12(p.nodes, 4, p.bd.hess);
    }
    if (in.ground)  // :361-369
        for (Index v : in.surf_verts) {
            const GroundDerivs gd =
                ground_barrier_derivs(in.pos[v], in.ground_normal, in.ground_height, in.dhat, in.kappa, project);
            if (!(gd.dist > 0) || gd.dist >= in.dhat) continue;
            val += dt2 * gd.value;
            for (int k = 0; k < 3; ++k) node_grad[v][k] += dt2 * gd.grad[k];
            Mat3 blk;
            for (int k = 0; k < 9; ++k) blk.m[k] = dt2 * gd.hess.m[k];
            out.emit(v, v, blk);
        }
    for (const auto& c : in.friction) {  // :371-382
        Vec3 dx[4];
        for (int k = 0; k < c.n_nodes; ++k) dx[k] = sub3(in.pos[c.nodes[k]], in.fr_base[c.nodes[k]]);
        const FrictionDerivs fd = friction_derivs(c, dx, in.mu, in.fr_eps);
        val += dt2 * fd.value;
        for (int a = 0; a < c.n_nodes; ++a)
            for (int k = 0; k < 3; ++k) node_grad[c.nodes[a]][k] += dt2 * fd.grad[3 * a + k];
        emit12(c.nodes, c.n_nodes, fd.hess);
    }
    return val;
}

// The contact terms of IncrementalPotential::value (incremental_potential.hpp:
// 133-157): +inf as soon as a stencil or a surface vertex touches.
inline Real contact_value(const ContactInput& in, Real dt2) {
    const Real shat = in.dhat * in.dhat;
    Real val = 0;
    for (const auto& c : in.pt) {
        const Real d2 = pt_dist2(in.pos[c[0]], in.pos[c[1]], in.pos[c[2]], in.pos[c[3]]);
        if (d2 <= 0) return std::numeric_limits<Real>::infinity();
        if (d2 < shat) val += dt2 * barrier_value(d2, shat, in.kappa);
    }
    for (const auto& c : in.ee) {
        const Real d2 = ee_dist2(in.pos[c[0]], in.pos[c[1]], in.pos[c[2]], in.pos[c[3]]);
        if (d2 <= 0) return std::numeric_limits<Real>::infinity();
        if (d2 < shat) val += dt2 * barrier_value(d2, shat, in.kappa);
    }
    if (in.ground)
        for (Index v : in.surf_verts) {
            const Real d = dot3(in.ground_normal, in.pos[v]) - in.ground_height;
            if (d <= 0) return std::numeric_limits<Real>::infinity();
            if (d < in.dhat) val += dt2 * barrier_value(d * d, shat, in.kappa);
        }
    for (const auto& c : in.friction) {
        Vec3 w;
        for (int k = 0; k < c.n_nodes; ++k)
            for (int a = 0; a < 3; ++a) w[a] += c.coeff[k] * (in.pos[c.nodes[k]][a] - in.fr_base[c.nodes[k]][a]);
        const Real u0 = dot3(c.t1, w), u1 = dot3(c.t2, w);
        val += dt2 * in.mu * c.lambda * friction_f0(std::sqrt(u0 * u0 + u1 * u1), in.fr_eps);
    }
    return val;
}

// contact/ccd.hpp:17-56 conservative advancement
constexpr Real kCcdGapFraction = 0.01, kCcdRescale = 0.9;
constexpr int kCcdMaxIters = 64;
template <class Dist2Fn>
Real conservative_toi(const Vec3* x0, const Vec3* d0, int n_side_a, int n_nodes, Dist2Fn&& dist2_of) {
    Vec3 x[4], d[4], mean;
    for (int i = 0; i < n_nodes; ++i) {
        x[i] = x0[i];
        d[i] = d0[i];
        for (int a = 0; a < 3; ++a) mean[a] += d[i][a];
    }
    for (int a = 0; a < 3; ++a) mean[a] /= n_nodes;
    Real max_a = 0, max_b = 0;
    for (int i = 0; i < n_nodes; ++i) {
        for (int a = 0; a < 3; ++a) d[i][a] -= mean[a];
        const Real len = std::sqrt(dot3(d[i], d[i]));
        Real& m = i < n_side_a ? max_a : max_b;
        m = std::max(m, len);
    }
    const Real speed = max_a + max_b;
    if (speed == 0) return 1;
    const Real g0 = std::sqrt(dist2_of(x));
    if (!(g0 > 0)) return 0;
    const Real gap = kCcdGapFraction * g0;
    Real t = 0;
    Vec3 cur[4];
    for (int i = 0; i < n_nodes; ++i) cur[i] = x[i];
    for (int iter = 0; iter < kCcdMaxIters; ++iter) {
        const Real g = std::sqrt(dist2_of(cur));
        if (g <= gap) return kCcdRescale * t;
        const Real step = (g - gap) / speed;
        if (t + step >= 1) return 1;
        t += step;
        for (int i = 0; i < n_nodes; ++i)
            for (int a = 0; a < 3; ++a) cur[i][a] = x[i][a] + t * d[i][a];
    }
    return kCcdRescale * t;
}
// ccd.hpp:58-86
inline Real pt_ccd_toi(const Vec3* x, const Vec3* d) {
    return conservative_toi(x, d, 1, 4, [](const Vec3* c) { return pt_dist2(c[0], c[1], c[2], c[3]); });
}
inline Real ee_ccd_toi(const Vec3* x, const Vec3* d) {
    return conservative_toi(x, d, 2, 4, [](const Vec3* c) { return ee_dist2(c[0], c[1], c[2], c[3]); });
}
inline Real ground_ccd_toi(const Vec3& x, const Vec3& dx, const Vec3& normal, Real height) {
    const Real g0 = dot3(normal, x) - height;
    if (!(g0 > 0)) return 0;
    const Real closing = -dot3(normal, dx);
    if (closing <= 0) return 1;
    const Real t_gap = (1 - kCcdGapFraction) * g0 / closing;
    if (t_gap >= 1) return 1;
    return kCcdRescale * t_gap;
}
// ccd.hpp:88-110 over GIVEN candidates (the ccd broad phase of :91 is separate)
inline Real ccd_step(const ContactInput& in, const std::vector<Vec3>& disp) {
    Real alpha = 1;
    for (std::size_t i = 0; i < in.pt.size() + in.ee.size(); ++i) {
        const bool is_pt = i < in.pt.size();
        const auto& st = is_pt ? in.pt[i] : in.ee[i - in.pt.size()];
        Vec3 x[4], d[4];
        for (int a = 0; a < 4; ++a) {
            x[a] = in.pos[st[a]];
            d[a] = disp[st[a]];
        }
        alpha = std::min(alpha, is_pt ? pt_ccd_toi(x, d) : ee_ccd_toi(x, d));
    }
    if (in.ground)
        for (Index v : in.surf_verts)
            alpha = std::min(alpha, ground_ccd_toi(in.pos[v], disp[v], in.ground_normal, in.ground_height));
    return alpha;
}

// contact/distance.hpp:226-256: the frame of a stencil's closest features —
// distance, unit normal from the second feature towards the first (UnitY at
// zero distance), relative-displacement coefficients
struct ContactFrame {
    Real dist = 0;
    Vec3 normal;
    Real coeff[4] = {0, 0, 0, 0};
};
inline ContactFrame frame_of(const Vec3& d) {
    ContactFrame f;
    f.dist = std::sqrt(dot3(d, d));
    if (f.dist > 0) {
        for (int a = 0; a < 3; ++a) f.normal[a] = d[a] / f.dist;
    } else {
        f.normal[1] = 1;
    }
    return f;
}
inline ContactFrame pt_contact_frame(const Vec3& p, const Vec3& t0, const Vec3& t1, const Vec3& t2) {
    const PtClass c = classify_pt(p, t0, t1, t2);
    Vec3 d;
    for (int a = 0; a < 3; ++a) d[a] = p[a] - ((c.beta[0] * t0[a] + c.beta[1] * t1[a]) + c.beta[2] * t2[a]);
    ContactFrame f = frame_of(d);
    f.coeff[0] = 1;
    f.coeff[1] = -c.beta[0];
    f.coeff[2] = -c.beta[1];
    f.coeff[3] = -c.beta[2];
    return f;
}
inline ContactFrame ee_contact_frame(const Vec3& a0, const Vec3& a1, const Vec3& b0, const Vec3& b1) {
    const EeClass c = classify_ee(a0, a1, b0, b1);
    Vec3 d;
    for (int a = 0; a < 3; ++a) d[a] = (a0[a] + c.s * (a1[a] - a0[a])) - (b0[a] + c.t * (b1[a] - b0[a]));
    ContactFrame f = frame_of(d);
    f.coeff[0] = 1 - c.s;
    f.coeff[1] = c.s;
    f.coeff[2] = -(1 - c.t);
    f.coeff[3] = -c.t;
    return f;
}
// friction.hpp:43-47
inline void tangent_basis(const Vec3& n, Vec3& t1, Vec3& t2) {
    Vec3 ref;
    ref[std::abs(n[0]) > 0.9 ? 1 : 0] = 1;
    auto cross = [](const Vec3& a, const Vec3& b) {
        Vec3 r;
        r[0] = a[1] * b[2] - a[2] * b[1];
        r[1] = a[2] * b[0] - a[0] * b[2];
        r[2] = a[0] * b[1] - a[1] * b[0];
        return r;
    };
    const Vec3 u = cross(n, ref);
    const Real z = dot3(u, u);  // Eigen normalized(): / sqrt(squaredNorm) when positive
    if (z > 0) {
        const Real nz = std::sqrt(z);
        for (int a = 0; a < 3; ++a) t1[a] = u[a] / nz;
    } else {
        t1 = u;
    }
    t2 = cross(n, t1);
}
// friction.hpp:93-149 build_friction_constraints for GIVEN candidates (the
// proximity broad phase of :99 is separate): active PT stencils, active EE
// stencils, then ground contacts of the surface vertices, in that order;
// lambda = -b'(d^2) 2 d, the lagged normal force
inline std::vector<FrictionConstraint> friction_constraints(const ContactInput& in) {
    std::vector<FrictionConstraint> out;
    const Real shat = in.dhat * in.dhat;
    auto normal_force = [&](Real dist) { return -barrier_d1(dist * dist, shat, in.kappa) * 2 * dist; };
    auto add = [&](const ContactFrame& f, const std::array<Index, 4>& nodes) {
        if (!(f.dist > 0) || f.dist >= in.dhat) return;
        FrictionConstraint fc;
        for (int k = 0; k < 4; ++k) {
            fc.nodes[k] = nodes[k];
            fc.coeff[k] = f.coeff[k];
        }
        fc.n_nodes = 4;
        tangent_basis(f.normal, fc.t1, fc.t2);
        fc.lambda = normal_force(f.dist);
        out.push_back(fc);
    };
    for (const auto& st : in.pt) add(pt_contact_frame(in.pos[st[0]], in.pos[st[1]], in.pos[st[2]], in.pos[st[3]]), st);
    for (const auto& st : in.ee) add(ee_contact_frame(in.pos[st[0]], in.pos[st[1]], in.pos[st[2]], in.pos[st[3]]), st);
    if (in.ground)
        for (Index v : in.surf_verts) {
            const Real dist = dot3(in.ground_normal, in.pos[v]) - in.ground_height;
            if (!(dist > 0) || dist >= in.dhat) continue;
            FrictionConstraint fc;
            fc.nodes[0] = v;
            fc.n_nodes = 1;
            fc.coeff[0] = 1;
            tangent_basis(in.ground_normal, fc.t1, fc.t2);
            fc.lambda = normal_force(dist);
            out.push_back(fc);
        }
    return out;
}

// contact/broad_phase.hpp:13-226: contact surface primitives over the
// contact-node universe, inflated (and swept) AABBs, a hash grid of the
// triangle / edge boxes, vertex-triangle and edge-edge candidates sorted and
// duplicate free, stencils sharing a node dropped.
struct ContactSurface {
    std::vector<Index> verts;
    std::vector<std::array<Index, 2>> edges;
    std::vector<std::array<Index, 3>> tris;
};
struct Aabb {  // :57-71
    Real lo[3] = {std::numeric_limits<Real>::max(), std::numeric_limits<Real>::max(),
                  std::numeric_limits<Real>::max()};
    Real hi[3] = {-std::numeric_limits<Real>::max(), -std::numeric_limits<Real>::max(),
                  -std::numeric_limits<Real>::max()};
    void grow(const Real* p) {
        for (int a = 0; a < 3; ++a) {
            lo[a] = std::min(lo[a], p[a]);
            hi[a] = std::max(hi[a], p[a]);
        }
    }
    void inflate(Real r) {
        for (int a = 0; a < 3; ++a) {
            lo[a] -= r;
            hi[a] += r;
        }
    }
    bool overlaps(const Aabb& o) const {
        for (int a = 0; a < 3; ++a)
            if (!(lo[a] <= o.hi[a] && o.lo[a] <= hi[a])) return false;
        return true;
    }
};
struct ContactCandidates {  // :76-79
    std::vector<std::array<Index, 2>> pt, ee;
};
class HashGrid {  // :83-123
public:
    void build(const std::vector<Aabb>& boxes, Real cell_size) {
        cell_ = cell_size;
        cells_.clear();
        for (std::size_t i = 0; i < boxes.size(); ++i)
            visit(boxes[i], [&](std::uint64_t key) { cells_[key].push_back(static_cast<Index>(i)); });
    }
    template <class F>
    void query(const Aabb& box, F&& fn) const {
        visit(box, [&](std::uint64_t key) {
            auto it = cells_.find(key);
            if (it == cells_.end()) return;
            for (Index id : it->second) fn(id);
        });
    }

private:
    template <class F>
    void visit(const Aabb& box, F&& fn) const {
        long lo[3], hi[3];
        for (int a = 0; a < 3; ++a) {
            lo[a] = static_cast<long>(std::floor(box.lo[a] / cell_));
            hi[a] = static_cast<long>(std::floor(box.hi[a] / cell_));
        }
        for (long x = lo[0]; x <= hi[0]; ++x)
            for (long y = lo[1]; y <= hi[1]; ++y)
                for (long z = lo[2]; z <= hi[2]; ++z) fn(pack(x, y, z));
    }
    static std::uint64_t pack(long x, long y, long z) {
        const std::uint64_t m = (1u << 21) - 1;
        auto wrap = [&](long v) { return static_cast<std::uint64_t>(v & static_cast<long>(m)); };
        return (wrap(x) << 42) | (wrap(y) << 21) | wrap(z);
    }
    Real cell_ = 1;
    std::unordered_map<std::uint64_t, std::vector<Index>> cells_;
};
inline Aabb swept_point(const std::vector<Vec3>& pos, const std::vector<Vec3>* disp, Index node) {  // :125-131
    Aabb box;
    box.grow(pos[node].v);
    if (disp) {
        Real e[3];
        for (int a = 0; a < 3; ++a) e[a] = pos[node][a] + (*disp)[node][a];
        box.grow(e);
    }
    return box;
}
inline void sort_unique(std::vector<std::array<Index, 2>>& pairs) {
    std::sort(pairs.begin(), pairs.end());
    pairs.erase(std::unique(pairs.begin(), pairs.end()), pairs.end());
}
// :143-211
inline ContactCandidates find_candidates(const ContactSurface& surf, const std::vector<Vec3>& pos,
                                         const std::vector<Vec3>* disp, Real inflate) {
    ContactCandidates out;
    const Real half = inflate / 2;
    std::vector<Aabb> tri_boxes(surf.tris.size());
    Real mean_extent = 0;
    for (std::size_t t = 0; t < surf.tris.size(); ++t) {
        Aabb box;
        for (Index v : surf.tris[t]) {
            const Aabb p = swept_point(pos, disp, v);
            box.grow(p.lo);
            box.grow(p.hi);
        }
        mean_extent += std::max({box.hi[0] - box.lo[0], box.hi[1] - box.lo[1], box.hi[2] - box.lo[2]});
        box.inflate(half);
        tri_boxes[t] = box;
    }
    std::vector<Aabb> edge_boxes(surf.edges.size());
    for (std::size_t e = 0; e < surf.edges.size(); ++e) {
        Aabb box;
        for (Index v : surf.edges[e]) {
            const Aabb p = swept_point(pos, disp, v);
            box.grow(p.lo);
            box.grow(p.hi);
        }
        box.inflate(half);
        edge_boxes[e] = box;
    }
    if (surf.tris.empty() && surf.edges.empty()) return out;
    mean_extent = surf.tris.empty() ? inflate : mean_extent / surf.tris.size();
    const Real cell = std::max(mean_extent + inflate, 1e-12);
    HashGrid tri_grid;
    tri_grid.build(tri_boxes, cell);
    for (std::size_t vi = 0; vi < surf.verts.size(); ++vi) {
        const Index node = surf.verts[vi];
        Aabb box = swept_point(pos, disp, node);
        box.inflate(half);
        tri_grid.query(box, [&](Index t) {
            const auto& tri = surf.tris[t];
            if (tri[0] == node || tri[1] == node || tri[2] == node) return;
            if (!box.overlaps(tri_boxes[t])) return;
            out.pt.push_back({static_cast<Index>(vi), t});
        });
    }
    sort_unique(out.pt);
    HashGrid edge_grid;
    edge_grid.build(edge_boxes, cell);
    for (std::size_t ei = 0; ei < surf.edges.size(); ++ei) {
        const auto& ea = surf.edges[ei];
        edge_grid.query(edge_boxes[ei], [&](Index ej) {
            if (ej <= static_cast<Index>(ei)) return;
            const auto& eb = surf.edges[ej];
            if (ea[0] == eb[0] || ea[0] == eb[1] || ea[1] == eb[0] || ea[1] == eb[1]) return;
            if (!edge_boxes[ei].overlaps(edge_boxes[ej])) return;
            out.ee.push_back({static_cast<Index>(ei), ej});
        });
    }
    sort_unique(out.ee);
    return out;
}

// ---------------------------------------------------------------------------
// Shell energies: energy/membrane.hpp:10-131 (FBW
// stretch, cubic strain limit, I6 shear), IncrementalPotential::
// membrane_stencil (incremental_potential.hpp:273-298) and the hinge
// bending of energy/bending.hpp:11-77 (dihedral angle by forward AD).
struct MembraneRest {
    Real inv[4];  // Mat2 column-major
    Real area = 0;
};
inline MembraneRest membrane_rest(const Vec3& p0, const Vec3& p1, const Vec3& p2) {  // membrane.hpp:17-32
    const Vec3 e1 = sub3(p1, p0), e2 = sub3(p2, p0);
    const Vec3 nrm = cross(e1, e2);
    const Real area2 = std::sqrt(dot3(nrm, nrm));
    const Real n1 = std::sqrt(dot3(e1, e1)), n2 = std::sqrt(dot3(e2, e2));
    if (!(area2 > 1e-14 * n1 * n2) || n1 == 0) throw std::invalid_argument("degenerate rest triangle");
    Vec3 u, nn;
    for (int k = 0; k < 3; ++k) {
        u[k] = e1[k] / n1;
        nn[k] = nrm[k] / area2;
    }
    const Vec3 v = cross(nn, u);
    const Real a = dot3(e1, u), b = dot3(e2, u), c = dot3(e1, v), d = dot3(e2, v);  // Dm << a, b, c, d (row-wise)
    const Real invdet = 1.0 / (a * d - b * c);
    MembraneRest r;
    r.inv[0] = d * invdet;   // (0,0)
    r.inv[1] = -c * invdet;  // (1,0)
    r.inv[2] = -b * invdet;  // (0,1)
    r.inv[3] = a * invdet;   // (1,1)
    r.area = 0.5 * area2;
    return r;
}
struct ShellMaterial {  // scene/mesh.hpp:17-24
    Real thickness = 1e-3, stretch = 5e4, strain_limit = 5e6, shear_fraction = 0.3, bending = 1e-6;
};
struct Stencil9 {
    Real value = 0;
    Real grad[9] = {};
    Real hess[81] = {};
};
// incremental_potential.hpp:273-298 with membrane.hpp:36-131
inline Stencil9 membrane_stencil(const Vec3& x0, const Vec3& x1, const Vec3& x2, const MembraneRest& rest,
                                 const ShellMaterial& m, bool project = true) {
    Real F[6];  // 3x2 column-major: D * inv
    for (int j = 0; j < 2; ++j)
        for (int k = 0; k < 3; ++k)
            F[3 * j + k] = (x1[k] - x0[k]) * rest.inv[2 * j] + (x2[k] - x0[k]) * rest.inv[2 * j + 1];
    const Real a_t = rest.area * m.thickness;
    Real value = 0, dF[6] = {}, H6[36] = {};
    // fbw_membrane (:54-75)
    {
        const Real scale = m.stretch * a_t;
        for (int dir = 0; dir < 2; ++dir) {
            const Real* f = F + 3 * dir;
            const Real I5v = f[0] * f[0] + f[1] * f[1] + f[2] * f[2];
            const Real sq = std::sqrt(I5v);
            value += scale * (sq - 1) * (sq - 1);
            for (int k = 0; k < 3; ++k) dF[3 * dir + k] += 2 * scale * (1 - 1 / sq) * f[k];
            const Real e1 = 2 * scale;
            Real e23 = 2 * scale * (1 - 1 / sq);
            if (project && e23 < 0) e23 = 0;
            for (int c = 0; c < 3; ++c)
                for (int r = 0; r < 3; ++r)
                    H6[6 * (3 * dir + c) + 3 * dir + r] +=
                        (r == c ? e23 : 0.0) + (e1 - e23) * (f[r] / sq) * (f[c] / sq);
        }
    }
    // cubic_strain_limit (:87-102)
    {
        const Real scale = m.strain_limit * a_t;
        for (int dir = 0; dir < 2; ++dir) {
            const Real* f = F + 3 * dir;
            const Real I5v = f[0] * f[0] + f[1] * f[1] + f[2] * f[2];
            if (I5v <= 1.0) continue;
            const Real sq = std::sqrt(I5v);
            value += scale * (sq - 1) * (sq - 1) * (sq - 1);
            for (int k = 0; k < 3; ++k) dF[3 * dir + k] += scale * (3 * (sq - 1) * (sq - 1) / sq) * f[k];
            const Real e1 = 6 * (sq - 1), e23 = 3 * (1 / sq + sq - 2);
            for (int c = 0; c < 3; ++c)
                for (int r = 0; r < 3; ++r)
                    H6[6 * (3 * dir + c) + 3 * dir + r] +=
                        scale * ((r == c ? e23 : 0.0) + ((e1 - e23) / I5v) * f[r] * f[c]);
        }
    }
    // shear_energy (:105-121)
    {
        const Real scale = m.shear_fraction * m.stretch * a_t;
        const Real* f0 = F;
        const Real* f1 = F + 3;
        const Real I6 = f0[0] * f1[0] + f0[1] * f1[1] + f0[2] * f1[2];
        value += scale * I6 * I6;
        for (int k = 0; k < 3; ++k) {
            dF[k] += 2 * scale * I6 * f1[k];
            dF[3 + k] += 2 * scale * I6 * f0[k];
        }
        const Real g[6] = {f1[0], f1[1], f1[2], f0[0], f0[1], f0[2]};
        Real S[36];
        for (int c = 0; c < 6; ++c)
            for (int r = 0; r < 6; ++r)
                S[6 * c + r] = 2 * scale * (g[r] * g[c] + I6 * ((r < 3) != (c < 3) && r % 3 == c % 3 ? 1.0 : 0.0));
        if (project) {
            Real P[36];
            oracle_eig::project_psd(6, S, P);
            for (int k = 0; k < 36; ++k) S[k] = P[k];
        }
        for (int k = 0; k < 36; ++k) H6[k] += S[k];
    }
    // chain rule through membrane_dFdx (:124-135): C(a, j), a = vertex
    Real C[3][2];
    for (int j = 0; j < 2; ++j) {
        C[0][j] = -rest.inv[2 * j] - rest.inv[2 * j + 1];
        C[1][j] = rest.inv[2 * j];
        C[2][j] = rest.inv[2 * j + 1];
    }
    Stencil9 out;
    out.value = value;
    for (int a = 0; a < 3; ++a)
        for (int k = 0; k < 3; ++k) out.grad[3 * a + k] = C[a][0] * dF[k] + C[a][1] * dF[3 + k];
    for (int b = 0; b < 3; ++b)
        for (int c = 0; c < 3; ++c)
            for (int a = 0; a < 3; ++a)
                for (int r = 0; r < 3; ++r) {
                    Real v = 0;
                    for (int j = 0; j < 2; ++j)
                        for (int l = 0; l < 2; ++l) v += C[a][j] * C[b][l] * H6[6 * (3 * l + c) + 3 * j + r];
                    out.hess[9 * (3 * b + c) + 3 * a + r] = v;
                }
    return out;
}

// bending.hpp:11-53
template <class T>
T dihedral_angle_g(const G3<T>& x0, const G3<T>& x1, const G3<T>& x2, const G3<T>& x3) {
    const G3<T> e = gsub(x1, x0);
    const G3<T> n1 = gcross(e, gsub(x2, x0));
    const G3<T> n2 = gcross(gsub(x3, x0), e);
    const T s = gdot(gcross(n1, n2), e) / sqrt(gnorm2(e));
    const T c = gdot(n1, n2);
    return atan2(s, c);
}
inline G3<Real> as_g(const Vec3& p) { return {p[0], p[1], p[2]}; }
struct HingeRest {
    Real rest_angle = 0, weight = 0;
};
inline HingeRest hinge_rest(const Vec3& p0, const Vec3& p1, const Vec3& p2, const Vec3& p3) {
    const Vec3 c1 = cross(sub3(p1, p0), sub3(p2, p0)), c2 = cross(sub3(p3, p0), sub3(p1, p0));
    const Real a1 = 0.5 * std::sqrt(dot3(c1, c1)), a2 = 0.5 * std::sqrt(dot3(c2, c2));
    if (!(a1 > 0) || !(a2 > 0)) throw std::invalid_argument("degenerate hinge rest triangles");
    HingeRest r;
    r.rest_angle = dihedral_angle_g<Real>(as_g(p0), as_g(p1), as_g(p2), as_g(p3));
    const Vec3 e = sub3(p1, p0);
    r.weight = 3 * dot3(e, e) / (a1 + a2);
    return r;
}
// bending.hpp:60-75: k w (theta - rest)^2 by forward AD, projected
inline Stencil12 hinge_bending(const Vec3& x0, const Vec3& x1, const Vec3& x2, const Vec3& x3, const HingeRest& rest,
                               Real k, bool project = true) {
    const Dual12 th = dihedral_angle_g(dual_point(x0, 0), dual_point(x1, 3), dual_point(x2, 6), dual_point(x3, 9));
    const Dual12 diff = th - rest.rest_angle;
    const Dual12 e = (k * rest.weight) * (diff * diff);
    Stencil12 out;
    out.value = e.v;
    for (int i = 0; i < 12; ++i) out.grad[i] = e.g[i];
    if (project)
        oracle_eig::project_psd(12, e.h, out.hess);
    else
        for (int i = 0; i < 144; ++i) out.hess[i] = e.h[i];
    return out;
}

// The deformable meshes of a scene in scene order (kind 0 solid -> the next
// FemSolids mesh, 1 shell -> the next shell), for ip_fem_assemble's element
// loop (incremental_potential.hpp:190-241).
struct FemShells {
    std::vector<std::int32_t> tris;          // 3 global slots per triangle
    std::vector<MembraneRest> tri_rest;
    std::vector<std::int64_t> tri_begin;     // per shell mesh, + 1
    std::vector<std::int32_t> hinges;        // 4 global slots per hinge
    std::vector<HingeRest> hinge_rest;
    std::vector<std::int64_t> hinge_begin;   // per shell mesh, + 1
    std::vector<ShellMaterial> material;     // per shell mesh
};


// One deformable solid part of the scene for the producer: tets as global
// slot ids (mesh offset applied), rest data and material per mesh.
struct FemSolids {
    std::vector<std::int32_t> tets;      // 4 per tet
    std::vector<TetRest> rest;           // per tet
    std::vector<std::int64_t> tet_begin; // per mesh, n_meshes + 1
    std::vector<Real> mu, lam;           // per mesh
};

// Affine bodies of the scene (scene.hpp Body): q, q_tilde, reduced mass
// (12 x 12 column-major), orthogonality stiffness and rest volume; body b
// owns block rows n_fem + 4 b .. + 3 (DofMap, abd_reduce.hpp:11-27).
struct Bodies {
    std::vector<Real> q, q_tilde, reduced_mass, kappa, volume;  // 12, 12, 144, 1, 1 per body
    std::size_t size() const { return kappa.size(); }
};

// IncrementalPotential::assemble for inertia + solid meshes + affine bodies,
// up to (not including) assemble_contact / filter_pinned / sort / reduce:
// returns the value, fills grad (3 (n + 4 nb), zeroed on pinned slots,
// :253-254) and the triplet stream in emission order (:170-249): inertia
// diagonals of every vertex, body inertia tiles (split_sym_12x12 of the
// reduced mass), 10 blocks per tet, body orthogonality tiles.
inline Real ip_fem_assemble(const std::vector<Vec3>& x, const std::vector<Vec3>& x_tilde, const std::vector<Real>& mass,
                            const FemSolids& fs, Real dt2, const std::vector<char>& pinned, std::vector<Real>& grad,
                            BlockTripletStream& stream, bool project = true, const Bodies* bodies = nullptr,
                            const FemShells* shells = nullptr, const std::vector<int>* mesh_kind = nullptr) {
    const std::size_t n = x.size();
    const std::size_t nb = bodies ? bodies->size() : 0;
    grad.assign(3 * (n + 4 * nb), 0.0);
    stream.keys.clear();
    stream.values.clear();
    Real val = 0;
    for (std::size_t v = 0; v < n; ++v) {  // :170-180
        Vec3 dx;
        for (int k = 0; k < 3; ++k) dx[k] = x[v][k] - x_tilde[v][k];
        val += 0.5 * mass[v] * (dx[0] * dx[0] + dx[1] * dx[1] + dx[2] * dx[2]);
        for (int k = 0; k < 3; ++k) grad[3 * v + k] += mass[v] * dx[k];
        Mat3 m;
        m(0, 0) = m(1, 1) = m(2, 2) = mass[v];
        stream.emit(static_cast<Index>(v), static_cast<Index>(v), m);
    }
    auto split_sym = [&](Index base, const Real* H) {  // block_split.hpp:19-23
        for (int ti = 0; ti < 4; ++ti)
            for (int tj = ti; tj < 4; ++tj) {
                Mat3 blk;
                for (int c = 0; c < 3; ++c)
                    for (int r = 0; r < 3; ++r) blk(r, c) = H[12 * (3 * tj + c) + 3 * ti + r];
                stream.emit(base + ti, base + tj, blk);
            }
    };
    for (std::size_t b = 0; b < nb; ++b) {  // :181-188
        const Index base = static_cast<Index>(n + 4 * b);
        const Real* M = &bodies->reduced_mass[144 * b];
        Real dq[12], g[12];
        for (int k = 0; k < 12; ++k) dq[k] = bodies->q[12 * b + k] - bodies->q_tilde[12 * b + k];
        Real dg = 0;
        for (int i = 0; i < 12; ++i) {
            Real s2 = 0;
            for (int k = 0; k < 12; ++k) s2 += M[12 * k + i] * dq[k];
            g[i] = s2;
        }
        for (int k = 0; k < 12; ++k) dg += dq[k] * g[k];
        val += 0.5 * dg;
        for (int k = 0; k < 12; ++k) grad[3 * base + k] += g[k];
        split_sym(base, M);
    }
    const std::size_t nt = fs.rest.size();
    std::vector<Stencil12> st(nt);
    std::vector<Real> tet_mu(nt), tet_lam(nt);
    for (std::size_t m = 0; m + 1 < fs.tet_begin.size(); ++m)
        for (std::int64_t t = fs.tet_begin[m]; t < fs.tet_begin[m + 1]; ++t) {
            tet_mu[t] = fs.mu[m];
            tet_lam[t] = fs.lam[m];
        }
#pragma omp parallel for schedule(static)
    for (std::int64_t t = 0; t < static_cast<std::int64_t>(nt); ++t) {  // :223-232 (parallel_for)
        const std::int32_t* te = &fs.tets[4 * t];
        st[t] = stable_neo_hookean(x[te[0]], x[te[1]], x[te[2]], x[te[3]], fs.rest[t], tet_mu[t], tet_lam[t], project);
    }
    auto scatter = [&](const std::int32_t* ids, int nn, Real value, const Real* g, const Real* H) {  // scatter9 / 12
        const int ld = 3 * nn;
        val += dt2 * value;
        for (int a = 0; a < nn; ++a)
            for (int k = 0; k < 3; ++k) grad[3 * ids[a] + k] += dt2 * g[3 * a + k];
        for (int a = 0; a < nn; ++a)
            for (int b = a; b < nn; ++b) {
                Mat3 blk;
                for (int c = 0; c < 3; ++c)
                    for (int r = 0; r < 3; ++r) blk(r, c) = dt2 * H[ld * (3 * b + c) + 3 * a + r];
                stream.emit(ids[a], ids[b], blk);
            }
    };
    auto solid_mesh = [&](std::size_t m) {  // :222-239
        for (std::int64_t t = fs.tet_begin[m]; t < fs.tet_begin[m + 1]; ++t)
            scatter(&fs.tets[4 * t], 4, st[t].value, st[t].grad, st[t].hess);
    };
    auto shell_mesh = [&](std::size_t m) {  // :190-221: triangles (scatter9), then hinges (scatter12)
        const FemShells& sh = *shells;
        for (std::int64_t t = sh.tri_begin[m]; t < sh.tri_begin[m + 1]; ++t) {
            const std::int32_t* tr = &sh.tris[3 * t];
            const Stencil9 s9 = membrane_stencil(x[tr[0]], x[tr[1]], x[tr[2]], sh.tri_rest[t], sh.material[m], project);
            scatter(tr, 3, s9.value, s9.grad, s9.hess);
        }
        for (std::int64_t h = sh.hinge_begin[m]; h < sh.hinge_begin[m + 1]; ++h) {
            const std::int32_t* hg = &sh.hinges[4 * h];
            const Stencil12 s12 = hinge_bending(x[hg[0]], x[hg[1]], x[hg[2]], x[hg[3]], sh.hinge_rest[h],
                                                sh.material[m].bending, project);
            scatter(hg, 4, s12.value, s12.grad, s12.hess);
        }
    };
    if (!mesh_kind) {
        for (std::size_t m = 0; m + 1 < fs.tet_begin.size(); ++m) solid_mesh(m);
    } else {
        std::size_t si = 0, hi = 0;
        for (int kind : *mesh_kind) {
            if (kind == 0)
                solid_mesh(si++);
            else
                shell_mesh(hi++);
        }
    }
    for (std::size_t b = 0; b < nb; ++b) {  // :242-249
        const Index base = static_cast<Index>(n + 4 * b);
        const Stencil12 st = abd_orthogonality(&bodies->q[12 * b], bodies->kappa[b], bodies->volume[b], project);
        val += dt2 * st.value;
        for (int k = 0; k < 12; ++k) grad[3 * base + k] += dt2 * st.grad[k];
        Real H[144];
        for (int k = 0; k < 144; ++k) H[k] = dt2 * st.hess[k];
        split_sym(base, H);
    }
    for (std::size_t v = 0; v < n + 4 * nb && v < pinned.size(); ++v)
        if (pinned[v])
            for (int k = 0; k < 3; ++k) grad[3 * v + k] = 0;
    return val;
}


}  // namespace oracle
