// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// extern "C" surface over the REFERENCE's own hot-path headers, compiled in
// place from /root/reference/proj/include (nothing copied) against the Eigen
// subset in oracle/eigen_shim, into oracle/_ref/libadipc_ref.so. Every entry
// has the signature of the oracle_* entry of the same suffix in
// oracle_capi.cpp, so oracle_py can drive either library with one set of
// wrappers (oracle_py.use_backend("reference")). Used only to pin the
// restatement (tests/test_oracle_vs_reference.py) and as bench.py's
// "reference" CPU arm; never by the product.
//
// Not exposed: ip_fem_assemble (IncrementalPotential::assemble, whose header
// drags in the contact stack; its element stencils ARE exposed: tet_rest,
// stable_neo_hookean, project_psd), filter_pinned (a private member of IncrementalPotential,
// solver/incremental_potential.hpp:410, whose header drags in the contact and
// energy stack) and the MAS shift count (the reference does not record it).
#include <cstring>
#include <random>
#include <sstream>
#include <stdexcept>
#include <string>

#include <Eigen/Cholesky>  // scene/mesh.hpp (pulled in by friction.hpp) uses LLT

#include "adipc/contact/barrier.hpp"
#include "adipc/contact/friction.hpp"
#include "adipc/solver/incremental_potential.hpp"
#include "adipc/energy/abd_energy.hpp"
#include "adipc/energy/bending.hpp"
#include "adipc/energy/membrane.hpp"
#include "adipc/energy/neo_hookean.hpp"
#include "adipc/energy/psd.hpp"
#include "adipc/precond/block_jacobi.hpp"
#include "adipc/precond/hierarchy.hpp"
#include "adipc/precond/mas.hpp"
#include "adipc/precond/partition.hpp"
#include "adipc/solver/pcg.hpp"
#include "adipc/sparse/abd_reduce.hpp"
#include "adipc/sparse/block_coo.hpp"
#include "adipc/sparse/block_split.hpp"
#include "adipc/sparse/reduction.hpp"
#include "adipc/sparse/srbk_spmv.hpp"

using namespace adipc;

namespace {

thread_local std::string g_err;

ExecPolicy make_pol(int det, int threads, int lane_width) {
    ExecPolicy p;
    p.deterministic = det != 0;
    p.threads = threads;
    p.lane_width = lane_width > 0 ? lane_width : 32;
    return p;
}

Mat3 load_mat3(const double* p) {
    Mat3 m;
    std::memcpy(m.data(), p, 72);
    return m;
}

BlockTripletStream load_stream(const std::uint64_t* keys, const double* vals, std::size_t T) {
    BlockTripletStream s;
    s.keys.assign(keys, keys + T);
    s.values.resize(T);
    for (std::size_t i = 0; i < T; ++i) s.values[i] = load_mat3(vals + 9 * i);
    return s;
}

void store_stream(const BlockTripletStream& s, std::uint64_t* keys, double* vals) {
    for (std::size_t i = 0; i < s.size(); ++i) {
        keys[i] = s.keys[i];
        std::memcpy(vals + 9 * i, s.values[i].data(), 72);
    }
}

SortedSymBlockCoo load_matrix(std::int32_t n_block_rows, std::size_t U, const std::uint32_t* rows,
                              const std::uint32_t* cols, const double* blocks) {
    SortedSymBlockCoo A;
    A.n_block_rows = n_block_rows;
    A.rows.assign(rows, rows + U);
    A.cols.assign(cols, cols + U);
    A.blocks.resize(U);
    for (std::size_t i = 0; i < U; ++i) A.blocks[i] = load_mat3(blocks + 9 * i);
    return A;
}

std::vector<std::pair<Index, Index>> load_edges(const std::int32_t* pairs, std::size_t n) {
    std::vector<std::pair<Index, Index>> e(n);
    for (std::size_t i = 0; i < n; ++i) e[i] = {pairs[2 * i], pairs[2 * i + 1]};
    return e;
}

VecX load_vec(const double* p, std::size_t n) {
    VecX v(static_cast<int>(n));
    if (n) std::memcpy(v.data(), p, n * 8);
    return v;
}

template <class V, int W>
int segment_reduce_w(const std::vector<Index>& o, const double* Vp, std::size_t nV, std::int32_t n_segments,
                     const ExecPolicy& pol, double* R) {
    std::vector<V> v(nV);
    for (std::size_t i = 0; i < nV; ++i) std::memcpy(v[i].data(), Vp + W * i, W * 8);
    auto r = fast_segment_reduction(o, v, n_segments, pol);
    for (std::size_t i = 0; i < r.size(); ++i) std::memcpy(R + W * i, r[i].data(), W * 8);
    return 0;
}

struct RefMatrix {
    SortedSymBlockCoo A;
};

struct RefMas {
    MasPreconditioner M;
};

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
int ref_max_threads() { return process_thread_default(); }
void ref_set_default_threads(int n) {
    if (n > 0) set_default_threads(n);
}

std::uint64_t ref_make_block_key(std::uint32_t r, std::uint32_t c) { return make_block_key(r, c); }

std::uint64_t ref_emit(std::int32_t r, std::int32_t c, const double* m9, double* out9) {
    BlockTripletStream s;
    s.emit(r, c, load_mat3(m9));
    std::memcpy(out9, s.values[0].data(), 72);
    return s.keys[0];
}

void ref_radix_sort_keys(std::uint64_t* keys, std::uint32_t* perm, std::size_t T) {
    std::vector<std::uint64_t> k(keys, keys + T);
    std::vector<std::uint32_t> p;
    detail::radix_sort_keys(k, p);
    if (T) {
        std::memcpy(keys, k.data(), T * 8);
        std::memcpy(perm, p.data(), T * 4);
    }
}

void ref_sort_stream(std::uint64_t* keys, double* vals, std::size_t T, int det, int threads, int lw) {
    BlockTripletStream s = load_stream(keys, vals, T);
    sort_stream(s, make_pol(det, threads, lw));
    store_stream(s, keys, vals);
}

std::int64_t ref_fast_hash_reduction(const std::uint64_t* keys, const double* vals, std::size_t T,
                                     std::int32_t n_block_rows, int det, int threads, int lw, std::uint32_t* rows,
                                     std::uint32_t* cols, double* blocks) {
    const BlockTripletStream s = load_stream(keys, vals, T);
    const SortedSymBlockCoo A = fast_hash_reduction(s, n_block_rows, make_pol(det, threads, lw));
    for (std::size_t i = 0; i < A.size(); ++i) {
        rows[i] = A.rows[i];
        cols[i] = A.cols[i];
        std::memcpy(blocks + 9 * i, A.blocks[i].data(), 72);
    }
    return static_cast<std::int64_t>(A.size());
}

int ref_segment_reduce(const std::int32_t* O, std::size_t nO, const double* V, std::size_t nV, int width,
                       std::int32_t n_segments, int det, int threads, int lw, double* R) {
    const ExecPolicy pol = make_pol(det, threads, lw);
    const std::vector<Index> o(O, O + nO);
    try {
        if (width == 1) {
            std::vector<Real> v(V, V + nV);
            auto r = fast_segment_reduction(o, v, n_segments, pol);
            if (!r.empty()) std::memcpy(R, r.data(), r.size() * 8);
            return 0;
        }
        if (width == 3) return segment_reduce_w<Vec3, 3>(o, V, nV, n_segments, pol, R);
        if (width == 9) return segment_reduce_w<Mat3, 9>(o, V, nV, n_segments, pol, R);
        g_err = "width must be 1, 3 or 9";
        return 1;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    }
}

void ref_srbk_spmv(std::int32_t n_block_rows, std::size_t U, const std::uint32_t* rows, const std::uint32_t* cols,
                   const double* blocks, const double* x, std::size_t nx, int det, int threads, int lw, double* y) {
    const SortedSymBlockCoo A = load_matrix(n_block_rows, U, rows, cols, blocks);
    std::vector<Vec3> xv(nx);
    for (std::size_t i = 0; i < nx; ++i) std::memcpy(xv[i].data(), x + 3 * i, 24);
    const auto yv = srbk_spmv(A, xv, make_pol(det, threads, lw));
    for (std::size_t i = 0; i < nx; ++i) std::memcpy(y + 3 * i, yv[i].data(), 24);
}

// dump_block_coo (srbk_spmv.hpp:52-60) into `out` (cap bytes); returns the text length
std::int64_t ref_dump_block_coo(std::int32_t n_block_rows, std::size_t U, const std::uint32_t* rows,
                                const std::uint32_t* cols, const double* blocks, char* out, std::size_t cap) {
    const SortedSymBlockCoo A = load_matrix(n_block_rows, U, rows, cols, blocks);
    std::ostringstream os;
    dump_block_coo(A, os);
    const std::string t = os.str();
    if (out && cap >= t.size()) std::memcpy(out, t.data(), t.size());
    return static_cast<std::int64_t>(t.size());
}

int ref_split(int kind, std::int32_t rb, std::int32_t cb, const double* H, std::uint64_t* keys, double* vals) {
    BlockTripletStream out;
    if (kind == 0 || kind == 1) {
        Mat12 m;
        std::memcpy(m.data(), H, 144 * 8);
        if (kind == 0)
            split_12x12(rb, cb, m, out);
        else
            split_sym_12x12(rb, m, out);
    } else if (kind == 2) {
        Mat12x3 m;
        std::memcpy(m.data(), H, 36 * 8);
        split_12x3(rb, cb, m, out);
    } else {
        Mat3x12 m;
        std::memcpy(m.data(), H, 36 * 8);
        split_3x12(rb, cb, m, out);
    }
    store_stream(out, keys, vals);
    return static_cast<int>(out.size());
}

std::int64_t ref_two_level_abd_reduce(const std::uint64_t* keys, const double* vals, std::size_t Tn,
                                      std::int32_t n_fem, std::int32_t n_bodies, std::size_t n_abd,
                                      const std::int32_t* abd_node_body, const double* jac36, int det, int threads,
                                      int lw, std::uint64_t* out_keys, double* out_vals) {
    const BlockTripletStream s = load_stream(keys, vals, Tn);
    DofMap m;
    m.n_fem_nodes = n_fem;
    m.n_bodies = n_bodies;
    m.abd_node_body.assign(abd_node_body, abd_node_body + n_abd);
    m.abd_node_jacobian.resize(n_abd);
    for (std::size_t i = 0; i < n_abd; ++i) std::memcpy(m.abd_node_jacobian[i].data(), jac36 + 36 * i, 36 * 8);
    const BlockTripletStream t = two_level_abd_reduce(s, m, make_pol(det, threads, lw));
    store_stream(t, out_keys, out_vals);
    return static_cast<std::int64_t>(t.size());
}

std::int64_t ref_filter_pinned(const std::uint64_t*, const double*, std::size_t, const std::uint8_t*, std::int32_t,
                               std::uint64_t*, double*) {
    g_err = "filter_pinned is private to IncrementalPotential in the reference";
    return -1;
}


// ---- element-Hessian producer: energy/neo_hookean.hpp + energy/psd.hpp (the
// reference's own code; psd.hpp's eigen-solver is the shim's, sym_eig.hpp) ----
static Vec3 ld3(const double* p) { return Vec3(p[0], p[1], p[2]); }

int ref_tet_rest(const double* p12, double* inv9, double* vol) {
    try {
        const TetRest r = tet_rest(ld3(p12), ld3(p12 + 3), ld3(p12 + 6), ld3(p12 + 9));
        std::memcpy(inv9, r.inv_rest_edges.data(), 72);
        *vol = r.volume;
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

void ref_stable_neo_hookean(const double* x12, const double* inv9, double vol, double mu, double lam, int project,
                            double* value, double* grad12, double* hess144) {
    TetRest r;
    r.inv_rest_edges = load_mat3(inv9);
    r.volume = vol;
    const Stencil12 s = stable_neo_hookean(ld3(x12), ld3(x12 + 3), ld3(x12 + 6), ld3(x12 + 9), r, mu, lam, project != 0);
    *value = s.value;
    std::memcpy(grad12, s.grad.data(), 96);
    std::memcpy(hess144, s.hess.data(), 144 * 8);
}

void ref_abd_orthogonality(const double* q12, double kappa, double volume, int project, double* value,
                           double* grad12, double* hess144) {
    Vec12 q;
    std::memcpy(q.data(), q12, 96);
    const Stencil12 s = abd_orthogonality(q, kappa, volume, project != 0);
    *value = s.value;
    std::memcpy(grad12, s.grad.data(), 96);
    std::memcpy(hess144, s.hess.data(), 1152);
}

int ref_membrane_rest(const double* p9, double* rest5) {
    try {
        const MembraneRest r = membrane_rest(ld3(p9), ld3(p9 + 3), ld3(p9 + 6));
        std::memcpy(rest5, r.inv_rest_edges.data(), 32);
        rest5[4] = r.area;
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}
// IncrementalPotential::membrane_stencil (incremental_potential.hpp:273-298,
// a private member) composed from the reference's own membrane.hpp functions
// in its exact sequence
void ref_membrane_stencil(const double* x9, const double* rest5, const double* material5, int project, double* value,
                          double* grad9, double* hess81) {
    Mat2 inv;
    std::memcpy(inv.data(), rest5, 32);
    const Mat3x2 F = membrane_deformation(ld3(x9), ld3(x9 + 3), ld3(x9 + 6), inv);
    const Real a_t = rest5[4] * material5[0];
    MembraneDerivs d = fbw_membrane(F, material5[1], a_t, project != 0);
    const MembraneDerivs lim = cubic_strain_limit(F, material5[2], a_t);
    const MembraneDerivs sh = shear_energy(F, material5[3] * material5[1], a_t, project != 0);
    d.value += lim.value + sh.value;
    d.dF += lim.dF + sh.dF;
    d.hess += lim.hess + sh.hess;
    const Eigen::Matrix<Real, 6, 9> J = membrane_dFdx(inv);
    const Mat3x2& dF = d.dF;
    Vec6 g6;
    g6 << dF.col(0), dF.col(1);
    *value = d.value;
    const Vec9 g = J.transpose() * g6;
    const Mat9 H = J.transpose() * d.hess * J;
    std::memcpy(grad9, g.data(), 72);
    std::memcpy(hess81, H.data(), 648);
}
int ref_hinge_rest(const double* p12, double* rest2) {
    try {
        const HingeRest r = hinge_rest(ld3(p12), ld3(p12 + 3), ld3(p12 + 6), ld3(p12 + 9));
        rest2[0] = r.rest_angle;
        rest2[1] = r.weight;
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}
void ref_hinge_bending(const double* x12, const double* rest2, double k, int project, double* value, double* grad12,
                       double* hess144) {
    HingeRest r;
    r.rest_angle = rest2[0];
    r.weight = rest2[1];
    const Stencil12 s = hinge_bending(ld3(x12), ld3(x12 + 3), ld3(x12 + 6), ld3(x12 + 9), r, k, project != 0);
    *value = s.value;
    std::memcpy(grad12, s.grad.data(), 96);
    std::memcpy(hess144, s.hess.data(), 1152);
}

void ref_project_psd(int n, const double* M, double* out) {
    MatX m(n, n);
    std::memcpy(m.data(), M, sizeof(double) * n * n);
    const MatX p = project_psd(m);
    std::memcpy(out, p.data(), sizeof(double) * n * n);
}


// ---- contact stencils: contact/distance.hpp + contact/barrier.hpp --------------
static void store_pair(const PairDerivs& pd, double* d2, double* g12, double* h144) {
    *d2 = pd.dist2;
    std::memcpy(g12, pd.grad.data(), 96);
    std::memcpy(h144, pd.hess.data(), 1152);
}
void ref_pt_dist2_derivs(const double* x12, double* d2, double* g12, double* h144) {
    store_pair(pt_dist2_derivs(ld3(x12), ld3(x12 + 3), ld3(x12 + 6), ld3(x12 + 9)), d2, g12, h144);
}
void ref_ee_dist2_derivs(const double* x12, double* d2, double* g12, double* h144) {
    store_pair(ee_dist2_derivs(ld3(x12), ld3(x12 + 3), ld3(x12 + 6), ld3(x12 + 9)), d2, g12, h144);
}
double ref_pt_dist2(const double* x12) { return pt_dist2(ld3(x12), ld3(x12 + 3), ld3(x12 + 6), ld3(x12 + 9)); }
double ref_ee_dist2(const double* x12) { return ee_dist2(ld3(x12), ld3(x12 + 3), ld3(x12 + 6), ld3(x12 + 9)); }
void ref_barrier_pair_derivs(double d2, const double* g12, const double* h144, double shat, double kappa, int project,
                             double* value, double* og12, double* oh144) {
    PairDerivs pd;
    pd.dist2 = d2;
    std::memcpy(pd.grad.data(), g12, 96);
    std::memcpy(pd.hess.data(), h144, 1152);
    const BarrierDerivs b = barrier_pair_derivs(pd, shat, kappa, project != 0);
    *value = b.value;
    std::memcpy(og12, b.grad.data(), 96);
    std::memcpy(oh144, b.hess.data(), 1152);
}
void ref_ground_barrier_derivs(const double* x3, const double* n3, double height, double dhat, double kappa,
                               int project, double* value, double* g3, double* h9, double* dist) {
    const GroundDerivs gd = ground_barrier_derivs(ld3(x3), ld3(n3), height, dhat, kappa, project != 0);
    *value = gd.value;
    std::memcpy(g3, gd.grad.data(), 24);
    std::memcpy(h9, gd.hess.data(), 72);
    *dist = gd.dist;
}

std::int32_t ref_subdomain_count(std::int32_t v, std::int32_t n, std::int32_t n_o) { return subdomain_count(v, n, n_o); }

std::int32_t ref_chunk_partition(std::int32_t v, std::int32_t cap, std::int32_t* part_of) {
    const Partition p = chunk_partition(v, cap);
    if (v) std::memcpy(part_of, p.part_of.data(), v * 4);
    return p.n_parts;
}

std::int32_t ref_partition_block_graph(std::int32_t v, const std::int32_t* pairs, std::size_t n_edges,
                                       std::int32_t cap, std::int32_t* part_of) {
    const Partition p = partition_block_graph(v, load_edges(pairs, n_edges), cap);
    if (v) std::memcpy(part_of, p.part_of.data(), v * 4);
    return p.n_parts;
}

std::int64_t ref_block_edges(std::size_t U, const std::uint32_t* rows, const std::uint32_t* cols,
                             std::int32_t* pairs) {
    SortedSymBlockCoo A;
    A.rows.assign(rows, rows + U);
    A.cols.assign(cols, cols + U);
    const auto e = block_edges(A);
    for (std::size_t i = 0; i < e.size(); ++i) {
        pairs[2 * i] = e[i].first;
        pairs[2 * i + 1] = e[i].second;
    }
    return static_cast<std::int64_t>(e.size());
}

void* ref_build_hierarchy(const std::int32_t* part_of, std::int32_t n_slots, std::int32_t n_parts,
                          std::int32_t capacity, const std::int32_t* pairs, std::size_t n_edges, int max_levels) {
    Partition l0;
    l0.part_of.assign(part_of, part_of + n_slots);
    l0.n_parts = n_parts;
    l0.capacity = capacity;
    return new MasHierarchy(build_hierarchy(l0, load_edges(pairs, n_edges), max_levels));
}
void ref_hierarchy_free(void* h) { delete static_cast<MasHierarchy*>(h); }
int ref_hierarchy_n_levels(void* h) { return static_cast<MasHierarchy*>(h)->n_levels(); }
void ref_hierarchy_level(void* hp, int l, std::int32_t* n_nodes, std::int32_t* n_parts, std::int32_t* part_of,
                         std::int32_t* agg) {
    const auto& L = static_cast<MasHierarchy*>(hp)->levels[l];
    *n_nodes = L.n_nodes;
    *n_parts = L.n_parts;
    if (part_of && L.n_nodes) std::memcpy(part_of, L.part_of.data(), L.n_nodes * 4);
    if (agg && !L.agg.empty()) std::memcpy(agg, L.agg.data(), L.agg.size() * 4);
}

void* ref_matrix_new(std::int32_t n_block_rows, std::size_t U, const std::uint32_t* rows, const std::uint32_t* cols,
                     const double* blocks) {
    return new RefMatrix{load_matrix(n_block_rows, U, rows, cols, blocks)};
}
void ref_matrix_free(void* m) { delete static_cast<RefMatrix*>(m); }

void* ref_mas_build(void* mat, void* hier) {
    auto* M = new MasPreconditioner();
    try {
        M->build(static_cast<RefMatrix*>(mat)->A, *static_cast<MasHierarchy*>(hier));
    } catch (const std::runtime_error& e) {
        g_err = e.what();
        delete M;
        return nullptr;
    }
    return static_cast<Preconditioner*>(M);
}
void ref_precond_free(void* p) { delete static_cast<Preconditioner*>(p); }
long ref_mas_shifts(void*) { return -1; }
int ref_mas_n_levels(void* p) { return static_cast<MasPreconditioner*>(static_cast<Preconditioner*>(p))->n_levels(); }
int ref_mas_level_matrix(void* p, int l, std::int32_t s, double* out) {
    const auto* M = static_cast<MasPreconditioner*>(static_cast<Preconditioner*>(p));
    const MatX& D = M->level_matrices(l)[s];
    if (out) std::memcpy(out, D.data(), D.size() * 8);
    return D.rows();
}

void* ref_jacobi_build(void* mat) {
    auto* J = new BlockJacobiPreconditioner();
    J->build(static_cast<RefMatrix*>(mat)->A);
    return static_cast<Preconditioner*>(J);
}

void ref_precond_apply(void* p, const double* r, std::size_t n, double* z) {
    const VecX rv = load_vec(r, n);
    VecX zv;
    static_cast<Preconditioner*>(p)->apply(rv, zv);
    std::memcpy(z, zv.data(), n * 8);
}

int ref_pcg_solve(void* mat, const double* b, std::size_t n, void* precond, double rel_tol, int restart,
                  int max_iters, int det, int threads, int lw, double* x, int* iters, double* rel_residual,
                  int* converged) {
    const VecX bv = load_vec(b, n);
    VecX xv;
    const PcgResult r = pcg_solve(static_cast<RefMatrix*>(mat)->A, bv, *static_cast<Preconditioner*>(precond),
                                  rel_tol, restart, max_iters, make_pol(det, threads, lw), xv);
    std::memcpy(x, xv.data(), n * 8);
    *iters = r.iters;
    *rel_residual = r.rel_residual;
    *converged = r.converged ? 1 : 0;
    return 0;
}

}  // extern "C"


extern "C" {
// ---- broad phase, contact frames, friction constraints: contact/broad_phase.hpp,
// distance.hpp:226-256, friction.hpp:43-149 (the scene headers they include
// compile against the Eigen subset) ------------------------------------------------
static ContactSurface ref_surface(std::int32_t n_verts, const std::int32_t* verts, std::int32_t n_edges,
                                  const std::int32_t* edges, std::int32_t n_tris, const std::int32_t* tris) {
    ContactSurface s;
    s.verts.assign(verts, verts + n_verts);
    for (std::int32_t e = 0; e < n_edges; ++e) s.edges.push_back({edges[2 * e], edges[2 * e + 1]});
    for (std::int32_t t = 0; t < n_tris; ++t) s.tris.push_back({tris[3 * t], tris[3 * t + 1], tris[3 * t + 2]});
    return s;
}
std::int64_t ref_find_candidates(std::int32_t n_nodes, const double* pos, const double* disp, std::int32_t n_verts,
                                 const std::int32_t* verts, std::int32_t n_edges, const std::int32_t* edges,
                                 std::int32_t n_tris, const std::int32_t* tris, double inflate, std::int32_t* pt_out,
                                 std::int64_t pt_cap, std::int32_t* ee_out, std::int64_t ee_cap,
                                 std::int64_t* n_ee_out) {
    std::vector<Vec3> p(n_nodes), d;
    for (std::int32_t v = 0; v < n_nodes; ++v) p[v] = ld3(pos + 3 * v);
    if (disp) {
        d.resize(n_nodes);
        for (std::int32_t v = 0; v < n_nodes; ++v) d[v] = ld3(disp + 3 * v);
    }
    const ContactSurface s = ref_surface(n_verts, verts, n_edges, edges, n_tris, tris);
    const ContactCandidates c = find_candidates(s, p, disp ? &d : nullptr, inflate);
    *n_ee_out = static_cast<std::int64_t>(c.ee.size());
    if (static_cast<std::int64_t>(c.pt.size()) > pt_cap || static_cast<std::int64_t>(c.ee.size()) > ee_cap) return -1;
    for (std::size_t i = 0; i < c.pt.size(); ++i) {
        pt_out[2 * i] = c.pt[i][0];
        pt_out[2 * i + 1] = c.pt[i][1];
    }
    for (std::size_t i = 0; i < c.ee.size(); ++i) {
        ee_out[2 * i] = c.ee[i][0];
        ee_out[2 * i + 1] = c.ee[i][1];
    }
    return static_cast<std::int64_t>(c.pt.size());
}
static void store_frame(const ContactFrame& f, double* dist, double* normal3, double* coeff4) {
    *dist = f.dist;
    for (int a = 0; a < 3; ++a) normal3[a] = f.normal[a];
    for (int k = 0; k < 4; ++k) coeff4[k] = f.coeff[k];
}
void ref_pt_contact_frame(const double* x12, double* dist, double* normal3, double* coeff4) {
    store_frame(pt_contact_frame(ld3(x12), ld3(x12 + 3), ld3(x12 + 6), ld3(x12 + 9)), dist, normal3, coeff4);
}
void ref_ee_contact_frame(const double* x12, double* dist, double* normal3, double* coeff4) {
    store_frame(ee_contact_frame(ld3(x12), ld3(x12 + 3), ld3(x12 + 6), ld3(x12 + 9)), dist, normal3, coeff4);
}
void ref_tangent_basis(const double* n3, double* t1, double* t2) {
    Vec3 a, b;
    tangent_basis(ld3(n3), a, b);
    for (int k = 0; k < 3; ++k) {
        t1[k] = a[k];
        t2[k] = b[k];
    }
}
// build_friction_constraints with its own proximity broad phase (friction.hpp:95-149)
std::int64_t ref_build_friction_constraints(std::int32_t n_nodes, const double* pos, std::int32_t n_verts,
                                           const std::int32_t* verts, std::int32_t n_edges, const std::int32_t* edges,
                                           std::int32_t n_tris, const std::int32_t* tris, int ground,
                                           const double* normal, double height, double dhat, double kappa,
                                           std::int64_t cap, std::int32_t* nodes4, std::int32_t* n_nodes_out,
                                           double* coeff4, double* t1, double* t2, double* lambda) {
    std::vector<Vec3> p(n_nodes);
    for (std::int32_t v = 0; v < n_nodes; ++v) p[v] = ld3(pos + 3 * v);
    const ContactSurface s = ref_surface(n_verts, verts, n_edges, edges, n_tris, tris);
    GroundPlane g;
    g.enabled = ground != 0;
    if (g.enabled) {
        g.normal = ld3(normal);
        g.height = height;
    }
    const std::vector<FrictionConstraint> fc = build_friction_constraints(s, p, g, dhat, kappa);
    if (static_cast<std::int64_t>(fc.size()) > cap) return -static_cast<std::int64_t>(fc.size()) - 1;
    for (std::size_t i = 0; i < fc.size(); ++i) {
        for (int k = 0; k < 4; ++k) {
            nodes4[4 * i + k] = fc[i].nodes[k];
            coeff4[4 * i + k] = fc[i].coeff[k];
        }
        n_nodes_out[i] = fc[i].n_nodes;
        for (int k = 0; k < 3; ++k) {
            t1[3 * i + k] = fc[i].t1[k];
            t2[3 * i + k] = fc[i].t2[k];
        }
        lambda[i] = fc[i].lambda;
    }
    return static_cast<std::int64_t>(fc.size());
}

// ---- the reference's IncrementalPotential::assemble on a scene built from
// arrays (scene/scene.hpp Scene::finalize, make_dof_map, broad_phase.hpp
// build_contact_surface; solver/incremental_potential.hpp:19-258), and the
// scene data it derives, exported so the device path runs on identical inputs
struct RefScene {
    Scene scene;
    ContactSurface surf;
    DofMap dofs;
    std::vector<FrictionConstraint> friction;
    std::vector<Vec3> fr_base;
    Real mu = 0, fr_eps = 1;
};
void* ref_scene_new(std::int32_t n_meshes, const std::int64_t* vert_begin, const double* rest,
                    const std::int64_t* tet_begin, const std::int32_t* tets, const double* youngs,
                    const double* poisson, const double* density, std::int32_t n_bodies,
                    const std::int64_t* bvert_begin, const double* brest, const std::int64_t* btet_begin,
                    const std::int32_t* btets, const double* bkappa, const double* bdensity, double dt, int ground,
                    const double* gnormal, double gheight, std::int32_t n_shells, const std::int64_t* svert_begin,
                    const double* srest, const std::int64_t* stri_begin, const std::int32_t* stris,
                    const double* smat6) {
    auto* r = new RefScene;
    Scene& sc = r->scene;
    sc.config.dt = dt;
    sc.ground.enabled = ground != 0;
    if (ground) {
        sc.ground.normal = ld3(gnormal);
        sc.ground.height = gheight;
    }
    for (std::int32_t m = 0; m < n_meshes; ++m) {
        DeformableMesh dm;
        dm.name = "mesh" + std::to_string(m);
        for (std::int64_t v = vert_begin[m]; v < vert_begin[m + 1]; ++v) dm.rest.push_back(ld3(rest + 3 * v));
        for (std::int64_t t = tet_begin[m]; t < tet_begin[m + 1]; ++t)
            dm.tets.push_back({tets[4 * t], tets[4 * t + 1], tets[4 * t + 2], tets[4 * t + 3]});
        dm.solid.youngs = youngs[m];
        dm.solid.poisson = poisson[m];
        dm.solid.density = density[m];
        sc.meshes.push_back(std::move(dm));
    }
    for (std::int32_t m = 0; m < n_shells; ++m) {  // shells after the solids (mesh order)
        DeformableMesh dm;
        dm.name = "shell" + std::to_string(m);
        dm.is_shell = true;
        for (std::int64_t v = svert_begin[m]; v < svert_begin[m + 1]; ++v) dm.rest.push_back(ld3(srest + 3 * v));
        for (std::int64_t t = stri_begin[m]; t < stri_begin[m + 1]; ++t)
            dm.tris.push_back({stris[3 * t], stris[3 * t + 1], stris[3 * t + 2]});
        const double* mt = smat6 + 6 * m;  // density, thickness, stretch, strain limit, shear fraction, bending
        dm.shell.density = mt[0];
        dm.shell.thickness = mt[1];
        dm.shell.stretch_stiffness = mt[2];
        dm.shell.strain_limit_stiffness = mt[3];
        dm.shell.shear_fraction = mt[4];
        dm.shell.bending_stiffness = mt[5];
        sc.meshes.push_back(std::move(dm));
    }
    for (std::int32_t b = 0; b < n_bodies; ++b) {
        AffineBody ab;
        ab.name = "body" + std::to_string(b);
        for (std::int64_t v = bvert_begin[b]; v < bvert_begin[b + 1]; ++v) ab.rest.push_back(ld3(brest + 3 * v));
        for (std::int64_t t = btet_begin[b]; t < btet_begin[b + 1]; ++t)
            ab.tets.push_back({btets[4 * t], btets[4 * t + 1], btets[4 * t + 2], btets[4 * t + 3]});
        ab.mat.kappa = bkappa[b];
        ab.mat.density = bdensity[b];
        sc.bodies.push_back(std::move(ab));
    }
    sc.finalize();
    r->surf = build_contact_surface(sc);
    r->dofs = make_dof_map(sc);
    return r;
}
void ref_scene_free(void* p) { delete static_cast<RefScene*>(p); }
// shell meshes' derived data (after the solids, mesh order): GLOBAL triangles
// and hinges, MembraneRest (Dm^-1 column-major 2x2, area), HingeRest (rest
// angle, weight), per-shell material (thickness, stretch, strain limit, shear
// fraction, bending) and per-shell triangle / hinge counts
void ref_scene_shell_sizes(void* p, std::int64_t* n_tris, std::int64_t* n_hinges) {
    const RefScene& r = *static_cast<RefScene*>(p);
    *n_tris = *n_hinges = 0;
    for (const auto& m : r.scene.meshes)
        if (m.is_shell) {
            *n_tris += static_cast<std::int64_t>(m.tris.size());
            *n_hinges += static_cast<std::int64_t>(m.hinges.size());
        }
}
void ref_scene_shell_export(void* p, std::int32_t* tris, double* tri_rest5, std::int32_t* hinges, double* hinge_rest2,
                            double* material5, std::int64_t* tri_count, std::int64_t* hinge_count) {
    const RefScene& r = *static_cast<RefScene*>(p);
    const Scene& sc = r.scene;
    std::int64_t t0 = 0, h0 = 0;
    int si = 0;
    for (std::size_t mi = 0; mi < sc.meshes.size(); ++mi) {
        const auto& m = sc.meshes[mi];
        if (!m.is_shell) continue;
        const Index off = sc.mesh_offset[mi];
        for (std::size_t t = 0; t < m.tris.size(); ++t, ++t0) {
            for (int k = 0; k < 3; ++k) tris[3 * t0 + k] = m.tris[t][k] + off;
            std::memcpy(tri_rest5 + 5 * t0, m.tri_rest_data[t].inv_rest_edges.data(), 32);
            tri_rest5[5 * t0 + 4] = m.tri_rest_data[t].area;
        }
        for (std::size_t h = 0; h < m.hinges.size(); ++h, ++h0) {
            for (int k = 0; k < 4; ++k) hinges[4 * h0 + k] = m.hinges[h][k] + off;
            hinge_rest2[2 * h0] = m.hinge_rest_data[h].rest_angle;
            hinge_rest2[2 * h0 + 1] = m.hinge_rest_data[h].weight;
        }
        material5[5 * si] = m.shell.thickness;
        material5[5 * si + 1] = m.shell.stretch_stiffness;
        material5[5 * si + 2] = m.shell.strain_limit_stiffness;
        material5[5 * si + 3] = m.shell.shear_fraction;
        material5[5 * si + 4] = m.shell.bending_stiffness;
        tri_count[si] = static_cast<std::int64_t>(m.tris.size());
        hinge_count[si] = static_cast<std::int64_t>(m.hinges.size());
        ++si;
    }
}
// sizes: n_fem, n_bodies, n_blocks, n_nodes, n_tets, n_surf_verts, n_edges, n_tris, n_meshes
void ref_scene_sizes(void* p, std::int64_t* out) {
    const RefScene& r = *static_cast<RefScene*>(p);
    std::int64_t nt = 0;
    for (const auto& m : r.scene.meshes) nt += static_cast<std::int64_t>(m.tets.size());
    out[0] = r.dofs.n_fem_nodes;
    out[1] = r.dofs.n_bodies;
    out[2] = r.dofs.n_blocks();
    out[3] = r.dofs.n_nodes();
    out[4] = nt;
    out[5] = static_cast<std::int64_t>(r.surf.verts.size());
    out[6] = static_cast<std::int64_t>(r.surf.edges.size());
    out[7] = static_cast<std::int64_t>(r.surf.tris.size());
    out[8] = static_cast<std::int64_t>(r.scene.meshes.size());
}
// the derived data: vertex masses, per-tet rest data (Dm^-1 column-major, volume) and GLOBAL
// tets, per-mesh mu / lambda, body reduced masses (column-major) / volumes, the abd node map and
// jacobians (column-major 3x12), the contact surface, the scene length
void ref_scene_export(void* p, double* mass, double* inv9, double* vol, std::int32_t* tets, double* mu, double* lam,
                      double* reduced_mass, double* body_volume, std::int32_t* abd_body, double* jac36,
                      std::int32_t* surf_verts, std::int32_t* edges, std::int32_t* tris, double* length_scale) {
    const RefScene& r = *static_cast<RefScene*>(p);
    const Scene& sc = r.scene;
    std::int64_t t0 = 0;
    for (std::size_t mi = 0; mi < sc.meshes.size(); ++mi) {
        const auto& m = sc.meshes[mi];
        const Index off = sc.mesh_offset[mi];
        for (Index v = 0; v < m.n_verts(); ++v) mass[off + v] = m.vertex_mass[v];
        if (m.is_shell) continue;
        for (std::size_t t = 0; t < m.tets.size(); ++t, ++t0) {
            std::memcpy(inv9 + 9 * t0, m.tet_rest_data[t].inv_rest_edges.data(), 72);
            vol[t0] = m.tet_rest_data[t].volume;
            for (int k = 0; k < 4; ++k) tets[4 * t0 + k] = m.tets[t][k] + off;
        }
        mu[mi] = m.solid.mu();
        lam[mi] = m.solid.lambda();
    }
    for (std::size_t b = 0; b < sc.bodies.size(); ++b) {
        std::memcpy(reduced_mass + 144 * b, sc.bodies[b].reduced_mass.data(), 144 * 8);
        body_volume[b] = sc.bodies[b].volume;
    }
    for (std::size_t a = 0; a < r.dofs.abd_node_body.size(); ++a) {
        abd_body[a] = r.dofs.abd_node_body[a];
        std::memcpy(jac36 + 36 * a, r.dofs.abd_node_jacobian[a].data(), 36 * 8);
    }
    for (std::size_t i = 0; i < r.surf.verts.size(); ++i) surf_verts[i] = r.surf.verts[i];
    for (std::size_t i = 0; i < r.surf.edges.size(); ++i) {
        edges[2 * i] = r.surf.edges[i][0];
        edges[2 * i + 1] = r.surf.edges[i][1];
    }
    for (std::size_t i = 0; i < r.surf.tris.size(); ++i)
        for (int k = 0; k < 3; ++k) tris[3 * i + k] = r.surf.tris[i][k];
    *length_scale = sc.length_scale;
}
static SystemState ref_state(const RefScene& r, const double* x, const double* q) {
    SystemState s;
    s.x.resize(r.dofs.n_fem_nodes);
    s.v.assign(r.dofs.n_fem_nodes, Vec3::Zero());
    for (Index v = 0; v < r.dofs.n_fem_nodes; ++v) s.x[v] = ld3(x + 3 * v);
    s.q.resize(r.dofs.n_bodies);
    s.qd.assign(r.dofs.n_bodies, Vec12::Zero());
    for (Index b = 0; b < r.dofs.n_bodies; ++b)
        for (int k = 0; k < 12; ++k) s.q[b][k] = q[12 * b + k];
    return s;
}
// the step-start friction freeze of newton.hpp:104-113 at state (x, q)
std::int64_t ref_scene_begin_friction(void* p, const double* x, const double* q, double dhat, double kappa, double mu,
                                      double eps) {
    RefScene& r = *static_cast<RefScene*>(p);
    const std::vector<Vec3> pos = contact_node_positions(r.scene, ref_state(r, x, q));
    r.friction = build_friction_constraints(r.surf, pos, r.scene.ground, dhat, kappa);
    r.fr_base = pos;
    r.mu = mu;
    r.fr_eps = eps;
    return static_cast<std::int64_t>(r.friction.size());
}
// IncrementalPotential::assemble (value, grad, reduced Hessian) at (x, q) with
// targets (x_tilde, q_tilde) and contact (dhat, kappa); returns U, or -U - 1
// when cap is too small
std::int64_t ref_scene_assemble(void* p, const double* x, const double* q, const double* x_tilde,
                                const double* q_tilde, double dhat, double kappa, int det, double* value,
                                double* grad, std::int64_t cap, std::uint32_t* rows, std::uint32_t* cols,
                                double* blocks) {
    RefScene& r = *static_cast<RefScene*>(p);
    IncrementalPotential ip(r.scene, r.surf, r.dofs, make_pol(det, 0, 0));
    std::vector<Vec3> xt(r.dofs.n_fem_nodes);
    for (Index v = 0; v < r.dofs.n_fem_nodes; ++v) xt[v] = ld3(x_tilde + 3 * v);
    std::vector<Vec12> qt(r.dofs.n_bodies);
    for (Index b = 0; b < r.dofs.n_bodies; ++b)
        for (int k = 0; k < 12; ++k) qt[b][k] = q_tilde[12 * b + k];
    ip.set_targets(xt, qt);
    ip.set_contact(dhat, kappa);
    if (!r.friction.empty()) ip.set_friction(r.friction, r.fr_base, r.mu, r.fr_eps);
    VecX g;
    SortedSymBlockCoo A;
    *value = ip.assemble(ref_state(r, x, q), g, A);
    for (Index k = 0; k < 3 * r.dofs.n_blocks(); ++k) grad[k] = g[k];
    if (static_cast<std::int64_t>(A.size()) > cap) return -static_cast<std::int64_t>(A.size()) - 1;
    for (std::size_t i = 0; i < A.size(); ++i) {
        rows[i] = A.rows[i];
        cols[i] = A.cols[i];
        std::memcpy(blocks + 9 * i, A.blocks[i].data(), 72);
    }
    return static_cast<std::int64_t>(A.size());
}
}  // extern "C"
