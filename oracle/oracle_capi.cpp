// ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.hpp header).
//
// extern "C" surface over the restated reference so pytest (ctypes) and the
// bench's CPU-baseline leg can drive it with plain pointers. Layout
// conventions match the product C-ABI (include/adipc_gpu.h): keys u64[T],
// blocks 9 doubles column-major (Eigen Mat3 storage), vectors flat 3n doubles.
// Also exposes the reference tests' std::mt19937 draws so the Python ports of
// the reference tests consume the identical random sequences.
#include <cstring>
#include <random>
#include <string>

#include "oracle.hpp"

using namespace oracle;

namespace {

thread_local std::string g_err;

ExecPolicy make_pol(int det, int threads, int lane_width) {
    ExecPolicy p;
    p.deterministic = det != 0;
    p.threads = threads;
    p.lane_width = lane_width > 0 ? lane_width : 32;
    return p;
}

BlockTripletStream load_stream(const std::uint64_t* keys, const double* vals, std::size_t T) {
    BlockTripletStream s;
    s.keys.assign(keys, keys + T);
    s.values.resize(T);
    if (T) std::memcpy(s.values.data(), vals, T * 9 * sizeof(double));
    return s;
}

void store_stream(const BlockTripletStream& s, std::uint64_t* keys, double* vals) {
    if (s.size() == 0) return;
    std::memcpy(keys, s.keys.data(), s.size() * sizeof(std::uint64_t));
    std::memcpy(vals, s.values.data(), s.size() * 9 * sizeof(double));
}

SortedSymBlockCoo load_matrix(std::int32_t n_block_rows, std::size_t U, const std::uint32_t* rows,
                              const std::uint32_t* cols, const double* blocks) {
    SortedSymBlockCoo A;
    A.n_block_rows = n_block_rows;
    A.rows.assign(rows, rows + U);
    A.cols.assign(cols, cols + U);
    A.blocks.resize(U);
    if (U) std::memcpy(A.blocks.data(), blocks, U * 9 * sizeof(double));
    return A;
}

std::vector<Edge> load_edges(const std::int32_t* pairs, std::size_t n) {
    std::vector<Edge> e(n);
    for (std::size_t i = 0; i < n; ++i) e[i] = {pairs[2 * i], pairs[2 * i + 1]};
    return e;
}

DofMap load_map(std::int32_t n_fem, std::int32_t n_bodies, std::size_t n_abd, const std::int32_t* body,
                const double* jac36) {
    DofMap m;
    m.n_fem_nodes = n_fem;
    m.n_bodies = n_bodies;
    m.abd_node_body.assign(body, body + n_abd);
    m.abd_node_jacobian.resize(n_abd, MatRC(3, 12));
    for (std::size_t i = 0; i < n_abd; ++i)
        std::memcpy(m.abd_node_jacobian[i].a.data(), jac36 + 36 * i, 36 * sizeof(double));
    return m;
}

}  // namespace

extern "C" {

const char* oracle_last_error() { return g_err.c_str(); }

int oracle_max_threads() { return process_thread_default(); }

void oracle_set_default_threads(int n) {  // parallel.hpp:36-38
    if (n > 0) process_thread_default() = n;
}

// ---- keys -----------------------------------------------------------------
std::uint64_t oracle_make_block_key(std::uint32_t r, std::uint32_t c) { return make_block_key(r, c); }

// emit(): canonicalise one block into (key, value); returns the key.
std::uint64_t oracle_emit(std::int32_t r, std::int32_t c, const double* m9, double* out9) {
    BlockTripletStream s;
    Mat3 m;
    std::memcpy(m.m, m9, sizeof(m.m));
    s.emit(r, c, m);
    std::memcpy(out9, s.values[0].m, sizeof(m.m));
    return s.keys[0];
}

// ---- sort / reduce ----------------------------------------------------------
void oracle_radix_sort_keys(std::uint64_t* keys, std::uint32_t* perm, std::size_t T) {
    std::vector<std::uint64_t> k(keys, keys + T);
    std::vector<std::uint32_t> p;
    radix_sort_keys(k, p);
    if (T) {
        std::memcpy(keys, k.data(), T * sizeof(std::uint64_t));
        std::memcpy(perm, p.data(), T * sizeof(std::uint32_t));
    }
}

void oracle_sort_stream(std::uint64_t* keys, double* vals, std::size_t T, int det, int threads, int lw) {
    BlockTripletStream s = load_stream(keys, vals, T);
    sort_stream(s, make_pol(det, threads, lw));
    store_stream(s, keys, vals);
}

// Sorted stream -> SortedSymBlockCoo. Output buffers sized >= T. Returns U.
std::int64_t oracle_fast_hash_reduction(const std::uint64_t* keys, const double* vals, std::size_t T,
                                        std::int32_t n_block_rows, int det, int threads, int lw,
                                        std::uint32_t* rows, std::uint32_t* cols, double* blocks) {
    const BlockTripletStream s = load_stream(keys, vals, T);
    const SortedSymBlockCoo A = fast_hash_reduction(s, n_block_rows, make_pol(det, threads, lw));
    const std::size_t U = A.size();
    if (U) {
        std::memcpy(rows, A.rows.data(), U * 4);
        std::memcpy(cols, A.cols.data(), U * 4);
        std::memcpy(blocks, A.blocks.data(), U * 72);
    }
    return static_cast<std::int64_t>(U);
}

// width: 1 (Real), 3 (Vec3) or 9 (Mat3). Returns 0, or 1 on size mismatch
// (std::invalid_argument in reduction.hpp:34).
int oracle_segment_reduce(const std::int32_t* O, std::size_t nO, const double* V, std::size_t nV, int width,
                          std::int32_t n_segments, int det, int threads, int lw, double* R) {
    const ExecPolicy pol = make_pol(det, threads, lw);
    const std::vector<Index> o(O, O + nO);
    try {
        if (width == 1) {
            std::vector<Real> v(V, V + nV);
            auto r = fast_segment_reduction(o, v, n_segments, pol);
            std::memcpy(R, r.data(), r.size() * sizeof(Real));
        } else if (width == 3) {
            std::vector<Vec3> v(nV);
            if (nV) std::memcpy(v.data(), V, nV * 24);
            auto r = fast_segment_reduction(o, v, n_segments, pol);
            if (!r.empty()) std::memcpy(R, r.data(), r.size() * 24);
        } else if (width == 9) {
            std::vector<Mat3> v(nV);
            if (nV) std::memcpy(v.data(), V, nV * 72);
            auto r = fast_segment_reduction(o, v, n_segments, pol);
            if (!r.empty()) std::memcpy(R, r.data(), r.size() * 72);
        } else {
            g_err = "width must be 1, 3 or 9";
            return 1;
        }
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    }
    return 0;
}

// ---- spmv ---------------------------------------------------------------
void oracle_srbk_spmv(std::int32_t n_block_rows, std::size_t U, const std::uint32_t* rows,
                      const std::uint32_t* cols, const double* blocks, const double* x, std::size_t nx,
                      int det, int threads, int lw, double* y) {
    const SortedSymBlockCoo A = load_matrix(n_block_rows, U, rows, cols, blocks);
    std::vector<Vec3> xv(nx);
    if (nx) std::memcpy(xv.data(), x, nx * 24);
    auto yv = srbk_spmv(A, xv, make_pol(det, threads, lw));
    if (nx) std::memcpy(y, yv.data(), nx * 24);
}

// ---- tiling / two-level ------------------------------------------------------
// kind: 0 split_12x12(rb, cb), 1 split_sym_12x12(rb), 2 split_12x3(rb, cb),
// 3 split_3x12(rb, cb). H column-major with its natural shape. Returns count.
int oracle_split(int kind, std::int32_t rb, std::int32_t cb, const double* H, std::uint64_t* keys,
                 double* vals) {
    BlockTripletStream out;
    if (kind == 0 || kind == 1) {
        MatRC m(12, 12);
        std::memcpy(m.a.data(), H, 144 * 8);
        if (kind == 0)
            split_12x12(rb, cb, m, out);
        else
            split_sym_12x12(rb, m, out);
    } else if (kind == 2) {
        MatRC m(12, 3);
        std::memcpy(m.a.data(), H, 36 * 8);
        split_12x3(rb, cb, m, out);
    } else {
        MatRC m(3, 12);
        std::memcpy(m.a.data(), H, 36 * 8);
        split_3x12(rb, cb, m, out);
    }
    store_stream(out, keys, vals);
    return static_cast<int>(out.size());
}

// Output capacity must be >= 16 * Tn. Returns the tile count.
std::int64_t oracle_two_level_abd_reduce(const std::uint64_t* keys, const double* vals, std::size_t Tn,
                                         std::int32_t n_fem, std::int32_t n_bodies, std::size_t n_abd,
                                         const std::int32_t* abd_node_body, const double* jac36, int det,
                                         int threads, int lw, std::uint64_t* out_keys, double* out_vals) {
    const BlockTripletStream s = load_stream(keys, vals, Tn);
    const DofMap m = load_map(n_fem, n_bodies, n_abd, abd_node_body, jac36);
    const BlockTripletStream t = two_level_abd_reduce(s, m, make_pol(det, threads, lw));
    store_stream(t, out_keys, out_vals);
    return static_cast<std::int64_t>(t.size());
}

// filter_pinned: output capacity >= T + n_slots. Returns new size.
std::int64_t oracle_filter_pinned(const std::uint64_t* keys, const double* vals, std::size_t T,
                                  const std::uint8_t* pinned, std::int32_t n_slots, std::uint64_t* out_keys,
                                  double* out_vals) {
    BlockTripletStream s = load_stream(keys, vals, T);
    std::vector<char> p(pinned, pinned + n_slots);
    filter_pinned(s, p);
    store_stream(s, out_keys, out_vals);
    return static_cast<std::int64_t>(s.size());
}


// ---- element-Hessian producer ---------------------------------
static Vec3 ld3(const double* p) {
    Vec3 v;
    for (int k = 0; k < 3; ++k) v[k] = p[k];
    return v;
}

// tet_rest (neo_hookean.hpp:13-27): p12 = 4 rest positions; 0 ok, 1 degenerate
int oracle_tet_rest(const double* p12, double* inv9, double* vol) {
    try {
        const TetRest r = tet_rest(ld3(p12), ld3(p12 + 3), ld3(p12 + 6), ld3(p12 + 9));
        for (int k = 0; k < 9; ++k) inv9[k] = r.inv_rest_edges.m[k];
        *vol = r.volume;
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

void oracle_stable_neo_hookean(const double* x12, const double* inv9, double vol, double mu, double lam, int project,
                               double* value, double* grad12, double* hess144) {
    TetRest r;
    for (int k = 0; k < 9; ++k) r.inv_rest_edges.m[k] = inv9[k];
    r.volume = vol;
    const Stencil12 s = stable_neo_hookean(ld3(x12), ld3(x12 + 3), ld3(x12 + 6), ld3(x12 + 9), r, mu, lam, project != 0);
    *value = s.value;
    for (int k = 0; k < 12; ++k) grad12[k] = s.grad[k];
    for (int k = 0; k < 144; ++k) hess144[k] = s.hess[k];
}

void oracle_project_psd(int n, const double* M, double* out) { oracle_eig::project_psd(n, M, out); }

// membrane.hpp:17-32 -> inv (2x2 column-major) + area; 0 ok, 1 degenerate
int oracle_membrane_rest(const double* p9, double* rest5) {
    try {
        const MembraneRest r = membrane_rest(ld3(p9), ld3(p9 + 3), ld3(p9 + 6));
        for (int k = 0; k < 4; ++k) rest5[k] = r.inv[k];
        rest5[4] = r.area;
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}
// incremental_potential.hpp:273-298; material5 = thickness, stretch, strain limit, shear fraction, bending
void oracle_membrane_stencil(const double* x9, const double* rest5, const double* material5, int project,
                             double* value, double* grad9, double* hess81) {
    MembraneRest r;
    for (int k = 0; k < 4; ++k) r.inv[k] = rest5[k];
    r.area = rest5[4];
    const ShellMaterial m{material5[0], material5[1], material5[2], material5[3], material5[4]};
    const Stencil9 s = membrane_stencil(ld3(x9), ld3(x9 + 3), ld3(x9 + 6), r, m, project != 0);
    *value = s.value;
    std::memcpy(grad9, s.grad, 72);
    std::memcpy(hess81, s.hess, 648);
}
int oracle_hinge_rest(const double* p12, double* rest2) {
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
void oracle_hinge_bending(const double* x12, const double* rest2, double k, int project, double* value,
                          double* grad12, double* hess144) {
    const Stencil12 s = hinge_bending(ld3(x12), ld3(x12 + 3), ld3(x12 + 6), ld3(x12 + 9), {rest2[0], rest2[1]}, k,
                                      project != 0);
    *value = s.value;
    std::memcpy(grad12, s.grad, 96);
    std::memcpy(hess144, s.hess, 1152);
}

void oracle_abd_orthogonality(const double* q12, double kappa, double volume, int project, double* value,
                              double* grad12, double* hess144) {
    const Stencil12 s = abd_orthogonality(q12, kappa, volume, project != 0);
    *value = s.value;
    std::memcpy(grad12, s.grad, 96);
    std::memcpy(hess144, s.hess, 1152);
}

// IncrementalPotential::assemble, inertia + solid meshes (see oracle.hpp):
// stream written to keys / vals9 (capacity n_verts + 10 n_tets), grad 3n;
// returns the stream length
std::int64_t oracle_ip_fem_assemble(std::int32_t n_verts, const double* x, const double* x_tilde, const double* mass,
                                    std::int32_t n_meshes, const std::int64_t* tet_begin, const double* mu,
                                    const double* lam, const std::int32_t* tets, const double* inv9, const double* vol,
                                    double dt2, const std::uint8_t* pinned, int project, std::uint64_t* keys,
                                    double* vals9, double* grad, double* value, std::int32_t n_bodies, const double* q,
                                    const double* q_tilde, const double* reduced_mass, const double* kappa,
                                    const double* body_volume, std::int32_t n_shells, const std::int64_t* tri_begin,
                                    const std::int32_t* tris, const double* tri_rest5, const std::int64_t* hinge_begin,
                                    const std::int32_t* hinges, const double* hinge_rest2, const double* material5,
                                    std::int32_t n_kinds, const std::int32_t* mesh_kind) {
    std::vector<Vec3> xs(n_verts), xt(n_verts);
    for (std::int32_t v = 0; v < n_verts; ++v) {
        xs[v] = ld3(x + 3 * v);
        xt[v] = ld3(x_tilde + 3 * v);
    }
    std::vector<Real> m(mass, mass + n_verts);
    FemSolids fs;
    const std::int64_t nt = tet_begin[n_meshes];
    fs.tets.assign(tets, tets + 4 * nt);
    fs.rest.resize(nt);
    for (std::int64_t t = 0; t < nt; ++t) {
        for (int k = 0; k < 9; ++k) fs.rest[t].inv_rest_edges.m[k] = inv9[9 * t + k];
        fs.rest[t].volume = vol[t];
    }
    fs.tet_begin.assign(tet_begin, tet_begin + n_meshes + 1);
    fs.mu.assign(mu, mu + n_meshes);
    fs.lam.assign(lam, lam + n_meshes);
    const std::int32_t n_slots = n_verts + 4 * n_bodies;
    std::vector<char> pin(n_slots, 0);
    if (pinned)
        for (std::int32_t v = 0; v < n_slots; ++v) pin[v] = static_cast<char>(pinned[v]);
    Bodies bodies;
    if (n_bodies > 0) {
        bodies.q.assign(q, q + 12 * n_bodies);
        bodies.q_tilde.assign(q_tilde, q_tilde + 12 * n_bodies);
        bodies.reduced_mass.assign(reduced_mass, reduced_mass + 144 * n_bodies);
        bodies.kappa.assign(kappa, kappa + n_bodies);
        bodies.volume.assign(body_volume, body_volume + n_bodies);
    }
    FemShells sh;
    std::vector<int> kinds(mesh_kind, mesh_kind + n_kinds);
    if (n_shells > 0) {
        sh.tri_begin.assign(tri_begin, tri_begin + n_shells + 1);
        sh.hinge_begin.assign(hinge_begin, hinge_begin + n_shells + 1);
        const std::int64_t ntr = tri_begin[n_shells], nh = hinge_begin[n_shells];
        sh.tris.assign(tris, tris + 3 * ntr);
        sh.hinges.assign(hinges, hinges + 4 * nh);
        sh.tri_rest.resize(ntr);
        for (std::int64_t t = 0; t < ntr; ++t) {
            for (int k = 0; k < 4; ++k) sh.tri_rest[t].inv[k] = tri_rest5[5 * t + k];
            sh.tri_rest[t].area = tri_rest5[5 * t + 4];
        }
        sh.hinge_rest.resize(nh);
        for (std::int64_t h = 0; h < nh; ++h) sh.hinge_rest[h] = {hinge_rest2[2 * h], hinge_rest2[2 * h + 1]};
        for (std::int32_t i = 0; i < n_shells; ++i)
            sh.material.push_back({material5[5 * i], material5[5 * i + 1], material5[5 * i + 2], material5[5 * i + 3],
                                   material5[5 * i + 4]});
    }
    std::vector<Real> g;
    BlockTripletStream s;
    *value = ip_fem_assemble(xs, xt, m, fs, dt2, pin, g, s, project != 0, &bodies, n_shells > 0 ? &sh : nullptr,
                             n_kinds > 0 ? &kinds : nullptr);
    for (std::size_t k = 0; k < g.size(); ++k) grad[k] = g[k];
    store_stream(s, keys, vals9);
    return static_cast<std::int64_t>(s.size());
}


// ---- contact producers -----------------------------------------
void oracle_pt_dist2_derivs(const double* x12, double* d2, double* g12, double* h144) {
    const PairDerivs pd = pt_dist2_derivs(ld3(x12), ld3(x12 + 3), ld3(x12 + 6), ld3(x12 + 9));
    *d2 = pd.dist2;
    std::memcpy(g12, pd.grad, 96);
    std::memcpy(h144, pd.hess, 1152);
}
void oracle_ee_dist2_derivs(const double* x12, double* d2, double* g12, double* h144) {
    const PairDerivs pd = ee_dist2_derivs(ld3(x12), ld3(x12 + 3), ld3(x12 + 6), ld3(x12 + 9));
    *d2 = pd.dist2;
    std::memcpy(g12, pd.grad, 96);
    std::memcpy(h144, pd.hess, 1152);
}
double oracle_pt_dist2(const double* x12) { return pt_dist2(ld3(x12), ld3(x12 + 3), ld3(x12 + 6), ld3(x12 + 9)); }
double oracle_ee_dist2(const double* x12) { return ee_dist2(ld3(x12), ld3(x12 + 3), ld3(x12 + 6), ld3(x12 + 9)); }
void oracle_barrier_pair_derivs(double d2, const double* g12, const double* h144, double shat, double kappa,
                                int project, double* value, double* og12, double* oh144) {
    PairDerivs pd;
    pd.dist2 = d2;
    std::memcpy(pd.grad, g12, 96);
    std::memcpy(pd.hess, h144, 1152);
    const BarrierDerivs b = barrier_pair_derivs(pd, shat, kappa, project != 0);
    *value = b.value;
    std::memcpy(og12, b.grad, 96);
    std::memcpy(oh144, b.hess, 1152);
}
void oracle_ground_barrier_derivs(const double* x3, const double* n3, double height, double dhat, double kappa,
                                  int project, double* value, double* g3, double* h9, double* dist) {
    const GroundDerivs gd = ground_barrier_derivs(ld3(x3), ld3(n3), height, dhat, kappa, project != 0);
    *value = gd.value;
    for (int k = 0; k < 3; ++k) g3[k] = gd.grad[k];
    std::memcpy(h9, gd.hess.m, 72);
    *dist = gd.dist;
}

static ContactInput contact_input(std::int32_t n_nodes, const double* pos, std::int64_t n_pt, const std::int32_t* pt,
                                  std::int64_t n_ee, const std::int32_t* ee, double dhat, double kappa, int ground,
                                  const double* normal, double height, std::int32_t n_sv, const std::int32_t* sv,
                                  std::int64_t n_fr, const std::int32_t* fr_nodes, const std::int32_t* fr_n,
                                  const double* fr_coeff, const double* fr_t1, const double* fr_t2,
                                  const double* fr_lambda, const double* fr_base, double mu, double eps) {
    ContactInput in;
    in.pos.resize(n_nodes);
    for (std::int32_t v = 0; v < n_nodes; ++v) in.pos[v] = ld3(pos + 3 * v);
    for (std::int64_t i = 0; i < n_pt; ++i) in.pt.push_back({pt[4 * i], pt[4 * i + 1], pt[4 * i + 2], pt[4 * i + 3]});
    for (std::int64_t i = 0; i < n_ee; ++i) in.ee.push_back({ee[4 * i], ee[4 * i + 1], ee[4 * i + 2], ee[4 * i + 3]});
    in.dhat = dhat;
    in.kappa = kappa;
    in.ground = ground != 0;
    if (normal) in.ground_normal = ld3(normal);
    in.ground_height = height;
    in.surf_verts.assign(sv, sv + n_sv);
    for (std::int64_t i = 0; i < n_fr; ++i) {
        FrictionConstraint c;
        c.n_nodes = fr_n[i];
        for (int k = 0; k < 4; ++k) {
            c.nodes[k] = fr_nodes[4 * i + k];
            c.coeff[k] = fr_coeff[4 * i + k];
        }
        c.t1 = ld3(fr_t1 + 3 * i);
        c.t2 = ld3(fr_t2 + 3 * i);
        c.lambda = fr_lambda[i];
        in.friction.push_back(c);
    }
    if (n_fr > 0) {
        in.fr_base.resize(n_nodes);
        for (std::int32_t v = 0; v < n_nodes; ++v) in.fr_base[v] = ld3(fr_base + 3 * v);
    }
    in.mu = mu;
    in.fr_eps = eps;
    return in;
}
#define ORACLE_CONTACT_ARGS                                                                                        \
    std::int32_t n_nodes, const double *pos, std::int64_t n_pt, const std::int32_t *pt, std::int64_t n_ee,        \
        const std::int32_t *ee, double dhat, double kappa, int ground, const double *normal, double height,       \
        std::int32_t n_sv, const std::int32_t *sv, std::int64_t n_fr, const std::int32_t *fr_nodes,              \
        const std::int32_t *fr_n, const double *fr_coeff, const double *fr_t1, const double *fr_t2,               \
        const double *fr_lambda, const double *fr_base, double mu, double eps
#define ORACLE_CONTACT_PASS                                                                                        \
    n_nodes, pos, n_pt, pt, n_ee, ee, dhat, kappa, ground, normal, height, n_sv, sv, n_fr, fr_nodes, fr_n,        \
        fr_coeff, fr_t1, fr_t2, fr_lambda, fr_base, mu, eps

// assemble_contact's node part: stream (keys / vals9), node gradient, value
std::int64_t oracle_contact_assemble(ORACLE_CONTACT_ARGS, double dt2, int project, std::uint64_t* keys, double* vals9,
                                     double* node_grad, double* value) {
    const ContactInput in = contact_input(ORACLE_CONTACT_PASS);
    std::vector<Vec3> g;
    BlockTripletStream s;
    *value = contact_assemble(in, dt2, g, s, project != 0);
    for (std::int32_t v = 0; v < n_nodes; ++v)
        for (int k = 0; k < 3; ++k) node_grad[3 * v + k] = g[v][k];
    store_stream(s, keys, vals9);
    return static_cast<std::int64_t>(s.size());
}
double oracle_contact_value(ORACLE_CONTACT_ARGS, double dt2) {
    return contact_value(contact_input(ORACLE_CONTACT_PASS), dt2);
}
double oracle_ccd_step(ORACLE_CONTACT_ARGS, const double* disp) {
    const ContactInput in = contact_input(ORACLE_CONTACT_PASS);
    std::vector<Vec3> d(n_nodes);
    for (std::int32_t v = 0; v < n_nodes; ++v) d[v] = ld3(disp + 3 * v);
    return ccd_step(in, d);
}


// broad_phase.hpp:143-211: candidates written as surface-slot pairs; returns
// n_pt, *n_ee_out = n_ee (capacities pt_cap / ee_cap pairs)
std::int64_t oracle_find_candidates(std::int32_t n_nodes, const double* pos, const double* disp, std::int32_t n_verts,
                                    const std::int32_t* verts, std::int32_t n_edges, const std::int32_t* edges,
                                    std::int32_t n_tris, const std::int32_t* tris, double inflate,
                                    std::int32_t* pt_out, std::int64_t pt_cap, std::int32_t* ee_out,
                                    std::int64_t ee_cap, std::int64_t* n_ee_out) {
    std::vector<Vec3> p(n_nodes), d;
    for (std::int32_t v = 0; v < n_nodes; ++v) p[v] = ld3(pos + 3 * v);
    if (disp) {
        d.resize(n_nodes);
        for (std::int32_t v = 0; v < n_nodes; ++v) d[v] = ld3(disp + 3 * v);
    }
    ContactSurface s;
    s.verts.assign(verts, verts + n_verts);
    for (std::int32_t e = 0; e < n_edges; ++e) s.edges.push_back({edges[2 * e], edges[2 * e + 1]});
    for (std::int32_t t = 0; t < n_tris; ++t) s.tris.push_back({tris[3 * t], tris[3 * t + 1], tris[3 * t + 2]});
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

// ---- partition / hierarchy ----------------------------------------------------
std::int32_t oracle_subdomain_count(std::int32_t v, std::int32_t n, std::int32_t n_o) {
    return subdomain_count(v, n, n_o);
}

std::int32_t oracle_chunk_partition(std::int32_t v, std::int32_t cap, std::int32_t* part_of) {
    const Partition p = chunk_partition(v, cap);
    if (v) std::memcpy(part_of, p.part_of.data(), v * 4);
    return p.n_parts;
}

std::int32_t oracle_partition_block_graph(std::int32_t v, const std::int32_t* pairs, std::size_t n_edges,
                                          std::int32_t cap, std::int32_t* part_of) {
    const Partition p = partition_block_graph(v, load_edges(pairs, n_edges), cap);
    if (v) std::memcpy(part_of, p.part_of.data(), v * 4);
    return p.n_parts;
}

std::int64_t oracle_block_edges(std::size_t U, const std::uint32_t* rows, const std::uint32_t* cols,
                                std::int32_t* pairs) {
    std::int64_t w = 0;
    for (std::size_t i = 0; i < U; ++i)
        if (rows[i] != cols[i]) {
            pairs[2 * w] = static_cast<std::int32_t>(rows[i]);
            pairs[2 * w + 1] = static_cast<std::int32_t>(cols[i]);
            ++w;
        }
    return w;
}

void* oracle_build_hierarchy(const std::int32_t* part_of, std::int32_t n_slots, std::int32_t n_parts,
                             std::int32_t capacity, const std::int32_t* pairs, std::size_t n_edges,
                             int max_levels) {
    Partition l0;
    l0.part_of.assign(part_of, part_of + n_slots);
    l0.n_parts = n_parts;
    l0.capacity = capacity;
    return new MasHierarchy(build_hierarchy(l0, load_edges(pairs, n_edges), max_levels));
}
void oracle_hierarchy_free(void* h) { delete static_cast<MasHierarchy*>(h); }
int oracle_hierarchy_n_levels(void* h) { return static_cast<MasHierarchy*>(h)->n_levels(); }
void oracle_hierarchy_level(void* hp, int l, std::int32_t* n_nodes, std::int32_t* n_parts,
                            std::int32_t* part_of, std::int32_t* agg) {
    const auto& L = static_cast<MasHierarchy*>(hp)->levels[l];
    *n_nodes = L.n_nodes;
    *n_parts = L.n_parts;
    if (part_of && L.n_nodes) std::memcpy(part_of, L.part_of.data(), L.n_nodes * 4);
    if (agg && !L.agg.empty()) std::memcpy(agg, L.agg.data(), L.agg.size() * 4);
}

// ---- preconditioners ------------------------------------------------------------
struct OracleMatrix {
    SortedSymBlockCoo A;
};

void* oracle_matrix_new(std::int32_t n_block_rows, std::size_t U, const std::uint32_t* rows,
                        const std::uint32_t* cols, const double* blocks) {
    return new OracleMatrix{load_matrix(n_block_rows, U, rows, cols, blocks)};
}
void oracle_matrix_free(void* m) { delete static_cast<OracleMatrix*>(m); }

// Returns a MasPreconditioner*, or null with oracle_last_error() set
// (std::runtime_error of mas.hpp:74-77).
void* oracle_mas_build(void* mat, void* hier) {
    auto* M = new MasPreconditioner();
    try {
        M->build(static_cast<OracleMatrix*>(mat)->A, *static_cast<MasHierarchy*>(hier));
    } catch (const std::runtime_error& e) {
        g_err = e.what();
        delete M;
        return nullptr;
    }
    return M;
}
void oracle_precond_free(void* p) { delete static_cast<Preconditioner*>(p); }
long oracle_mas_shifts(void* p) { return static_cast<MasPreconditioner*>(p)->shifts_applied; }
int oracle_mas_n_levels(void* p) { return static_cast<int>(static_cast<MasPreconditioner*>(p)->levels_.size()); }
// dim of subdomain s at level l; copies the dense restricted matrix if out != null
int oracle_mas_level_matrix(void* p, int l, std::int32_t s, double* out) {
    const auto& ld = static_cast<MasPreconditioner*>(p)->levels_[l];
    if (out) std::memcpy(out, ld.dense[s].data(), ld.dense[s].size() * 8);
    return ld.dim[s];
}

void* oracle_jacobi_build(void* mat) {
    auto* J = new BlockJacobiPreconditioner();
    J->build(static_cast<OracleMatrix*>(mat)->A);
    return J;
}

void oracle_precond_apply(void* p, const double* r, std::size_t n, double* z) {
    std::vector<Real> rv(r, r + n), zv;
    static_cast<Preconditioner*>(p)->apply(rv, zv);
    std::memcpy(z, zv.data(), n * 8);
}

int oracle_pcg_solve(void* mat, const double* b, std::size_t n, void* precond, double rel_tol, int restart,
                     int max_iters, int det, int threads, int lw, double* x, int* iters, double* rel_residual,
                     int* converged) {
    std::vector<Real> bv(b, b + n), xv;
    const PcgResult r = pcg_solve(static_cast<OracleMatrix*>(mat)->A, bv, *static_cast<Preconditioner*>(precond),
                                  rel_tol, restart, max_iters, make_pol(det, threads, lw), xv);
    std::memcpy(x, xv.data(), n * 8);
    *iters = r.iters;
    *rel_residual = r.rel_residual;
    *converged = r.converged ? 1 : 0;
    return 0;
}

#include "capi_rng.inc"

}  // extern "C"


extern "C" {
// ---- contact frames, tangent basis, friction constraints (restated; see oracle.hpp) ----
static void store_frame(const ContactFrame& f, double* dist, double* normal3, double* coeff4) {
    *dist = f.dist;
    for (int a = 0; a < 3; ++a) normal3[a] = f.normal[a];
    for (int k = 0; k < 4; ++k) coeff4[k] = f.coeff[k];
}
void oracle_pt_contact_frame(const double* x12, double* dist, double* normal3, double* coeff4) {
    store_frame(pt_contact_frame(ld3(x12), ld3(x12 + 3), ld3(x12 + 6), ld3(x12 + 9)), dist, normal3, coeff4);
}
void oracle_ee_contact_frame(const double* x12, double* dist, double* normal3, double* coeff4) {
    store_frame(ee_contact_frame(ld3(x12), ld3(x12 + 3), ld3(x12 + 6), ld3(x12 + 9)), dist, normal3, coeff4);
}
void oracle_tangent_basis(const double* n3, double* t1, double* t2) {
    Vec3 a, b;
    tangent_basis(ld3(n3), a, b);
    for (int k = 0; k < 3; ++k) {
        t1[k] = a[k];
        t2[k] = b[k];
    }
}
// friction constraints for GIVEN candidates (the ContactInput's stencils)
std::int64_t oracle_friction_constraints(ORACLE_CONTACT_ARGS, std::int64_t cap, std::int32_t* nodes4,
                                         std::int32_t* n_nodes_out, double* coeff4, double* t1, double* t2,
                                         double* lambda) {
    const std::vector<FrictionConstraint> fc = friction_constraints(contact_input(ORACLE_CONTACT_PASS));
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
}  // extern "C"
