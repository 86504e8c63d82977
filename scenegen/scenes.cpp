// Synthetic scene generators for the benchmark configurations
// (BASELINE.json configs 1-5). Host C++, used by bench.py and
// the tests to build the triplet streams the hot path consumes; they stand in
// for the reference's element/contact producers (OUT OF SCOPE, SURVEY §2 rows
// 17-18), reusing the reference's mesh generators and emission order:
//   geometry/shapes.hpp:21-76      make_grid, make_box_tets (6 tets per cell)
//   scene/mesh.hpp:146-165          lumped masses (rho V / 4 per tet vertex)
//   energy/neo_hookean.hpp:44-103   stable Neo-Hookean Hessian; at the rest
//                                   state F = I it is PSD, so the first Newton
//                                   matrix needs no eigen-projection
//   solver/incremental_potential.hpp:170-249  emission order: mass diagonals,
//                                   body mass tiles, element stencils
//                                   (scatter9 / scatter12), orthogonality tiles
//   solver/newton.hpp:204-241       rest_edges (element cliques + body cliques)
// Contact stencils (cfg 3/4) are seeded PSD 12x12 matrices L L^T on 4-node
// stencils between neighbouring objects, fed to two_level_abd_reduce.
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <random>
#include <vector>

namespace {

using Index = std::int32_t;

struct M3 {
    double m[9] = {0};  // column-major
    double& operator()(int r, int c) { return m[3 * c + r]; }
    double operator()(int r, int c) const { return m[3 * c + r]; }
};

struct Scene {
    Index n_blocks = 0, n_fem = 0, n_bodies = 0;
    std::vector<std::uint64_t> keys, node_keys;
    std::vector<double> vals, node_vals;
    std::vector<Index> abd_body;
    std::vector<double> abd_jac;  // 36 per abd node
    std::vector<std::uint8_t> pinned;
    std::vector<Index> rest_edges;  // pairs
    // deformable solid mesh of FEM-only scenes (the element producer's input):
    // rest positions (3 per vertex), tets (4 global slots each), vertex masses
    std::vector<double> mesh_verts, mesh_mass;
    std::vector<Index> mesh_tets;
    double mu = 0, lam = 0;

    void emit(std::vector<std::uint64_t>& ks, std::vector<double>& vs, Index r, Index c, const double* b) {
        if (r <= c) {
            ks.push_back((static_cast<std::uint64_t>(r) << 32) | static_cast<std::uint32_t>(c));
            vs.insert(vs.end(), b, b + 9);
        } else {
            ks.push_back((static_cast<std::uint64_t>(c) << 32) | static_cast<std::uint32_t>(r));
            for (int j = 0; j < 3; ++j)
                for (int i = 0; i < 3; ++i) vs.push_back(b[3 * i + j]);  // transpose
        }
    }
    void emit(Index r, Index c, const double* b) { emit(keys, vals, r, c, b); }
    void emit_node(Index r, Index c, const double* b) { emit(node_keys, node_vals, r, c, b); }
};

struct Vec3d {
    double x, y, z;
};

struct TetMesh {
    std::vector<Vec3d> verts;
    std::vector<std::array<Index, 4>> tets;
};

// geometry/shapes.hpp:56-76
TetMesh make_box_tets(int nx, int ny, int nz, double sx, double sy, double sz) {
    static const int kCube[6][4] = {{0, 1, 3, 7}, {0, 3, 2, 7}, {0, 2, 6, 7}, {0, 6, 4, 7}, {0, 4, 5, 7}, {0, 5, 1, 7}};
    TetMesh m;
    const int vx = nx + 1, vy = ny + 1, vz = nz + 1;
    auto vid = [&](int i, int j, int k) { return static_cast<Index>((k * vy + j) * vx + i); };
    for (int k = 0; k < vz; ++k)
        for (int j = 0; j < vy; ++j)
            for (int i = 0; i < vx; ++i) m.verts.push_back({sx * i / nx, sy * j / ny, sz * k / nz});
    for (int k = 0; k < nz; ++k)
        for (int j = 0; j < ny; ++j)
            for (int i = 0; i < nx; ++i) {
                Index c[8];
                for (int b = 0; b < 8; ++b) c[b] = vid(i + (b & 1), j + ((b >> 1) & 1), k + ((b >> 2) & 1));
                for (const auto& t : kCube) m.tets.push_back({c[t[0]], c[t[1]], c[t[2]], c[t[3]]});
            }
    return m;
}

// geometry/shapes.hpp:79-104
TetMesh make_ellipsoid_tets(int n, double rx, double ry, double rz) {
    TetMesh box = make_box_tets(n, n, n, 2 * rx, 2 * ry, 2 * rz);
    TetMesh m;
    std::vector<Index> remap(box.verts.size(), -1);
    for (const auto& t : box.tets) {
        double cx = 0, cy = 0, cz = 0;
        for (Index v : t) {
            cx += box.verts[v].x;
            cy += box.verts[v].y;
            cz += box.verts[v].z;
        }
        cx = cx / 4 - rx;
        cy = cy / 4 - ry;
        cz = cz / 4 - rz;
        if (cx * cx / (rx * rx) + cy * cy / (ry * ry) + cz * cz / (rz * rz) > 1.0) continue;
        std::array<Index, 4> nt;
        for (int a = 0; a < 4; ++a) {
            if (remap[t[a]] < 0) {
                remap[t[a]] = static_cast<Index>(m.verts.size());
                m.verts.push_back(box.verts[t[a]]);
            }
            nt[a] = remap[t[a]];
        }
        m.tets.push_back(nt);
    }
    return m;
}

M3 inverse3(const M3& a, double* det_out) {
    M3 c;
    c(0, 0) = a(1, 1) * a(2, 2) - a(1, 2) * a(2, 1);
    c(1, 0) = a(1, 2) * a(2, 0) - a(1, 0) * a(2, 2);
    c(2, 0) = a(1, 0) * a(2, 1) - a(1, 1) * a(2, 0);
    const double det = a(0, 0) * c(0, 0) + a(0, 1) * c(1, 0) + a(0, 2) * c(2, 0);
    c(0, 1) = a(0, 2) * a(2, 1) - a(0, 1) * a(2, 2);
    c(1, 1) = a(0, 0) * a(2, 2) - a(0, 2) * a(2, 0);
    c(2, 1) = a(0, 1) * a(2, 0) - a(0, 0) * a(2, 1);
    c(0, 2) = a(0, 1) * a(1, 2) - a(0, 2) * a(1, 1);
    c(1, 2) = a(0, 2) * a(1, 0) - a(0, 0) * a(1, 2);
    c(2, 2) = a(0, 0) * a(1, 1) - a(0, 1) * a(1, 0);
    M3 inv;
    for (int k = 0; k < 9; ++k) inv.m[k] = c.m[k] / det;
    *det_out = det;
    return inv;
}

// Stable Neo-Hookean Hessian at F = I (neo_hookean.hpp:44-101): V dFdx^T H9 dFdx.
void rest_tet_hessian(const Vec3d* p, double mu, double lam, double* H /*12x12 col-major*/, double* vol) {
    M3 Dm;
    const Vec3d e[3] = {{p[1].x - p[0].x, p[1].y - p[0].y, p[1].z - p[0].z},
                        {p[2].x - p[0].x, p[2].y - p[0].y, p[2].z - p[0].z},
                        {p[3].x - p[0].x, p[3].y - p[0].y, p[3].z - p[0].z}};
    for (int c = 0; c < 3; ++c) {
        Dm(0, c) = e[c].x;
        Dm(1, c) = e[c].y;
        Dm(2, c) = e[c].z;
    }
    double det;
    const M3 B = inverse3(Dm, &det);
    const double V = det / 6.0;
    *vol = V;
    double J[9][12] = {{0}};
    for (int j = 0; j < 3; ++j)
        for (int c = 0; c < 3; ++c)
            for (int k = 0; k < 3; ++k) {
                J[3 * j + k][3 * (c + 1) + k] += B(c, j);
                J[3 * j + k][k] -= B(c, j);
            }
    double H9[9][9] = {{0}};
    const double vecI[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
    for (int a = 0; a < 9; ++a)
        for (int b = 0; b < 9; ++b) H9[a][b] = (a == b ? mu : 0.0) + lam * vecI[a] * vecI[b];
    // + dJcoef * HJ with dJcoef = lam (J - 1) - mu = -mu at rest
    auto cross = [](int axis, double s, double (*out)[3]) {
        double a[3] = {0, 0, 0};
        a[axis] = s;
        const double m[3][3] = {{0, -a[2], a[1]}, {a[2], 0, -a[0]}, {-a[1], a[0], 0}};
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) out[r][c] = m[r][c];
    };
    auto put = [&](int br, int bc, int axis, double s) {
        double m[3][3];
        cross(axis, s, m);
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) H9[3 * br + r][3 * bc + c] += -mu * m[r][c];
    };
    put(0, 1, 2, -1);
    put(0, 2, 1, 1);
    put(1, 0, 2, 1);
    put(1, 2, 0, -1);
    put(2, 0, 1, -1);
    put(2, 1, 0, 1);
    double T[9][12] = {{0}};  // H9 * J
    for (int a = 0; a < 9; ++a)
        for (int c = 0; c < 12; ++c) {
            double s = 0;
            for (int b = 0; b < 9; ++b) s += H9[a][b] * J[b][c];
            T[a][c] = s;
        }
    for (int r = 0; r < 12; ++r)
        for (int c = 0; c < 12; ++c) {
            double s = 0;
            for (int a = 0; a < 9; ++a) s += J[a][r] * T[a][c];
            H[12 * c + r] = V * s;
        }
}

// One deformable tet mesh appended at slot offset `off` (mass diagonals are
// emitted separately, first, like incremental_potential.hpp:170-180).
struct FemPart {
    TetMesh mesh;
    Index off;
    double mu, lam, rho;
    std::vector<double> mass;
};

void fem_masses(FemPart& f) {
    f.mass.assign(f.mesh.verts.size(), 0.0);
    for (const auto& t : f.mesh.tets) {
        const Vec3d p[4] = {f.mesh.verts[t[0]], f.mesh.verts[t[1]], f.mesh.verts[t[2]], f.mesh.verts[t[3]]};
        const double d = (p[1].x - p[0].x) * ((p[2].y - p[0].y) * (p[3].z - p[0].z) - (p[2].z - p[0].z) * (p[3].y - p[0].y)) -
                         (p[2].x - p[0].x) * ((p[1].y - p[0].y) * (p[3].z - p[0].z) - (p[1].z - p[0].z) * (p[3].y - p[0].y)) +
                         (p[3].x - p[0].x) * ((p[1].y - p[0].y) * (p[2].z - p[0].z) - (p[1].z - p[0].z) * (p[2].y - p[0].y));
        const double mt = f.rho * d / 6.0;
        for (Index v : t) f.mass[v] += mt / 4;
    }
}

void emit_mass(Scene& s, const FemPart& f) {
    for (std::size_t v = 0; v < f.mass.size(); ++v) {
        double b[9] = {f.mass[v], 0, 0, 0, f.mass[v], 0, 0, 0, f.mass[v]};
        s.emit(f.off + static_cast<Index>(v), f.off + static_cast<Index>(v), b);
    }
}

void emit_tets(Scene& s, const FemPart& f, double dt2) {
    double H[144], vol;
    for (const auto& t : f.mesh.tets) {
        const Vec3d p[4] = {f.mesh.verts[t[0]], f.mesh.verts[t[1]], f.mesh.verts[t[2]], f.mesh.verts[t[3]]};
        rest_tet_hessian(p, f.mu, f.lam, H, &vol);
        for (int a = 0; a < 4; ++a)  // scatter12 (incremental_potential.hpp:310-318)
            for (int b = a; b < 4; ++b) {
                double blk[9];
                for (int c = 0; c < 3; ++c)
                    for (int r = 0; r < 3; ++r) blk[3 * c + r] = dt2 * H[12 * (3 * b + c) + 3 * a + r];
                s.emit(f.off + t[a], f.off + t[b], blk);
            }
        for (int a = 0; a < 4; ++a)  // rest_edges clique (newton.hpp:218-224)
            for (int b = a + 1; b < 4; ++b) {
                s.rest_edges.push_back(std::min(f.off + t[a], f.off + t[b]));
                s.rest_edges.push_back(std::max(f.off + t[a], f.off + t[b]));
            }
    }
}

void finish_edges(Scene& s) {  // sort + unique (newton.hpp:238-240)
    std::vector<std::uint64_t> e(s.rest_edges.size() / 2);
    for (std::size_t i = 0; i < e.size(); ++i)
        e[i] = (static_cast<std::uint64_t>(s.rest_edges[2 * i]) << 32) | static_cast<std::uint32_t>(s.rest_edges[2 * i + 1]);
    std::sort(e.begin(), e.end());
    e.erase(std::unique(e.begin(), e.end()), e.end());
    s.rest_edges.resize(2 * e.size());
    for (std::size_t i = 0; i < e.size(); ++i) {
        s.rest_edges[2 * i] = static_cast<Index>(e[i] >> 32);
        s.rest_edges[2 * i + 1] = static_cast<Index>(e[i] & 0xFFFFFFFFu);
    }
}

// random PSD 12x12 = scale * L L^T / 12, L ~ N(0,1)
void random_psd12(std::mt19937& rng, double scale, double* H) {
    std::normal_distribution<double> nd(0.0, 1.0);
    double L[144];
    for (double& v : L) v = nd(rng);
    for (int r = 0; r < 12; ++r)
        for (int c = 0; c < 12; ++c) {
            double s = 0;
            for (int k = 0; k < 12; ++k) s += L[12 * k + r] * L[12 * k + c];
            H[12 * c + r] = scale * s / 12.0;
        }
}

void emit_stencil12(Scene& s, const Index* ids, const double* H, bool node_stream) {
    for (int a = 0; a < 4; ++a)
        for (int b = a; b < 4; ++b) {
            double blk[9];
            for (int c = 0; c < 3; ++c)
                for (int r = 0; r < 3; ++r) blk[3 * c + r] = H[12 * (3 * b + c) + 3 * a + r];
            if (node_stream)
                s.emit_node(ids[a], ids[b], blk);
            else
                s.emit(ids[a], ids[b], blk);
        }
}

// Affine body: Jacobians, reduced mass tiles, orthogonality tiles
// (scene/mesh.hpp:196-258, incremental_potential.hpp:181-188, 242-249).
struct Body {
    TetMesh mesh;
    Vec3d shift;
    double rho, kappa;
    std::vector<double> mass;
    double volume = 0;
};

void body_prepare(Body& b) {
    FemPart f{b.mesh, 0, 0, 0, b.rho, {}};
    fem_masses(f);
    b.mass = f.mass;
    b.volume = 0;
    for (double m : b.mass) b.volume += m / b.rho;
}

void body_jacobian(const Vec3d& rest, double* J36) {  // mesh.hpp:196-201, column-major 3x12
    std::memset(J36, 0, 36 * sizeof(double));
    for (int r = 0; r < 3; ++r) J36[3 * r + r] = 1.0;
    const double x[3] = {rest.x, rest.y, rest.z};
    for (int r = 0; r < 3; ++r)
        for (int k = 0; k < 3; ++k) J36[3 * (3 + 3 * r + k) + r] = x[k];
}

void emit_sym12(Scene& s, Index base, const double* H) {  // split_sym_12x12
    for (int ti = 0; ti < 4; ++ti)
        for (int tj = ti; tj < 4; ++tj) {
            double blk[9];
            for (int c = 0; c < 3; ++c)
                for (int r = 0; r < 3; ++r) blk[3 * c + r] = H[12 * (3 * tj + c) + 3 * ti + r];
            s.emit(base + ti, base + tj, blk);
        }
}

void body_mass_matrix(const Body& b, double* M) {  // sum m J^T J
    std::memset(M, 0, 144 * sizeof(double));
    double J[36];
    for (std::size_t v = 0; v < b.mesh.verts.size(); ++v) {
        const Vec3d p = {b.mesh.verts[v].x + b.shift.x, b.mesh.verts[v].y + b.shift.y, b.mesh.verts[v].z + b.shift.z};
        body_jacobian(p, J);
        for (int r = 0; r < 12; ++r)
            for (int c = 0; c < 12; ++c) {
                double s = 0;
                for (int k = 0; k < 3; ++k) s += J[3 * r + k] * J[3 * c + k];
                M[12 * c + r] += b.mass[v] * s;
            }
    }
}

// jitter > 0: every vertex moved by jitter * (cell size) * U(-1, 1) per axis
// (std::mt19937(seed)) — the cfg5 batch of scenes, seeds 5..12 (SURVEY.md
// §8d): same connectivity and pins, different element shapes and values.
Scene* fem_box(int nx, int ny, int nz, double sx, double sy, double sz, double E, double nu, double rho, double dt,
               int pin_x0, double jitter, unsigned seed) {
    auto* s = new Scene();
    FemPart f{make_box_tets(nx, ny, nz, sx, sy, sz), 0, E / (2 * (1 + nu)), E * nu / ((1 + nu) * (1 - 2 * nu)), rho, {}};
    std::vector<std::uint8_t> on_x0(f.mesh.verts.size(), 0);
    for (std::size_t v = 0; v < f.mesh.verts.size(); ++v) on_x0[v] = f.mesh.verts[v].x <= 1e-12 ? 1 : 0;
    if (jitter > 0) {
        std::mt19937 rng(seed);
        std::uniform_real_distribution<double> ud(-1.0, 1.0);
        const double hx = sx / nx, hy = sy / ny, hz = sz / nz;
        for (auto& v : f.mesh.verts) {
            v.x += jitter * hx * ud(rng);
            v.y += jitter * hy * ud(rng);
            v.z += jitter * hz * ud(rng);
        }
    }
    fem_masses(f);
    for (const auto& v : f.mesh.verts) s->mesh_verts.insert(s->mesh_verts.end(), {v.x, v.y, v.z});
    for (const auto& t : f.mesh.tets) s->mesh_tets.insert(s->mesh_tets.end(), t.begin(), t.end());
    s->mesh_mass = f.mass;
    s->mu = f.mu;
    s->lam = f.lam;
    s->n_fem = s->n_blocks = static_cast<Index>(f.mesh.verts.size());
    s->keys.reserve(f.mesh.verts.size() + 10 * f.mesh.tets.size());
    s->vals.reserve(9 * (f.mesh.verts.size() + 10 * f.mesh.tets.size()));
    emit_mass(*s, f);
    emit_tets(*s, f, dt * dt);
    s->pinned.assign(s->n_blocks, 0);
    if (pin_x0)
        for (std::size_t v = 0; v < f.mesh.verts.size(); ++v)
            if (on_x0[v]) s->pinned[v] = 1;
    finish_edges(*s);
    return s;
}

// cfg2: cloth grid (shapes.hpp:21-40) with scatter9 triangle stencils and
// scatter12 hinge stencils; seeded PSD values stand in for the FBW membrane,
// cubic strain limit and bending Hessians (energy/membrane.hpp, bending.hpp).
Scene* cloth(int nx, int ny, double sx, double sy, unsigned seed) {
    auto* s = new Scene();
    std::mt19937 rng(seed);
    const Index n = nx * ny;
    s->n_fem = s->n_blocks = n;
    auto id = [nx](int i, int j) { return static_cast<Index>(j * nx + i); };
    std::vector<std::array<Index, 3>> tris;
    for (int j = 0; j + 1 < ny; ++j)
        for (int i = 0; i + 1 < nx; ++i) {
            if ((i + j) % 2 == 0) {
                tris.push_back({id(i, j), id(i + 1, j), id(i + 1, j + 1)});
                tris.push_back({id(i, j), id(i + 1, j + 1), id(i, j + 1)});
            } else {
                tris.push_back({id(i, j), id(i + 1, j), id(i, j + 1)});
                tris.push_back({id(i + 1, j), id(i + 1, j + 1), id(i, j + 1)});
            }
        }
    // lumped shell masses: rho * area * thickness / 3 (mesh.hpp:150-155)
    const double area = 0.5 * (sx / (nx - 1)) * (sy / (ny - 1));
    std::vector<double> mass(n, 0.0);
    for (const auto& t : tris)
        for (Index v : t) mass[v] += 200.0 * area * 1e-3 / 3;
    for (Index v = 0; v < n; ++v) {
        double b[9] = {mass[v], 0, 0, 0, mass[v], 0, 0, 0, mass[v]};
        s->emit(v, v, b);
    }
    const double dt2 = 1e-4;
    std::normal_distribution<double> nd(0.0, 1.0);
    for (const auto& t : tris) {  // scatter9: 6 blocks per triangle
        double L[81], H[81];
        for (double& v : L) v = nd(rng);
        for (int r = 0; r < 9; ++r)
            for (int c = 0; c < 9; ++c) {
                double acc = 0;
                for (int k = 0; k < 9; ++k) acc += L[9 * k + r] * L[9 * k + c];
                H[9 * c + r] = dt2 * 5e4 * 1e-3 * area * acc / 9.0;
            }
        for (int a = 0; a < 3; ++a)
            for (int b = a; b < 3; ++b) {
                double blk[9];
                for (int c = 0; c < 3; ++c)
                    for (int r = 0; r < 3; ++r) blk[3 * c + r] = H[9 * (3 * b + c) + 3 * a + r];
                s->emit(t[a], t[b], blk);
            }
        for (int a = 0; a < 3; ++a)
            for (int b = a + 1; b < 3; ++b) {
                s->rest_edges.push_back(std::min(t[a], t[b]));
                s->rest_edges.push_back(std::max(t[a], t[b]));
            }
    }
    // hinges: interior edges shared by two triangles (mesh.hpp:100-120)
    std::map<std::uint64_t, std::vector<Index>> opp;
    for (const auto& t : tris)
        for (int e = 0; e < 3; ++e) {
            Index a = t[e], b = t[(e + 1) % 3], o = t[(e + 2) % 3];
            if (a > b) std::swap(a, b);
            opp[(static_cast<std::uint64_t>(a) << 32) | static_cast<std::uint32_t>(b)].push_back(o);
        }
    for (const auto& [k, o] : opp) {
        if (o.size() != 2) continue;
        const Index ids[4] = {static_cast<Index>(k >> 32), static_cast<Index>(k & 0xFFFFFFFFu), o[0], o[1]};
        double H[144];
        random_psd12(rng, dt2 * 1e-2, H);
        emit_stencil12(*s, ids, H, false);
        for (int a = 0; a < 4; ++a)
            for (int b = a + 1; b < 4; ++b) {
                s->rest_edges.push_back(std::min(ids[a], ids[b]));
                s->rest_edges.push_back(std::max(ids[a], ids[b]));
            }
    }
    s->pinned.assign(n, 0);
    s->pinned[id(0, ny - 1)] = 1;  // two top corners (scenes/drape.toml)
    s->pinned[id(nx - 1, ny - 1)] = 1;
    finish_edges(*s);
    return s;
}

// Bodies + FEM parts with contact stencils between neighbouring objects.
// Each object is (kind, index); contact nodes: FEM vertices first, then ABD
// vertices per body (abd_reduce.hpp:9-27 DofMap layout).
Scene* contact_scene(std::vector<FemPart>& fems, std::vector<Body>& bodies, double dt,
                     const std::vector<std::pair<int, int>>& neighbours /* object ids */, int stencils_per_pair,
                     unsigned seed) {
    auto* s = new Scene();
    std::mt19937 rng(seed);
    const double dt2 = dt * dt;
    Index off = 0;
    for (auto& f : fems) {
        f.off = off;
        fem_masses(f);
        off += static_cast<Index>(f.mesh.verts.size());
    }
    s->n_fem = off;
    s->n_bodies = static_cast<Index>(bodies.size());
    s->n_blocks = s->n_fem + 4 * s->n_bodies;
    std::vector<Index> body_node0(bodies.size());
    Index node = s->n_fem;
    double J[36];
    for (std::size_t b = 0; b < bodies.size(); ++b) {
        body_prepare(bodies[b]);
        body_node0[b] = node;
        for (const auto& v : bodies[b].mesh.verts) {
            s->abd_body.push_back(static_cast<Index>(b));
            body_jacobian({v.x + bodies[b].shift.x, v.y + bodies[b].shift.y, v.z + bodies[b].shift.z}, J);
            s->abd_jac.insert(s->abd_jac.end(), J, J + 36);
            ++node;
        }
    }
    for (auto& f : fems) emit_mass(*s, f);
    double M[144];
    for (std::size_t b = 0; b < bodies.size(); ++b) {  // body reduced-mass tiles
        body_mass_matrix(bodies[b], M);
        emit_sym12(*s, s->n_fem + 4 * static_cast<Index>(b), M);
    }
    for (auto& f : fems) emit_tets(*s, f, dt2);
    for (std::size_t b = 0; b < bodies.size(); ++b) {  // orthogonality tiles (PSD stand-in on the A part)
        double H[144] = {0};
        for (int k = 3; k < 12; ++k) H[12 * k + k] = dt2 * bodies[b].kappa * bodies[b].volume * 4.0;
        emit_sym12(*s, s->n_fem + 4 * static_cast<Index>(b), H);
        const Index base = s->n_fem + 4 * static_cast<Index>(b);
        for (int a = 0; a < 4; ++a)
            for (int c = a + 1; c < 4; ++c) {
                s->rest_edges.push_back(base + a);
                s->rest_edges.push_back(base + c);
            }
    }
    // contact stencils: 4 distinct nodes drawn from the two objects
    const int n_fem_objs = static_cast<int>(fems.size());
    auto pick_node = [&](int obj) -> Index {
        if (obj < n_fem_objs) {
            const auto& f = fems[obj];
            std::uniform_int_distribution<Index> u(0, static_cast<Index>(f.mesh.verts.size()) - 1);
            return f.off + u(rng);
        }
        const int b = obj - n_fem_objs;
        std::uniform_int_distribution<Index> u(0, static_cast<Index>(bodies[b].mesh.verts.size()) - 1);
        return body_node0[b] + u(rng);
    };
    for (const auto& [oa, ob] : neighbours)
        for (int k = 0; k < stencils_per_pair; ++k) {
            Index ids[4];
            for (int t = 0; t < 4; ++t) ids[t] = pick_node(t < 2 ? oa : ob);
            if (ids[0] == ids[1] || ids[2] == ids[3]) continue;
            std::sort(ids, ids + 4);
            double H[144];
            random_psd12(rng, dt2 * 1e5, H);
            emit_stencil12(*s, ids, H, true);
        }
    s->pinned.assign(s->n_blocks, 0);
    finish_edges(*s);
    return s;
}

Scene* abd_stack(int bx, int by, int bz, unsigned seed) {  // cfg3
    std::vector<FemPart> fems;
    std::vector<Body> bodies;
    const double size = 0.1, gap = 1e-3;
    for (int k = 0; k < bz; ++k)
        for (int j = 0; j < by; ++j)
            for (int i = 0; i < bx; ++i) {
                Body b{make_box_tets(2, 2, 2, size, size, size), {i * (size + gap), j * (size + gap), k * (size + gap)},
                       1000.0, 1e8, {}, 0};
                bodies.push_back(std::move(b));
            }
    std::vector<std::pair<int, int>> nb;
    auto bid = [&](int i, int j, int k) { return (k * by + j) * bx + i; };
    for (int k = 0; k < bz; ++k)
        for (int j = 0; j < by; ++j)
            for (int i = 0; i < bx; ++i) {
                if (i + 1 < bx) nb.push_back({bid(i, j, k), bid(i + 1, j, k)});
                if (j + 1 < by) nb.push_back({bid(i, j, k), bid(i, j + 1, k)});
                if (k + 1 < bz) nb.push_back({bid(i, j, k), bid(i, j, k + 1)});
            }
    return contact_scene(fems, bodies, 0.01, nb, 20, seed);
}

Scene* hybrid(int n_soft, int soft_res, int n_gears, int gear_res, int stencils_per_pair, double E,
              unsigned seed) {  // cfg4
    std::vector<FemPart> fems;
    std::vector<Body> bodies;
    const double nu = 0.3;
    for (int f = 0; f < n_soft; ++f)
        fems.push_back(FemPart{make_box_tets(soft_res, soft_res, soft_res, 0.2, 0.2, 0.2), 0, E / (2 * (1 + nu)),
                               E * nu / ((1 + nu) * (1 - 2 * nu)), 1000.0, {}});
    for (int g = 0; g < n_gears; ++g)
        bodies.push_back(Body{make_ellipsoid_tets(gear_res, 0.1, 0.05, 0.1), {0.25 * g, 0.3, 0}, 1000.0, 1e8, {}, 0});
    const int n_obj = n_soft + n_gears;
    std::vector<std::pair<int, int>> nb;
    for (int a = 0; a < n_obj; ++a) {  // ring + chords: FEM-FEM, FEM-ABD, ABD-ABD pairs
        nb.push_back({a, (a + 1) % n_obj});
        nb.push_back({a, (a + 3) % n_obj});
    }
    for (auto& p : nb)
        if (p.first > p.second) std::swap(p.first, p.second);
    return contact_scene(fems, bodies, 0.01, nb, stencils_per_pair, seed);
}

}  // namespace

extern "C" {

void* adipc_scene_fem_box(int nx, int ny, int nz, double sx, double sy, double sz, double E, double nu, double rho,
                          double dt, int pin_x0, double jitter, unsigned seed) {
    return fem_box(nx, ny, nz, sx, sy, sz, E, nu, rho, dt, pin_x0, jitter, seed);
}
void* adipc_scene_cloth(int nx, int ny, double sx, double sy, unsigned seed) { return cloth(nx, ny, sx, sy, seed); }
void* adipc_scene_abd_stack(int bx, int by, int bz, unsigned seed) { return abd_stack(bx, by, bz, seed); }
void* adipc_scene_hybrid(int n_soft, int soft_res, int n_gears, int gear_res, int stencils_per_pair, double E,
                         unsigned seed) {
    return hybrid(n_soft, soft_res, n_gears, gear_res, stencils_per_pair, E, seed);
}
void adipc_scene_free(void* s) { delete static_cast<Scene*>(s); }

// the solid mesh of a FEM-only scene: out = {n_verts, n_tets}; mat = {mu, lambda}
void adipc_scene_mesh_sizes(void* sp, std::int64_t* out, double* mat) {
    const Scene& s = *static_cast<Scene*>(sp);
    out[0] = static_cast<std::int64_t>(s.mesh_mass.size());
    out[1] = static_cast<std::int64_t>(s.mesh_tets.size() / 4);
    mat[0] = s.mu;
    mat[1] = s.lam;
}
void adipc_scene_copy_mesh(void* sp, double* verts, std::int32_t* tets, double* mass) {
    const Scene& s = *static_cast<Scene*>(sp);
    if (!s.mesh_verts.empty()) std::memcpy(verts, s.mesh_verts.data(), 8 * s.mesh_verts.size());
    if (!s.mesh_tets.empty()) std::memcpy(tets, s.mesh_tets.data(), 4 * s.mesh_tets.size());
    if (!s.mesh_mass.empty()) std::memcpy(mass, s.mesh_mass.data(), 8 * s.mesh_mass.size());
}

// out: n_blocks, n_fem, n_bodies, n_abd_nodes, T, Tn, n_rest_edges
void adipc_scene_sizes(void* sp, std::int64_t* out) {
    const Scene& s = *static_cast<Scene*>(sp);
    out[0] = s.n_blocks;
    out[1] = s.n_fem;
    out[2] = s.n_bodies;
    out[3] = static_cast<std::int64_t>(s.abd_body.size());
    out[4] = static_cast<std::int64_t>(s.keys.size());
    out[5] = static_cast<std::int64_t>(s.node_keys.size());
    out[6] = static_cast<std::int64_t>(s.rest_edges.size() / 2);
}

void adipc_scene_copy(void* sp, std::uint64_t* keys, double* vals, std::uint64_t* node_keys, double* node_vals,
                      std::int32_t* abd_body, double* jac36, std::uint8_t* pinned, std::int32_t* rest_edges) {
    const Scene& s = *static_cast<Scene*>(sp);
    auto cp = [](void* dst, const void* src, std::size_t bytes) {
        if (dst && bytes) std::memcpy(dst, src, bytes);
    };
    cp(keys, s.keys.data(), 8 * s.keys.size());
    cp(vals, s.vals.data(), 8 * s.vals.size());
    cp(node_keys, s.node_keys.data(), 8 * s.node_keys.size());
    cp(node_vals, s.node_vals.data(), 8 * s.node_vals.size());
    cp(abd_body, s.abd_body.data(), 4 * s.abd_body.size());
    cp(jac36, s.abd_jac.data(), 8 * s.abd_jac.size());
    cp(pinned, s.pinned.data(), s.pinned.size());
    cp(rest_edges, s.rest_edges.data(), 4 * s.rest_edges.size());
}

}  // extern "C"
