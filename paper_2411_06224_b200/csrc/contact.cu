// Device contact producers: the contact-node part of
// IncrementalPotential::assemble_contact (solver/incremental_potential.hpp:
// 322-384) for given candidate stencils — point-triangle and edge-edge barrier
// stencils (closest-feature classification + per-feature squared distance
// with first and second derivatives, contact/distance.hpp:13-223; log barrier
// chain rule + PSD projection, contact/barrier.hpp:14-66), the ground
// half-space barrier (barrier.hpp:70-91) and lagged friction
// (contact/friction.hpp:12-91) — written as the node stream in the
// reference's emission order (active PT pairs, active EE pairs, ground
// contacts, friction constraints), which adipc_gpu_assemble_contact_device
// feeds through two_level_abd_reduce on the device. Plus the contact terms of
// the line-search value (incremental_potential.hpp:133-157) and the
// conservative-advancement CCD step bound (contact/ccd.hpp:17-110).
//
// A value-only pass classifies every candidate and flags it active when the
// feature's squared distance (the duals' value arithmetic, bitwise) is below
// dhat^2 — the reference's test on pd.dist2 — a prefix sum compacts the
// active pairs, and the derivative pass runs one thread per ACTIVE pair. The
// reference differentiates with second-order duals over the 12 stencil
// coordinates (core/dual2.hpp); the derivative pass here uses the closed
// forms of dist_derivs.cuh over the feature's 1-3 difference vectors (the
// same derivatives to rounding, without a 91-double dual per intermediate).
#include <cmath>
#include <cstring>
#include <limits>

#include "context.hpp"
#include "dist_derivs.cuh"
#include "psd.cuh"
#include "scan.cuh"

namespace adipc_gpu {

namespace {

constexpr int kContactThreads = 128;

// ---- plain-double classification and value paths (distance.hpp:13-155) ----
struct V3 {
    double x, y, z;
};
__device__ __forceinline__ V3 vsub(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
__device__ __forceinline__ double vdot(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
__device__ __forceinline__ V3 vcross(V3 a, V3 b) {
    return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
__device__ __forceinline__ V3 ld(const double* pos, int v) {
    return {pos[3 * static_cast<std::int64_t>(v)], pos[3 * static_cast<std::int64_t>(v) + 1],
            pos[3 * static_cast<std::int64_t>(v) + 2]};
}

// PtRegion: 0 V0, 1 V1, 2 V2, 3 E01, 4 E12, 5 E20, 6 Interior
__device__ int classify_pt(V3 p, V3 t0, V3 t1, V3 t2, double* beta) {
    const V3 ab = vsub(t1, t0), ac = vsub(t2, t0), ap = vsub(p, t0);
    const double d1 = vdot(ab, ap), d2 = vdot(ac, ap);
    if (d1 <= 0 && d2 <= 0) {
        beta[0] = 1, beta[1] = 0, beta[2] = 0;
        return 0;
    }
    const V3 bp = vsub(p, t1);
    const double d3 = vdot(ab, bp), d4 = vdot(ac, bp);
    if (d3 >= 0 && d4 <= d3) {
        beta[0] = 0, beta[1] = 1, beta[2] = 0;
        return 1;
    }
    const double vc = d1 * d4 - d3 * d2;
    if (vc <= 0 && d1 >= 0 && d3 <= 0) {
        const double v = d1 / (d1 - d3);
        beta[0] = 1 - v, beta[1] = v, beta[2] = 0;
        return 3;
    }
    const V3 cp = vsub(p, t2);
    const double d5 = vdot(ab, cp), d6 = vdot(ac, cp);
    if (d6 >= 0 && d5 <= d6) {
        beta[0] = 0, beta[1] = 0, beta[2] = 1;
        return 2;
    }
    const double vb = d5 * d2 - d1 * d6;
    if (vb <= 0 && d2 >= 0 && d6 <= 0) {
        const double w = d2 / (d2 - d6);
        beta[0] = 1 - w, beta[1] = 0, beta[2] = w;
        return 5;
    }
    const double va = d3 * d6 - d5 * d4;
    if (va <= 0 && d4 - d3 >= 0 && d5 - d6 >= 0) {
        const double w = (d4 - d3) / ((d4 - d3) + (d5 - d6));
        beta[0] = 0, beta[1] = 1 - w, beta[2] = w;
        return 4;
    }
    const double denom = 1.0 / (va + vb + vc);
    const double v = vb * denom, w = vc * denom;
    beta[0] = 1 - v - w, beta[1] = v, beta[2] = w;
    return 6;
}

// EeRegion: 0 A0B0, 1 A0B1, 2 A1B0, 3 A1B1, 4 A0Int, 5 A1Int, 6 IntB0, 7 IntB1, 8 Interior
__device__ int classify_ee(V3 a0, V3 a1, V3 b0, V3 b1, double* s_out, double* t_out) {
    const V3 da = vsub(a1, a0), db = vsub(b1, b0), r = vsub(a0, b0);
    const double a = vdot(da, da), e = vdot(db, db);
    const double f = vdot(db, r), c = vdot(da, r), b = vdot(da, db);
    const double denom = a * e - b * b;
    double s = 0;
    bool s_int = false;
    if (denom > 1e-12 * a * e) {
        s = (b * f - c * e) / denom;
        if (s <= 0)
            s = 0;
        else if (s >= 1)
            s = 1;
        else
            s_int = true;
    }
    double t = e > 0 ? (b * s + f) / e : 0;
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
        s_int = s > 0 && s < 1;
        if (s <= 0)
            s = 0;
        else if (s >= 1)
            s = 1;
    }
    *s_out = s;
    *t_out = t;
    const bool s_end = !s_int, t_end = t == 0 || t == 1;
    if (s_end && t_end) return s == 0 ? (t == 0 ? 0 : 1) : (t == 0 ? 2 : 3);
    if (s_end) return s == 0 ? 4 : 5;
    if (t_end) return t == 0 ? 6 : 7;
    return 8;
}

// the dual's value of the active feature, in plain doubles (same arithmetic)
__device__ double pp_v(V3 a, V3 b) {
    const V3 d = vsub(a, b);
    return (d.x * d.x + d.y * d.y) + d.z * d.z;
}
__device__ double pe_v(V3 p, V3 e0, V3 e1) {
    const V3 d = vsub(e1, e0), w = vsub(p, e0);
    const V3 c = vcross(w, d);
    return ((c.x * c.x + c.y * c.y) + c.z * c.z) * (1.0 / ((d.x * d.x + d.y * d.y) + d.z * d.z));
}
__device__ double hn_v(V3 q0, V3 q1, V3 r0, V3 r1, V3 o, V3 base) {
    const V3 n = vcross(vsub(q1, q0), vsub(r1, r0));
    const V3 u = vsub(o, base);
    const double h = (u.x * n.x + u.y * n.y) + u.z * n.z;
    return (h * h) * (1.0 / ((n.x * n.x + n.y * n.y) + n.z * n.z));
}
// stencil x[4]: kind 0 PT (p, t0, t1, t2), 1 EE (a0, a1, b0, b1)
__device__ double feature_dist2(int kind, const V3* x, int* region) {
    double b3[3], s, t;
    if (kind == 0) {
        const int r = classify_pt(x[0], x[1], x[2], x[3], b3);
        *region = r;
        switch (r) {
            case 0: return pp_v(x[0], x[1]);
            case 1: return pp_v(x[0], x[2]);
            case 2: return pp_v(x[0], x[3]);
            case 3: return pe_v(x[0], x[1], x[2]);
            case 4: return pe_v(x[0], x[2], x[3]);
            case 5: return pe_v(x[0], x[3], x[1]);
            default: return hn_v(x[1], x[2], x[1], x[3], x[0], x[1]);
        }
    }
    const int r = classify_ee(x[0], x[1], x[2], x[3], &s, &t);
    *region = r;
    switch (r) {
        case 0: return pp_v(x[0], x[2]);
        case 1: return pp_v(x[0], x[3]);
        case 2: return pp_v(x[1], x[2]);
        case 3: return pp_v(x[1], x[3]);
        case 4: return pe_v(x[0], x[2], x[3]);
        case 5: return pe_v(x[1], x[2], x[3]);
        case 6: return pe_v(x[2], x[0], x[1]);
        case 7: return pe_v(x[3], x[0], x[1]);
        default: return hn_v(x[0], x[1], x[2], x[3], x[2], x[0]);
    }
}
// the same feature's squared distance with derivatives (result in W.s0)
// the closest-point value path of pt_dist2 / ee_dist2 (ccd, line-search value)
__device__ double closest_dist2(int kind, const V3* x) {
    if (kind == 0) {
        double b3[3];
        classify_pt(x[0], x[1], x[2], x[3], b3);
        const V3 c = {b3[0] * x[1].x + b3[1] * x[2].x + b3[2] * x[3].x, b3[0] * x[1].y + b3[1] * x[2].y + b3[2] * x[3].y,
                      b3[0] * x[1].z + b3[1] * x[2].z + b3[2] * x[3].z};
        const V3 d = vsub(x[0], c);
        return vdot(d, d);
    }
    double s, t;
    classify_ee(x[0], x[1], x[2], x[3], &s, &t);
    const V3 pa = {x[0].x + s * (x[1].x - x[0].x), x[0].y + s * (x[1].y - x[0].y), x[0].z + s * (x[1].z - x[0].z)};
    const V3 pb = {x[2].x + t * (x[3].x - x[2].x), x[2].y + t * (x[3].y - x[2].y), x[2].z + t * (x[3].z - x[2].z)};
    const V3 d = vsub(pa, pb);
    return vdot(d, d);
}

// barrier.hpp:14-31
__device__ double barrier_value(double s, double shat, double kappa) {
    if (s >= shat) return 0;
    const double r = s - shat;
    return -kappa * r * r * log(s / shat);
}
__device__ double barrier_d1(double s, double shat, double kappa) {
    if (s >= shat) return 0;
    const double r = s - shat;
    return -kappa * (2 * r * log(s / shat) + r * r / s);
}
__device__ double barrier_d2(double s, double shat, double kappa) {
    if (s >= shat) return 0;
    const double r = s - shat;
    return -kappa * (2 * log(s / shat) + 4 * r / s - r * r / (s * s));
}

__device__ __forceinline__ void load_stencil(const double* pos, const int* st, V3* x) {
    for (int a = 0; a < 4; ++a) x[a] = ld(pos, st[a]);
}
__device__ __forceinline__ void emit_block(std::uint64_t* keys, double* vals, std::int64_t q, int ra, int rb,
                                           const double* blk /*3x3 col-major of (ra, rb)*/) {
    const bool flip = ra > rb;
    const std::uint32_t r0 = static_cast<std::uint32_t>(flip ? rb : ra), c0 = static_cast<std::uint32_t>(flip ? ra : rb);
    keys[q] = (static_cast<std::uint64_t>(r0) << 32) | c0;
    double* o = vals + 9 * q;
    for (int c = 0; c < 3; ++c)
        for (int r = 0; r < 3; ++r) o[3 * c + r] = flip ? blk[3 * r + c] : blk[3 * c + r];
}

struct ContactArgs {
    const double* pos;
    std::int64_t n_pt, n_ee;
    const int* pt;
    const int* ee;
    double dhat, kappa, dt2;
    int ground;
    double gn[3], gh;
    std::int32_t n_sv;
    const int* sv;
    std::int64_t n_fr;
    const int* fr_nodes;
    const int* fr_n;
    const double* fr_coeff;
    const double* fr_t1;
    const double* fr_t2;
    const double* fr_lambda;
    const double* fr_base;
    double mu, fr_eps;
    int project;
};

__device__ __forceinline__ const int* stencil_of(const ContactArgs& a, std::int64_t i, int* kind) {
    *kind = i < a.n_pt ? 0 : 1;
    return i < a.n_pt ? a.pt + 4 * i : a.ee + 4 * (i - a.n_pt);
}

// pass 1: active flags (the reference keeps a pair iff pd.dist2 < shat) and
// ground activity (0 < d < dhat)
__global__ void k_contact_active(ContactArgs a, std::int32_t* __restrict__ pair_on, std::int32_t* __restrict__ gnd_on) {
    const double shat = a.dhat * a.dhat;
    const std::int64_t np = a.n_pt + a.n_ee;
    for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < np + a.n_sv;
         i += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        if (i < np) {
            int kind, region;
            V3 x[4];
            load_stencil(a.pos, stencil_of(a, i, &kind), x);
            pair_on[i] = feature_dist2(kind, x, &region) < shat ? 1 : 0;
        } else {
            const V3 p = ld(a.pos, a.sv[i - np]);
            const double d = (a.gn[0] * p.x + a.gn[1] * p.y) + a.gn[2] * p.z - a.gh;
            gnd_on[i - np] = (d > 0 && d < a.dhat) ? 1 : 0;
        }
    }
}

// active pair indices in emission order (list[rank[i]] = i)
__global__ void k_active_list(const std::int32_t* __restrict__ on, const std::int64_t* __restrict__ rank,
                              std::int64_t n, std::int64_t* __restrict__ list) {
    for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<std::int64_t>(gridDim.x) * blockDim.x)
        if (on[i]) list[rank[i]] = i;
}

// pass 2: one thread per active pair -> 10 blocks at 10 * rank, node
// gradient, value. The feature's derivatives in closed form over its
// difference vectors (dist_derivs.cuh) and the barrier chain rule there
// (Hf = b2 g g^T + b1 d2(dist2)); the PSD test / projection on the reduction
// to the 9-dimensional complement of the translations (the 12 x 12 S^T Hf S
// is never formed), the blocks emitted from Hf (already PSD) or from the
// projected reduction
__global__ void __launch_bounds__(kContactThreads) k_contact_pairs(ContactArgs a, const std::int64_t* __restrict__ list,
                                                                   std::int64_t n_active,
                                                                   std::uint64_t* __restrict__ keys,
                                                                   double* __restrict__ vals,
                                                                   double* __restrict__ node_grad,
                                                                   double* __restrict__ value) {
    const double shat = a.dhat * a.dhat;
    double e = 0;
    for (std::int64_t j = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; j < n_active;
         j += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        const std::int64_t i = list[j];
        int kind, region;
        const int* st = stencil_of(a, i, &kind);
        V3 xv[4];
        load_stencil(a.pos, st, xv);
        feature_dist2(kind, xv, &region);
        double x[12];
        for (int n = 0; n < 4; ++n) {
            x[3 * n] = xv[n].x;
            x[3 * n + 1] = xv[n].y;
            x[3 * n + 2] = xv[n].z;
        }
        FeatDerivs f;
        feature_derivs(kind, region, x, f);
        const double b1 = barrier_d1(f.v, shat, a.kappa), b2 = barrier_d2(f.v, shat, a.kappa);
        e += barrier_value(f.v, shat, a.kappa);
        const int m = 3 * f.nvec;
        for (int c = 0; c < m; ++c)
            for (int r = 0; r < m; ++r) f.H[9 * c + r] = b2 * (f.g[r] * f.g[c]) + b1 * f.H[9 * c + r];
        // node coefficients of the feature vectors, and R = S (Q (x) I3):
        // the 9-dimensional translation complement straight from the
        // feature space (M = R^T Hf R, no 12 x 12)
        double C[4][3], R[3][3];
        for (int n = 0; n < 4; ++n)
            for (int p = 0; p < 3; ++p) C[n][p] = p < f.nvec ? feat_coef(f, p, n) : 0.0;
        for (int p = 0; p < 3; ++p)
            for (int j = 0; j < 3; ++j) {
                double r = 0;
                for (int n = 0; n < 4; ++n) r += C[n][p] * helmert(n, j);
                R[p][j] = r;
            }
        for (int n = 0; n < 4; ++n)
            for (int k = 0; k < 3; ++k) {
                double gk = 0;
                for (int p = 0; p < f.nvec; ++p) gk += C[n][p] * f.g[3 * p + k];
                red_add_f64(node_grad + 3 * static_cast<std::int64_t>(st[n]) + k, a.dt2 * (b1 * gk));
            }
        bool projected = false;
        double M[81];
        if (a.project) {
            for (int l = 0; l < 3; ++l)
                for (int c = 0; c < 3; ++c)
                    for (int j = 0; j < 3; ++j)
                        for (int r = 0; r < 3; ++r) {
                            double sum = 0;
                            for (int q = 0; q < f.nvec; ++q)
                                for (int p = 0; p < f.nvec; ++p)
                                    sum += R[p][j] * R[q][l] * f.H[9 * (3 * q + c) + 3 * p + r];
                            M[9 * (3 * l + c) + 3 * j + r] = sum;
                        }
            if (!psd9(M)) {
                project9(M);
                projected = true;
            }
        }
        const std::int64_t base = 10 * j;
        int q = 0;
        for (int p0 = 0; p0 < 4; ++p0)
            for (int p1 = p0; p1 < 4; ++p1, ++q) {
                double blk[9];
                for (int c = 0; c < 3; ++c)
                    for (int r = 0; r < 3; ++r) {
                        double sum = 0;
                        if (projected) {  // (Q (x) I3) proj(M) (Q (x) I3)^T, block (p0, p1)
                            for (int l = 0; l < 3; ++l)
                                for (int jj = 0; jj < 3; ++jj)
                                    sum += helmert(p0, jj) * helmert(p1, l) * M[9 * (3 * l + c) + 3 * jj + r];
                        } else {  // S^T Hf S, block (p0, p1)
                            for (int qq = 0; qq < f.nvec; ++qq)
                                for (int p = 0; p < f.nvec; ++p)
                                    sum += C[p0][p] * C[p1][qq] * f.H[9 * (3 * qq + c) + 3 * p + r];
                        }
                        blk[3 * c + r] = a.dt2 * sum;
                    }
                emit_block(keys, vals, base + q, st[p0], st[p1], blk);
            }
    }
    block_sum_atomic(a.dt2 * e, value);
}

// ground half-space barrier (barrier.hpp:70-91), one diagonal block per
// active surface vertex, after the pairs
__global__ void k_contact_ground(ContactArgs a, const std::int32_t* __restrict__ on,
                                 const std::int64_t* __restrict__ rank, std::int64_t base,
                                 std::uint64_t* __restrict__ keys, double* __restrict__ vals,
                                 double* __restrict__ node_grad, double* __restrict__ value) {
    const double shat = a.dhat * a.dhat;
    double e = 0;
    for (std::int64_t j = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; j < a.n_sv;
         j += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        if (!on[j]) continue;
        const int v = a.sv[j];
        const V3 p = ld(a.pos, v);
        const double dist = (a.gn[0] * p.x + a.gn[1] * p.y) + a.gn[2] * p.z - a.gh;
        const double s = dist * dist;
        e += barrier_value(s, shat, a.kappa);
        const double gs = barrier_d1(s, shat, a.kappa) * 2 * dist;
        for (int k = 0; k < 3; ++k) red_add_f64(node_grad + 3 * static_cast<std::int64_t>(v) + k, a.dt2 * (gs * a.gn[k]));
        const double sd = dist * dist;
        double c = 4 * sd * barrier_d2(sd, a.dhat * a.dhat, a.kappa) + 2 * barrier_d1(sd, a.dhat * a.dhat, a.kappa);
        if (a.project && c < 0) c = 0;
        double blk[9];
        for (int cc = 0; cc < 3; ++cc)
            for (int r = 0; r < 3; ++r) blk[3 * cc + r] = a.dt2 * ((c * a.gn[r]) * a.gn[cc]);
        emit_block(keys, vals, base + rank[j], v, v, blk);
    }
    block_sum_atomic(a.dt2 * e, value);
}

// friction.hpp:12-36
__device__ double fr_f0(double y, double eps) { return y >= eps ? y : -y * y * y / (3 * eps * eps) + y * y / eps + eps / 3; }
__device__ double fr_f1(double y, double eps) { return y >= eps ? 1 : y * (2 * eps - y) / (eps * eps); }
__device__ double fr_f1y(double y, double eps) { return y >= eps ? 1 / y : (2 * eps - y) / (eps * eps); }
__device__ double fr_f2(double y, double eps) { return y >= eps ? 0 : 2 * (eps - y) / (eps * eps); }

// lagged friction (friction.hpp:58-91), n (n + 1) / 2 blocks per constraint
__global__ void k_contact_friction(ContactArgs a, const std::int64_t* __restrict__ off, std::int64_t base,
                                   std::uint64_t* __restrict__ keys, double* __restrict__ vals,
                                   double* __restrict__ node_grad, double* __restrict__ value) {
    double e = 0;
    for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < a.n_fr;
         i += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        const int n = a.fr_n[i];
        const int* nodes = a.fr_nodes + 4 * i;
        const double* co = a.fr_coeff + 4 * i;
        const V3 t1 = {a.fr_t1[3 * i], a.fr_t1[3 * i + 1], a.fr_t1[3 * i + 2]};
        const V3 t2 = {a.fr_t2[3 * i], a.fr_t2[3 * i + 1], a.fr_t2[3 * i + 2]};
        V3 w = {0, 0, 0};
        for (int k = 0; k < n; ++k) {
            const V3 dx = vsub(ld(a.pos, nodes[k]), ld(a.fr_base, nodes[k]));
            w = {w.x + co[k] * dx.x, w.y + co[k] * dx.y, w.z + co[k] * dx.z};
        }
        const double u0 = vdot(t1, w), u1 = vdot(t2, w);
        const double y = sqrt(u0 * u0 + u1 * u1);
        const double scale = a.mu * a.fr_lambda[i];
        e += scale * fr_f0(y, a.fr_eps);
        double in[4];
        V3 gw = {0, 0, 0};
        if (y > 1e-14 * a.fr_eps) {
            const double h0 = u0 / y, h1 = u1 / y, f1 = scale * fr_f1(y, a.fr_eps);
            gw = {f1 * (t1.x * h0 + t2.x * h1), f1 * (t1.y * h0 + t2.y * h1), f1 * (t1.z * h0 + t2.z * h1)};
            const double f2 = fr_f2(y, a.fr_eps), fy = fr_f1y(y, a.fr_eps);
            in[0] = scale * (f2 * (h0 * h0) + fy * (1 - h0 * h0));
            in[1] = scale * (f2 * (h1 * h0) + fy * (0 - h1 * h0));
            in[2] = scale * (f2 * (h0 * h1) + fy * (0 - h0 * h1));
            in[3] = scale * (f2 * (h1 * h1) + fy * (1 - h1 * h1));
        } else {
            const double fy = scale * fr_f1y(0, a.fr_eps);
            in[0] = fy, in[1] = 0, in[2] = 0, in[3] = fy;
        }
        const double T1[3] = {t1.x, t1.y, t1.z}, T2[3] = {t2.x, t2.y, t2.z}, G[3] = {gw.x, gw.y, gw.z};
        double hw[9];
        for (int j = 0; j < 3; ++j)
            for (int r = 0; r < 3; ++r) {
                const double q0 = in[0] * T1[j] + in[2] * T2[j], q1 = in[1] * T1[j] + in[3] * T2[j];
                hw[3 * j + r] = T1[r] * q0 + T2[r] * q1;
            }
        for (int k = 0; k < n; ++k)
            for (int c = 0; c < 3; ++c)
                red_add_f64(node_grad + 3 * static_cast<std::int64_t>(nodes[k]) + c, a.dt2 * (co[k] * G[c]));
        std::int64_t q = base + off[i];
        for (int p0 = 0; p0 < n; ++p0)
            for (int p1 = p0; p1 < n; ++p1, ++q) {
                double blk[9];
                for (int m = 0; m < 9; ++m) blk[m] = a.dt2 * (co[p0] * co[p1] * hw[m]);
                emit_block(keys, vals, q, nodes[p0], nodes[p1], blk);
            }
    }
    block_sum_atomic(a.dt2 * e, value);
}

__global__ void k_friction_blocks(const int* __restrict__ fr_n, std::int64_t n, std::int32_t* __restrict__ cnt) {
    for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<std::int64_t>(gridDim.x) * blockDim.x)
        cnt[i] = fr_n[i] * (fr_n[i] + 1) / 2;
}

// contact terms of IncrementalPotential::value (:133-157): flag[0] = 1 when a
// stencil or a surface vertex touches (the value is +inf)
__global__ void k_contact_value(ContactArgs a, double* __restrict__ value, int* __restrict__ touch) {
    const double shat = a.dhat * a.dhat;
    const std::int64_t np = a.n_pt + a.n_ee;
    double e = 0;
    for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < np + a.n_sv + a.n_fr;
         i += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        if (i < np) {
            int kind;
            V3 x[4];
            load_stencil(a.pos, stencil_of(a, i, &kind), x);
            const double d2 = closest_dist2(kind, x);
            if (d2 <= 0) atomicOr(touch, 1);
            if (d2 < shat) e += barrier_value(d2, shat, a.kappa);
        } else if (i < np + a.n_sv) {
            const V3 p = ld(a.pos, a.sv[i - np]);
            const double d = (a.gn[0] * p.x + a.gn[1] * p.y) + a.gn[2] * p.z - a.gh;
            if (d <= 0) atomicOr(touch, 1);
            if (d < a.dhat) e += barrier_value(d * d, shat, a.kappa);
        } else {
            const std::int64_t f = i - np - a.n_sv;
            const int* nodes = a.fr_nodes + 4 * f;
            const double* co = a.fr_coeff + 4 * f;
            V3 w = {0, 0, 0};
            for (int k = 0; k < a.fr_n[f]; ++k) {
                const V3 dx = vsub(ld(a.pos, nodes[k]), ld(a.fr_base, nodes[k]));
                w = {w.x + co[k] * dx.x, w.y + co[k] * dx.y, w.z + co[k] * dx.z};
            }
            const V3 t1 = {a.fr_t1[3 * f], a.fr_t1[3 * f + 1], a.fr_t1[3 * f + 2]};
            const V3 t2 = {a.fr_t2[3 * f], a.fr_t2[3 * f + 1], a.fr_t2[3 * f + 2]};
            const double u0 = vdot(t1, w), u1 = vdot(t2, w);
            e += a.mu * a.fr_lambda[f] * fr_f0(sqrt(u0 * u0 + u1 * u1), a.fr_eps);
        }
    }
    block_sum_atomic(a.dt2 * e, value);
}

// contact/ccd.hpp:17-56, 80-86: conservative advancement per stencil, ground
// closing time per surface vertex; the step bound is the minimum (atomicMin on
// the bit pattern of non-negative doubles)
constexpr double kCcdGap = 0.01, kCcdRescale = 0.9;
constexpr int kCcdMaxIters = 64;
__device__ double conservative_toi(int kind, const V3* x, V3* d) {
    const int n_side_a = kind == 0 ? 1 : 2;
    V3 mean = {0, 0, 0};
    for (int i = 0; i < 4; ++i) mean = {mean.x + d[i].x, mean.y + d[i].y, mean.z + d[i].z};
    mean = {mean.x / 4, mean.y / 4, mean.z / 4};
    double max_a = 0, max_b = 0;
    for (int i = 0; i < 4; ++i) {
        d[i] = vsub(d[i], mean);
        const double len = sqrt(vdot(d[i], d[i]));
        if (i < n_side_a)
            max_a = fmax(max_a, len);
        else
            max_b = fmax(max_b, len);
    }
    const double speed = max_a + max_b;
    if (speed == 0) return 1;
    const double g0 = sqrt(closest_dist2(kind, x));
    if (!(g0 > 0)) return 0;
    const double gap = kCcdGap * g0;
    double t = 0;
    V3 cur[4] = {x[0], x[1], x[2], x[3]};
    for (int it = 0; it < kCcdMaxIters; ++it) {
        const double g = sqrt(closest_dist2(kind, cur));
        if (g <= gap) return kCcdRescale * t;
        const double step = (g - gap) / speed;
        if (t + step >= 1) return 1;
        t += step;
        for (int i = 0; i < 4; ++i) cur[i] = {x[i].x + t * d[i].x, x[i].y + t * d[i].y, x[i].z + t * d[i].z};
    }
    return kCcdRescale * t;
}
__global__ void k_ccd(ContactArgs a, const double* __restrict__ disp, unsigned long long* __restrict__ alpha) {
    const std::int64_t np = a.n_pt + a.n_ee;
    double best = 1;
    for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < np + a.n_sv;
         i += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        if (i < np) {
            int kind;
            const int* st = stencil_of(a, i, &kind);
            V3 x[4], d[4];
            load_stencil(a.pos, st, x);
            load_stencil(disp, st, d);
            best = fmin(best, conservative_toi(kind, x, d));
        } else if (a.ground) {
            const int v = a.sv[i - np];
            const V3 p = ld(a.pos, v), dp = ld(disp, v);
            const double g0 = (a.gn[0] * p.x + a.gn[1] * p.y) + a.gn[2] * p.z - a.gh;
            double toi;
            if (!(g0 > 0)) {
                toi = 0;
            } else {
                const double closing = -((a.gn[0] * dp.x + a.gn[1] * dp.y) + a.gn[2] * dp.z);
                if (closing <= 0) {
                    toi = 1;
                } else {
                    const double t_gap = (1 - kCcdGap) * g0 / closing;
                    toi = t_gap >= 1 ? 1 : kCcdRescale * t_gap;
                }
            }
            best = fmin(best, toi);
        }
    }
    for (int o = 16; o > 0; o >>= 1) best = fmin(best, __shfl_xor_sync(0xffffffffu, best, o));
    if ((threadIdx.x & 31) == 0) atomicMin(alpha, static_cast<unsigned long long>(__double_as_longlong(best)));
}

// ---- friction constraints at the step start (friction.hpp:43-149) -----------
// the frame of candidate i (distance.hpp:226-256) or ground contact j:
// distance, unit normal, coefficients; false when not in contact range
__device__ bool friction_frame(const ContactArgs& a, std::int64_t i, double* dist, double* nrm, double* coeff,
                               int* nodes, int* n_nodes) {
    const std::int64_t np = a.n_pt + a.n_ee;
    if (i >= np) {
        const int v = a.sv[i - np];
        const V3 p = ld(a.pos, v);
        const double dd = (a.gn[0] * p.x + a.gn[1] * p.y) + a.gn[2] * p.z - a.gh;
        *dist = dd;
        nrm[0] = a.gn[0];
        nrm[1] = a.gn[1];
        nrm[2] = a.gn[2];
        nodes[0] = v;
        nodes[1] = nodes[2] = nodes[3] = -1;
        coeff[0] = 1;
        coeff[1] = coeff[2] = coeff[3] = 0;
        *n_nodes = 1;
        return dd > 0 && dd < a.dhat;
    }
    int kind;
    const int* st = stencil_of(a, i, &kind);
    V3 x[4];
    load_stencil(a.pos, st, x);
    double d[3];
    if (kind == 0) {
        double b[3];
        classify_pt(x[0], x[1], x[2], x[3], b);
        d[0] = x[0].x - ((b[0] * x[1].x + b[1] * x[2].x) + b[2] * x[3].x);
        d[1] = x[0].y - ((b[0] * x[1].y + b[1] * x[2].y) + b[2] * x[3].y);
        d[2] = x[0].z - ((b[0] * x[1].z + b[1] * x[2].z) + b[2] * x[3].z);
        coeff[0] = 1;
        coeff[1] = -b[0];
        coeff[2] = -b[1];
        coeff[3] = -b[2];
    } else {
        double sv, tv;
        classify_ee(x[0], x[1], x[2], x[3], &sv, &tv);
        d[0] = (x[0].x + sv * (x[1].x - x[0].x)) - (x[2].x + tv * (x[3].x - x[2].x));
        d[1] = (x[0].y + sv * (x[1].y - x[0].y)) - (x[2].y + tv * (x[3].y - x[2].y));
        d[2] = (x[0].z + sv * (x[1].z - x[0].z)) - (x[2].z + tv * (x[3].z - x[2].z));
        coeff[0] = 1 - sv;
        coeff[1] = sv;
        coeff[2] = -(1 - tv);
        coeff[3] = -tv;
    }
    const double dn = sqrt((d[0] * d[0] + d[1] * d[1]) + d[2] * d[2]);
    *dist = dn;
    if (dn > 0) {
        nrm[0] = d[0] / dn;
        nrm[1] = d[1] / dn;
        nrm[2] = d[2] / dn;
    } else {
        nrm[0] = 0;
        nrm[1] = 1;
        nrm[2] = 0;
    }
    for (int k = 0; k < 4; ++k) nodes[k] = st[k];
    *n_nodes = 4;
    return dn > 0 && dn < a.dhat;
}

__global__ void k_friction_flags(ContactArgs a, std::int64_t n, std::int32_t* __restrict__ on) {
    for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        double dist, nrm[3], coeff[4];
        int nodes[4], nn;
        on[i] = friction_frame(a, i, &dist, nrm, coeff, nodes, &nn) ? 1 : 0;
    }
}

__global__ void k_friction_emit(ContactArgs a, std::int64_t n, const std::int32_t* __restrict__ on,
                                const std::int64_t* __restrict__ rank, std::int32_t* __restrict__ o_nodes,
                                std::int32_t* __restrict__ o_n, double* __restrict__ o_coeff,
                                double* __restrict__ o_t1, double* __restrict__ o_t2, double* __restrict__ o_lambda) {
    const double shat = a.dhat * a.dhat;
    for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        if (!on[i]) continue;
        double dist, nrm[3], coeff[4];
        int nodes[4], nn;
        friction_frame(a, i, &dist, nrm, coeff, nodes, &nn);
        const std::int64_t q = rank[i];
        // tangent_basis (friction.hpp:43-47): t1 = normalized(n x ref), t2 = n x t1
        const bool ydir = fabs(nrm[0]) > 0.9;
        double u[3];
        if (ydir) {  // ref = (0, 1, 0)
            u[0] = nrm[1] * 0.0 - nrm[2] * 1.0;
            u[1] = nrm[2] * 0.0 - nrm[0] * 0.0;
            u[2] = nrm[0] * 1.0 - nrm[1] * 0.0;
        } else {  // ref = (1, 0, 0)
            u[0] = nrm[1] * 0.0 - nrm[2] * 0.0;
            u[1] = nrm[2] * 1.0 - nrm[0] * 0.0;
            u[2] = nrm[0] * 0.0 - nrm[1] * 1.0;
        }
        const double z = (u[0] * u[0] + u[1] * u[1]) + u[2] * u[2];
        double t1[3];
        if (z > 0) {
            const double nz = sqrt(z);
            for (int k = 0; k < 3; ++k) t1[k] = u[k] / nz;
        } else {
            for (int k = 0; k < 3; ++k) t1[k] = u[k];
        }
        const double t2[3] = {nrm[1] * t1[2] - nrm[2] * t1[1], nrm[2] * t1[0] - nrm[0] * t1[2],
                              nrm[0] * t1[1] - nrm[1] * t1[0]};
        for (int k = 0; k < 4; ++k) {
            o_nodes[4 * q + k] = nodes[k];
            o_coeff[4 * q + k] = coeff[k];
        }
        o_n[q] = nn;
        for (int k = 0; k < 3; ++k) {
            o_t1[3 * q + k] = t1[k];
            o_t2[3 * q + k] = t2[k];
        }
        o_lambda[q] = -barrier_d1(dist * dist, shat, a.kappa) * 2 * dist;
    }
}

ContactArgs contact_args(const ContactDesc& d, double dt2, int project) {
    ContactArgs a{};
    a.pos = d.pos;
    a.n_pt = d.n_pt;
    a.n_ee = d.n_ee;
    a.pt = d.pt;
    a.ee = d.ee;
    a.dhat = d.dhat;
    a.kappa = d.kappa;
    a.dt2 = dt2;
    a.ground = d.ground;
    for (int k = 0; k < 3; ++k) a.gn[k] = d.ground_normal[k];
    a.gh = d.ground_height;
    a.n_sv = d.ground ? d.n_surf_verts : 0;
    a.sv = d.surf_verts;
    a.n_fr = d.n_friction;
    a.fr_nodes = d.fr_nodes;
    a.fr_n = d.fr_n_nodes;
    a.fr_coeff = d.fr_coeff;
    a.fr_t1 = d.fr_t1;
    a.fr_t2 = d.fr_t2;
    a.fr_lambda = d.fr_lambda;
    a.fr_base = d.fr_base;
    a.mu = d.mu;
    a.fr_eps = d.fr_eps;
    a.project = project;
    return a;
}

}  // namespace

std::int64_t contact_emit(Ctx& c, const ContactDesc& d, double dt2, int project, std::uint64_t* d_keys, double* d_vals,
                          std::int64_t capacity, double* d_node_grad, double* d_value) {
    cudaStream_t st = c.stream;
    const ContactArgs a = contact_args(d, dt2, project);
    const std::int64_t np = a.n_pt + a.n_ee;
    ADIPC_CUDA(cudaMemsetAsync(d_value, 0, sizeof(double), st));
    if (d.n_nodes > 0) ADIPC_CUDA(cudaMemsetAsync(d_node_grad, 0, sizeof(double) * 3 * d.n_nodes, st));
    c.ct_on.reserve(static_cast<std::size_t>(std::max<std::int64_t>(np + a.n_sv + a.n_fr, 1)));
    c.ct_rank.reserve(static_cast<std::size_t>(std::max<std::int64_t>(np + a.n_sv + a.n_fr, 1) + 3));
    std::int32_t* pair_on = c.ct_on.p;
    std::int32_t* gnd_on = c.ct_on.p + np;
    std::int32_t* fr_cnt = c.ct_on.p + np + a.n_sv;
    std::int64_t* pair_rank = c.ct_rank.p;               // np + 1
    std::int64_t* gnd_rank = c.ct_rank.p + np + 1;        // n_sv + 1
    std::int64_t* fr_off = c.ct_rank.p + np + a.n_sv + 2;  // n_fr + 1
    if (np + a.n_sv > 0) {
        k_contact_active<<<grid_for(np + a.n_sv, 256, 16), 256, 0, st>>>(a, pair_on, gnd_on);
        ADIPC_LAUNCH_CHECK();
    }
    if (a.n_fr > 0) {
        k_friction_blocks<<<grid_for(a.n_fr, 256, 16), 256, 0, st>>>(a.fr_n, a.n_fr, fr_cnt);
        ADIPC_LAUNCH_CHECK();
    }
    exclusive_scan(pair_on, np, pair_rank, c.scan_scratch, st);
    exclusive_scan(gnd_on, a.n_sv, gnd_rank, c.scan_scratch, st);
    exclusive_scan(fr_cnt, a.n_fr, fr_off, c.scan_scratch, st);
    std::int64_t h[3] = {0, 0, 0};
    ADIPC_CUDA(cudaMemcpyAsync(&h[0], pair_rank + np, 8, cudaMemcpyDeviceToHost, st));
    ADIPC_CUDA(cudaMemcpyAsync(&h[1], gnd_rank + a.n_sv, 8, cudaMemcpyDeviceToHost, st));
    ADIPC_CUDA(cudaMemcpyAsync(&h[2], fr_off + a.n_fr, 8, cudaMemcpyDeviceToHost, st));
    ADIPC_CUDA(cudaStreamSynchronize(st));
    const std::int64_t T = 10 * h[0] + h[1] + h[2];
    if (T > capacity) throw StatusError(kInvalidArgument, "contact stream capacity too small");
    if (h[0] > 0) {
        c.ct_work.reserve(static_cast<std::size_t>(h[0]) * sizeof(std::int64_t));
        std::int64_t* list = reinterpret_cast<std::int64_t*>(c.ct_work.p);
        k_active_list<<<grid_for(np, 256, 16), 256, 0, st>>>(pair_on, pair_rank, np, list);
        ADIPC_LAUNCH_CHECK();
        k_contact_pairs<<<grid_for(h[0], kContactThreads, 8), kContactThreads, 0, st>>>(a, list, h[0], d_keys, d_vals,
                                                                                        d_node_grad, d_value);
        ADIPC_LAUNCH_CHECK();
    }
    if (h[1] > 0) {
        k_contact_ground<<<grid_for(a.n_sv, 256, 16), 256, 0, st>>>(a, gnd_on, gnd_rank, 10 * h[0], d_keys, d_vals,
                                                                    d_node_grad, d_value);
        ADIPC_LAUNCH_CHECK();
    }
    if (a.n_fr > 0) {
        k_contact_friction<<<grid_for(a.n_fr, 256, 16), 256, 0, st>>>(a, fr_off, 10 * h[0] + h[1], d_keys, d_vals,
                                                                      d_node_grad, d_value);
        ADIPC_LAUNCH_CHECK();
    }
    return T;
}

std::int64_t friction_constraints(Ctx& c, const ContactDesc& d, std::int64_t capacity, std::int32_t* d_nodes4,
                                  std::int32_t* d_n, double* d_coeff4, double* d_t1, double* d_t2, double* d_lambda) {
    cudaStream_t st = c.stream;
    const ContactArgs a = contact_args(d, 0.0, 1);
    const std::int64_t n = a.n_pt + a.n_ee + a.n_sv;
    if (n == 0) return 0;
    c.ct_on.reserve(static_cast<std::size_t>(n));
    c.ct_rank.reserve(static_cast<std::size_t>(n) + 1);
    k_friction_flags<<<grid_for(n, 256, 16), 256, 0, st>>>(a, n, c.ct_on.p);
    ADIPC_LAUNCH_CHECK();
    exclusive_scan(c.ct_on.p, n, c.ct_rank.p, c.scan_scratch, st);
    std::int64_t total = 0;
    ADIPC_CUDA(cudaMemcpyAsync(&total, c.ct_rank.p + n, sizeof(total), cudaMemcpyDeviceToHost, st));
    ADIPC_CUDA(cudaStreamSynchronize(st));
    if (total > capacity) throw StatusError(kInvalidArgument, "friction constraint capacity too small");
    if (total > 0) {
        k_friction_emit<<<grid_for(n, 128, 16), 128, 0, st>>>(a, n, c.ct_on.p, c.ct_rank.p, d_nodes4, d_n, d_coeff4,
                                                             d_t1, d_t2, d_lambda);
        ADIPC_LAUNCH_CHECK();
    }
    return total;
}

double contact_value(Ctx& c, const ContactDesc& d, double dt2) {
    cudaStream_t st = c.stream;
    const ContactArgs a = contact_args(d, dt2, 1);
    c.ct_scal.reserve(2);
    ADIPC_CUDA(cudaMemsetAsync(c.ct_scal.p, 0, 2 * sizeof(double), st));
    const std::int64_t n = a.n_pt + a.n_ee + a.n_sv + a.n_fr;
    if (n > 0) {
        k_contact_value<<<grid_for(n, 256, 16), 256, 0, st>>>(a, c.ct_scal.p, reinterpret_cast<int*>(c.ct_scal.p + 1));
        ADIPC_LAUNCH_CHECK();
    }
    double h[2];
    ADIPC_CUDA(cudaMemcpyAsync(h, c.ct_scal.p, sizeof(h), cudaMemcpyDeviceToHost, st));
    ADIPC_CUDA(cudaStreamSynchronize(st));
    int touch = 0;
    std::memcpy(&touch, &h[1], sizeof(int));
    return touch ? std::numeric_limits<double>::infinity() : h[0];
}

double ccd_step(Ctx& c, const ContactDesc& d, const double* d_disp) {
    cudaStream_t st = c.stream;
    const ContactArgs a = contact_args(d, 0.0, 1);
    c.ct_scal.reserve(2);
    const double one = 1.0;
    ADIPC_CUDA(cudaMemcpyAsync(c.ct_scal.p, &one, sizeof(double), cudaMemcpyHostToDevice, st));
    const std::int64_t n = a.n_pt + a.n_ee + a.n_sv;
    if (n > 0) {
        k_ccd<<<grid_for(n, 128, 16), 128, 0, st>>>(a, d_disp, reinterpret_cast<unsigned long long*>(c.ct_scal.p));
        ADIPC_LAUNCH_CHECK();
    }
    double alpha = 1;
    ADIPC_CUDA(cudaMemcpyAsync(&alpha, c.ct_scal.p, sizeof(double), cudaMemcpyDeviceToHost, st));
    ADIPC_CUDA(cudaStreamSynchronize(st));
    return alpha;
}

}  // namespace adipc_gpu
