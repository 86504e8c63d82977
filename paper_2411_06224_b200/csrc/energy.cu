// Device element-Hessian producer: the inertia + solid-mesh
// part of IncrementalPotential::assemble (solver/incremental_potential.hpp:
// 170-180 inertia, 222-239 tets, scatter12 :310-318, pinned gradient
// :253-254) with the polynomial stable Neo-Hookean stencil
// (energy/neo_hookean.hpp:64-104) projected to the PSD cone (energy/psd.hpp:
// 8-14). The triplet stream is written in the reference's emission order
// (every vertex's inertia diagonal, then 10 blocks per tet, a <= b, emit()
// canonicalisation), so the existing filter + sort + reduce turns it into the
// same SortedSymBlockCoo — the 1.5 GB stream never crosses PCIe.
//
// One thread per tet, everything in registers:
//  * vec(F) = (C^T (x) I3) x12 with C = G^T Dm^-1 (4 x 3, G the edge
//    operator of neo_hookean.hpp:44-54), so the 12 x 12 Hessian
//    dFdx^T H9 dFdx is a bilinear form in the rows c_a of C:
//      H_ab = V [ mu (c_a.c_b) I + lam u_a u_b^T + dJcoef [-F (c_a x c_b)]_x ],
//      u_a = cof c_a  (H9 = mu I + lam vec(cof) vec(cof)^T + dJcoef HJ,
//      neo_hookean.hpp:90-99; HJ's six cross-product blocks collapse to one
//      cross-product matrix per block pair).
//  * PSD projection in the 9-dimensional complement of the translations:
//    C = Q R with Q a fixed orthonormal basis of 1-perp in R^4 (Helmert), so
//    H12 = (Q (x) I3) M (Q (x) I3)^T with M_jl = the same bilinear form on the
//    rows r_j of R = Q^T C. The projection of H12 is (Q (x) I3) proj(M)
//    (Q (x) I3)^T (the 3 translation eigenvalues of H12 are exactly 0).
//    Fast path: if M + tau I (tau = 1e-12 tr M) passes a Cholesky, every
//    eigenvalue is > -tau and H12 is emitted as is (the reference clamps
//    eigenvalues in (-tau, 0): a difference below 1e-11 |H|). Otherwise a
//    cyclic Jacobi eigen-decomposition of M (per-thread local arrays; only
//    indefinite elements take it) and proj(M) = V max(w, 0) V^T.
#include "context.hpp"
#include "dual.cuh"
#include "psd.cuh"

namespace adipc_gpu {

namespace {

constexpr int kFemThreads = 128;

struct TetState {
    double F[9];    // column-major
    double cof[9];  // columns f1 x f2, f2 x f0, f0 x f1 (neo_hookean.hpp:29-35)
    double mu, lam, dJ, V;
};

// H_xy = V [ mu (x.y) I + lam (cof x)(cof y)^T + dJ [-F (x cross y)]_x ], 3x3 column-major
__device__ __forceinline__ void stencil_block(const TetState& s, const double* x, const double* y, double* h) {
    double ux[3], uy[3], w[3], xy;
    xy = x[0] * y[0] + x[1] * y[1] + x[2] * y[2];
    for (int k = 0; k < 3; ++k) {
        ux[k] = s.cof[k] * x[0] + s.cof[3 + k] * x[1] + s.cof[6 + k] * x[2];
        uy[k] = s.cof[k] * y[0] + s.cof[3 + k] * y[1] + s.cof[6 + k] * y[2];
    }
    const double z0 = x[1] * y[2] - x[2] * y[1], z1 = x[2] * y[0] - x[0] * y[2], z2 = x[0] * y[1] - x[1] * y[0];
    for (int k = 0; k < 3; ++k) w[k] = -(s.F[k] * z0 + s.F[3 + k] * z1 + s.F[6 + k] * z2);
    // [w]_x column-major: (0,1) = -w2, (0,2) = w1, (1,2) = -w0
    const double W[9] = {0, w[2], -w[1], -w[2], 0, w[0], w[1], -w[0], 0};
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int r = 0; r < 3; ++r)
            h[3 * c + r] = s.V * ((r == c ? s.mu * xy : 0.0) + s.lam * ux[r] * uy[c] + s.dJ * W[3 * c + r]);
}

// inertia (incremental_potential.hpp:170-180): one thread per vertex
__global__ void k_fem_inertia(std::int32_t n, const double* __restrict__ x, const double* __restrict__ xt,
                              const double* __restrict__ mass, std::uint64_t* __restrict__ keys,
                              double* __restrict__ vals, double* __restrict__ grad, double* __restrict__ value) {
    double e = 0;
    for (std::int64_t v = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; v < n;
         v += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        const double m = mass[v];
        const double d0 = x[3 * v] - xt[3 * v], d1 = x[3 * v + 1] - xt[3 * v + 1], d2 = x[3 * v + 2] - xt[3 * v + 2];
        e += 0.5 * m * (d0 * d0 + d1 * d1 + d2 * d2);
        if (grad) {
            grad[3 * v] = m * d0;
            grad[3 * v + 1] = m * d1;
            grad[3 * v + 2] = m * d2;
        }
        if (!keys) continue;  // value only (the line search)
        keys[v] = (static_cast<std::uint64_t>(v) << 32) | static_cast<std::uint64_t>(v);
        double* o = vals + 9 * v;
#pragma unroll
        for (int k = 0; k < 9; ++k) o[k] = (k % 4 == 0) ? m : 0.0;
    }
    block_sum_atomic(e, value);
}

// tets of one mesh: stream entries [base + 10 t, base + 10 t + 10)
__global__ void __launch_bounds__(kFemThreads) k_fem_tets(std::int64_t n_tets, const std::int32_t* __restrict__ tets,
                                                         const double* __restrict__ inv9, const double* __restrict__ vol,
                                                         const double* __restrict__ x, double mu, double lam,
                                                         double dt2, int project, std::uint64_t* __restrict__ keys,
                                                         double* __restrict__ vals, double* __restrict__ grad,
                                                         double* __restrict__ value, double* __restrict__ defer_m,
                                                         std::int64_t* __restrict__ defer_t,
                                                         unsigned long long* __restrict__ defer_n) {
    double e = 0;
    for (std::int64_t t = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; t < n_tets;
         t += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        const int4 id = reinterpret_cast<const int4*>(tets)[t];
        const int ids[4] = {id.x, id.y, id.z, id.w};
        double B[9];
#pragma unroll
        for (int k = 0; k < 9; ++k) B[k] = inv9[9 * t + k];
        TetState s;
        s.V = vol[t];
        s.mu = mu;
        s.lam = lam;
        double xa[4][3];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int k = 0; k < 3; ++k) xa[a][k] = x[3 * static_cast<std::int64_t>(ids[a]) + k];
        // C = G^T B (rows c_a): c_0 = -(B row 0 + row 1 + row 2), c_a = B row a-1
        double C[4][3];
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            C[0][j] = ((0.0 - B[3 * j]) - B[3 * j + 1]) - B[3 * j + 2];
            C[1][j] = B[3 * j];
            C[2][j] = B[3 * j + 1];
            C[3][j] = B[3 * j + 2];
        }
        // F = Ds B (neo_hookean.hpp:69-73)
#pragma unroll
        for (int j = 0; j < 3; ++j)
#pragma unroll
            for (int k = 0; k < 3; ++k)
                s.F[3 * j + k] = (xa[1][k] - xa[0][k]) * B[3 * j] + (xa[2][k] - xa[0][k]) * B[3 * j + 1] +
                                 (xa[3][k] - xa[0][k]) * B[3 * j + 2];
        const double* f0 = s.F;
        const double* f1 = s.F + 3;
        const double* f2 = s.F + 6;
        auto crossp = [](const double* a, const double* b, double* c) {
            c[0] = a[1] * b[2] - a[2] * b[1];
            c[1] = a[2] * b[0] - a[0] * b[2];
            c[2] = a[0] * b[1] - a[1] * b[0];
        };
        crossp(f1, f2, s.cof);
        crossp(f2, f0, s.cof + 3);
        crossp(f0, f1, s.cof + 6);
        const double J = f0[0] * s.cof[0] + f0[1] * s.cof[1] + f0[2] * s.cof[2];
        double IC = 0;
#pragma unroll
        for (int k = 0; k < 9; ++k) IC += s.F[k] * s.F[k];
        e += s.V * (0.5 * mu * (IC - 3) - mu * (J - 1) + 0.5 * lam * (J - 1) * (J - 1));
        s.dJ = lam * (J - 1) - mu;
        // gradient V dFdx^T vec(P), P = mu F + dJ cof: g_a = V P c_a
        double P[9];
#pragma unroll
        for (int k = 0; k < 9; ++k) P[k] = mu * s.F[k] + s.dJ * s.cof[k];
        if (grad) {
#pragma unroll
            for (int a = 0; a < 4; ++a) {
                const std::int64_t o = 3 * static_cast<std::int64_t>(ids[a]);
#pragma unroll
                for (int k = 0; k < 3; ++k)
                    red_add_f64(grad + o + k,
                                dt2 * (s.V * (P[k] * C[a][0] + P[3 + k] * C[a][1] + P[6 + k] * C[a][2])));
            }
        }
        if (!keys) continue;  // value (+ gradient) only
        // PSD test in the reduced space: R = Q^T C, M_jl = stencil(r_j, r_l)
        bool psd = !project;
        double R[3][3];
        if (project) {
#pragma unroll
            for (int j = 0; j < 3; ++j)
#pragma unroll
                for (int i = 0; i < 3; ++i)
                    R[j][i] = helmert(0, j) * C[0][i] + helmert(1, j) * C[1][i] + helmert(2, j) * C[2][i] +
                              helmert(3, j) * C[3][i];
            double L[45];
            double tr = 0;
#pragma unroll
            for (int j = 0; j < 3; ++j)
#pragma unroll
                for (int l = 0; l <= j; ++l) {
                    double h[9];
                    stencil_block(s, R[j], R[l], h);
#pragma unroll
                    for (int c = 0; c < 3; ++c)
#pragma unroll
                        for (int r = 0; r < 3; ++r)
                            if (3 * j + r >= 3 * l + c) L[pk(3 * j + r, 3 * l + c)] = h[3 * c + r];
                }
#pragma unroll
            for (int i = 0; i < 9; ++i) tr += L[pk(i, i)];
            psd = tr > 0 && shifted_cholesky_ok(L, 1e-12 * tr);
        }
        const std::int64_t base = 10 * t;
        if (psd) {
            int q = 0;
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = a; b < 4; ++b, ++q) {
                    double h[9];
                    stencil_block(s, C[a], C[b], h);
                    const bool flip = ids[a] > ids[b];
                    const std::uint32_t r0 = static_cast<std::uint32_t>(flip ? ids[b] : ids[a]);
                    const std::uint32_t c0 = static_cast<std::uint32_t>(flip ? ids[a] : ids[b]);
                    keys[base + q] = (static_cast<std::uint64_t>(r0) << 32) | c0;
                    double* o = vals + 9 * (base + q);
#pragma unroll
                    for (int c = 0; c < 3; ++c)
#pragma unroll
                        for (int r = 0; r < 3; ++r) o[3 * c + r] = dt2 * (flip ? h[3 * r + c] : h[3 * c + r]);
                }
        } else {
            // indefinite: the reduced matrix (packed lower, 45 doubles) goes to
            // the deferred list (fem_emit passes one whenever it emits with
            // projection); k_fem_project projects it and emits the ten blocks
            // with a lean, shared-memory working set
            const unsigned long long slot = atomicAdd(defer_n, 1ull);
#pragma unroll
            for (int j = 0; j < 3; ++j)
#pragma unroll
                for (int l = 0; l <= j; ++l) {
                    double h[9];
                    stencil_block(s, R[j], R[l], h);
#pragma unroll
                    for (int c = 0; c < 3; ++c)
#pragma unroll
                        for (int r = 0; r < 3; ++r)
                            if (3 * j + r >= 3 * l + c) defer_m[45 * slot + pk(3 * j + r, 3 * l + c)] = h[3 * c + r];
                }
            defer_t[slot] = t;
        }
    }
    block_sum_atomic(dt2 * e, value);
}


// The deferred projections of k_fem_tets: one thread per indefinite stencil,
// its work arrays (eigenvectors, tridiagonal) in shared memory laid out
// thread-minor (conflict-free), the same Householder + implicit-QL
// projection as project_sym<9>, then V max(w, 0) V^T lifted through Q (x) I3
// into the stencil's ten blocks at its own stream positions.
constexpr int kProjThreads = 64;
__global__ void __launch_bounds__(kProjThreads) k_fem_project(const unsigned long long* __restrict__ count,
                                                               const double* __restrict__ defer_m,
                                                               const std::int64_t* __restrict__ defer_t,
                                                               const std::int32_t* __restrict__ tets, double dt2,
                                                               std::uint64_t* __restrict__ keys,
                                                               double* __restrict__ vals) {
    constexpr int N = 9, T = kProjThreads;
    extern __shared__ double sm[];
    double* Vs = sm;                  // V[i][j] at (N * i + j) * T + tid
    double* ds = sm + N * N * T;      // d[i] at i * T + tid
    double* es = ds + N * T;          // e[i]
    const int tid = threadIdx.x;
    auto V = [&](int i, int j) -> double& { return Vs[(N * i + j) * T + tid]; };
    auto d = [&](int i) -> double& { return ds[i * T + tid]; };
    auto e = [&](int i) -> double& { return es[i * T + tid]; };
    const unsigned long long n = *count;
    for (unsigned long long w = blockIdx.x * static_cast<unsigned long long>(T) + tid; w < n;
         w += static_cast<unsigned long long>(gridDim.x) * T) {
        const double* Mp = defer_m + 45 * w;
        for (int i = 0; i < N; ++i)
            for (int j = 0; j <= i; ++j) V(i, j) = V(j, i) = Mp[pk(i, j)];
        // tred2
        for (int j = 0; j < N; ++j) d(j) = V(N - 1, j);
        for (int i = N - 1; i > 0; --i) {
            double scale = 0, h = 0;
            for (int k = 0; k < i; ++k) scale += fabs(d(k));
            if (scale == 0) {
                e(i) = d(i - 1);
                for (int j = 0; j < i; ++j) {
                    d(j) = V(i - 1, j);
                    V(i, j) = 0;
                    V(j, i) = 0;
                }
            } else {
                for (int k = 0; k < i; ++k) {
                    d(k) /= scale;
                    h += d(k) * d(k);
                }
                double f = d(i - 1);
                double g = sqrt(h);
                if (f > 0) g = -g;
                e(i) = scale * g;
                h -= f * g;
                d(i - 1) = f - g;
                for (int j = 0; j < i; ++j) e(j) = 0;
                for (int j = 0; j < i; ++j) {
                    f = d(j);
                    V(j, i) = f;
                    g = e(j) + V(j, j) * f;
                    for (int k = j + 1; k <= i - 1; ++k) {
                        g += V(k, j) * d(k);
                        e(k) += V(k, j) * f;
                    }
                    e(j) = g;
                }
                f = 0;
                for (int j = 0; j < i; ++j) {
                    e(j) /= h;
                    f += e(j) * d(j);
                }
                const double hh = f / (h + h);
                for (int j = 0; j < i; ++j) e(j) -= hh * d(j);
                for (int j = 0; j < i; ++j) {
                    f = d(j);
                    g = e(j);
                    for (int k = j; k <= i - 1; ++k) V(k, j) -= (f * e(k) + g * d(k));
                    d(j) = V(i - 1, j);
                    V(i, j) = 0;
                }
            }
            d(i) = h;
        }
        for (int i = 0; i < N - 1; ++i) {
            V(N - 1, i) = V(i, i);
            V(i, i) = 1;
            const double h = d(i + 1);
            if (h != 0) {
                for (int k = 0; k <= i; ++k) d(k) = V(k, i + 1) / h;
                for (int j = 0; j <= i; ++j) {
                    double g = 0;
                    for (int k = 0; k <= i; ++k) g += V(k, i + 1) * V(k, j);
                    for (int k = 0; k <= i; ++k) V(k, j) -= g * d(k);
                }
            }
            for (int k = 0; k <= i; ++k) V(k, i + 1) = 0;
        }
        for (int j = 0; j < N; ++j) {
            d(j) = V(N - 1, j);
            V(N - 1, j) = 0;
        }
        V(N - 1, N - 1) = 1;
        e(0) = 0;
        // tql2
        for (int i = 1; i < N; ++i) e(i - 1) = e(i);
        e(N - 1) = 0;
        double f = 0, tst1 = 0;
        const double eps = 2.220446049250313e-16;
        for (int l = 0; l < N; ++l) {
            tst1 = fmax(tst1, fabs(d(l)) + fabs(e(l)));
            int m = l;
            while (m < N - 1 && fabs(e(m)) > eps * tst1) ++m;
            if (m > l) {
                for (int iter = 0; iter < 64; ++iter) {
                    double g = d(l);
                    double p = (d(l + 1) - g) / (2.0 * e(l));
                    double r = hypot(p, 1.0);
                    if (p < 0) r = -r;
                    d(l) = e(l) / (p + r);
                    d(l + 1) = e(l) * (p + r);
                    const double dl1 = d(l + 1);
                    double h = g - d(l);
                    for (int i = l + 2; i < N; ++i) d(i) -= h;
                    f += h;
                    p = d(m);
                    double c = 1, c2 = 1, c3 = 1, sn = 0, s2 = 0;
                    const double el1 = e(l + 1);
                    for (int i = m - 1; i >= l; --i) {
                        c3 = c2;
                        c2 = c;
                        s2 = sn;
                        g = c * e(i);
                        h = c * p;
                        r = hypot(p, e(i));
                        e(i + 1) = sn * r;
                        sn = e(i) / r;
                        c = p / r;
                        p = c * d(i) - sn * g;
                        d(i + 1) = h + sn * (c * g + sn * d(i));
                        for (int k = 0; k < N; ++k) {
                            h = V(k, i + 1);
                            V(k, i + 1) = sn * V(k, i) + c * h;
                            V(k, i) = c * V(k, i) - sn * h;
                        }
                    }
                    p = -sn * s2 * c3 * el1 * e(l) / dl1;
                    e(l) = sn * p;
                    d(l) = c * p;
                    if (!(fabs(e(l)) > eps * tst1)) break;
                }
            }
            d(l) += f;
            e(l) = 0;
        }
        // W = V diag(sqrt(max(w, 0))) in place: P = W W^T
        for (int k = 0; k < N; ++k) {
            const double sw = d(k) > 0 ? sqrt(d(k)) : 0.0;
            for (int i = 0; i < N; ++i) V(i, k) *= sw;
        }
        const std::int64_t t = defer_t[w];
        const int4 id = reinterpret_cast<const int4*>(tets)[t];
        const int ids[4] = {id.x, id.y, id.z, id.w};
        const std::int64_t base = 10 * t;
        int q = 0;
        for (int a = 0; a < 4; ++a) {
            double Za[3][N];  // rows of (Q (x) I3) W for node a
            for (int r = 0; r < 3; ++r)
                for (int k = 0; k < N; ++k)
                    Za[r][k] = helmert(a, 0) * V(r, k) + helmert(a, 1) * V(3 + r, k) + helmert(a, 2) * V(6 + r, k);
            for (int b = a; b < 4; ++b, ++q) {
                double h[9];
                for (int c = 0; c < 3; ++c) {
                    double zb[N];
                    for (int k = 0; k < N; ++k)
                        zb[k] = helmert(b, 0) * V(c, k) + helmert(b, 1) * V(3 + c, k) + helmert(b, 2) * V(6 + c, k);
                    for (int r = 0; r < 3; ++r) {
                        double sum = 0;
                        for (int k = 0; k < N; ++k) sum += Za[r][k] * zb[k];
                        h[3 * c + r] = sum;
                    }
                }
                const bool flip = ids[a] > ids[b];
                const std::uint32_t r0 = static_cast<std::uint32_t>(flip ? ids[b] : ids[a]);
                const std::uint32_t c0 = static_cast<std::uint32_t>(flip ? ids[a] : ids[b]);
                keys[base + q] = (static_cast<std::uint64_t>(r0) << 32) | c0;
                double* o = vals + 9 * (base + q);
                for (int c = 0; c < 3; ++c)
                    for (int r = 0; r < 3; ++r) o[3 * c + r] = dt2 * (flip ? h[3 * r + c] : h[3 * c + r]);
            }
        }
    }
}

// affine-body inertia (incremental_potential.hpp:181-188): g = M dq written
// to the body's 12 gradient entries, 0.5 dq.g to the value, the reduced mass
// as split_sym_12x12 tiles (block_split.hpp:19-23)
__global__ void k_body_inertia(std::int32_t nb, std::int32_t base0, const double* __restrict__ q,
                               const double* __restrict__ qt, const double* __restrict__ M12,
                               std::uint64_t* __restrict__ keys, double* __restrict__ vals, double* __restrict__ grad,
                               double* __restrict__ value) {
    double e = 0;
    for (std::int64_t b = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; b < nb;
         b += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        const double* M = M12 + 144 * b;
        double dq[12], g[12];
        for (int k = 0; k < 12; ++k) dq[k] = q[12 * b + k] - qt[12 * b + k];
        double dg = 0;
        for (int i = 0; i < 12; ++i) {
            double s = 0;
            for (int k = 0; k < 12; ++k) s += M[12 * k + i] * dq[k];
            g[i] = s;
        }
        for (int k = 0; k < 12; ++k) dg += dq[k] * g[k];
        e += 0.5 * dg;
        const std::int64_t base = base0 + 4 * b;
        if (grad)
            for (int k = 0; k < 12; ++k) grad[3 * base + k] = g[k];
        if (!keys) continue;
        int t = 0;
        for (int ti = 0; ti < 4; ++ti)
            for (int tj = ti; tj < 4; ++tj, ++t) {
                const std::int64_t o = 10 * b + t;
                keys[o] = (static_cast<std::uint64_t>(base + ti) << 32) | static_cast<std::uint64_t>(base + tj);
                for (int c = 0; c < 3; ++c)
                    for (int r = 0; r < 3; ++r) vals[9 * o + 3 * c + r] = M[12 * (3 * tj + c) + 3 * ti + r];
            }
    }
    block_sum_atomic(e, value);
}

// affine-body orthogonality (energy/abd_energy.hpp:19-42; :242-249): the
// stencil lives on the 9 affine dofs only, so its PSD projection is the 9 x 9
// block's; dt^2-scaled split_sym_12x12 tiles, gradient added
__global__ void k_body_orth(std::int32_t nb, std::int32_t base0, const double* __restrict__ q,
                            const double* __restrict__ kappa, const double* __restrict__ vol, double dt2, int project,
                            std::uint64_t* __restrict__ keys, double* __restrict__ vals, double* __restrict__ grad,
                            double* __restrict__ value) {
    double e = 0;
    for (std::int64_t b = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; b < nb;
         b += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        double A[3][3], C[3][3], AAt[3][3];
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) A[r][c] = q[12 * b + 3 + 3 * r + c];
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) {
                C[r][c] = (A[0][r] * A[0][c] + A[1][r] * A[1][c] + A[2][r] * A[2][c]) - (r == c ? 1.0 : 0.0);
                AAt[r][c] = A[r][0] * A[c][0] + A[r][1] * A[c][1] + A[r][2] * A[c][2];
            }
        const double kv = kappa[b] * vol[b];
        double cn = 0;
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) cn += C[r][c] * C[r][c];
        e += kv * cn;
        const std::int64_t base = base0 + 4 * b;
        for (int r = 0; r < 3 && grad; ++r)
            for (int c = 0; c < 3; ++c)
                red_add_f64(grad + 3 * base + 3 + 3 * r + c,
                            dt2 * ((4 * kv * A[r][0]) * C[0][c] + (4 * kv * A[r][1]) * C[1][c] + (4 * kv * A[r][2]) * C[2][c]));
        if (!keys) continue;
        double M[81];  // the affine 9 x 9 block, column-major
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c)
                for (int s2 = 0; s2 < 3; ++s2)
                    for (int t = 0; t < 3; ++t)
                        M[9 * (3 * s2 + t) + 3 * r + c] =
                            4 * kv * (A[r][t] * A[s2][c] + (r == s2 ? C[t][c] : 0.0) + (t == c ? AAt[r][s2] : 0.0));
        if (project && !psd9(M)) project9(M);
        auto h12 = [&](int i, int j) { return (i < 3 || j < 3) ? 0.0 : M[9 * (j - 3) + (i - 3)]; };
        int t = 0;
        for (int ti = 0; ti < 4; ++ti)
            for (int tj = ti; tj < 4; ++tj, ++t) {
                const std::int64_t o = 10 * b + t;
                keys[o] = (static_cast<std::uint64_t>(base + ti) << 32) | static_cast<std::uint64_t>(base + tj);
                for (int c = 0; c < 3; ++c)
                    for (int r = 0; r < 3; ++r) vals[9 * o + 3 * c + r] = dt2 * h12(3 * ti + r, 3 * tj + c);
            }
    }
    block_sum_atomic(dt2 * e, value);
}


// ---- shells (cfg2 cloth): membrane triangles and hinges ----------------------
struct ShellParams {
    double thickness, stretch, strain_limit, shear_fraction, bending;
};

// IncrementalPotential::membrane_stencil (incremental_potential.hpp:273-298;
// energy/membrane.hpp:36-135): FBW stretch (per-axis eigenvalue clamp), cubic
// strain limit, I6 shear (its 6 x 6 Hessian projected), then the chain rule
// through membrane_dFdx as a bilinear form in C = G^T Dm^-1 (3 x 2); scatter9
// (:300-308): 6 blocks, a <= b
__global__ void __launch_bounds__(128) k_shell_tris(std::int64_t n_tris, const std::int32_t* __restrict__ tris,
                                                    const double* __restrict__ rest5, const double* __restrict__ x,
                                                    ShellParams m, double dt2, int project,
                                                    std::uint64_t* __restrict__ keys, double* __restrict__ vals,
                                                    double* __restrict__ grad, double* __restrict__ value) {
    double e = 0;
    for (std::int64_t t = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; t < n_tris;
         t += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        const int ids[3] = {tris[3 * t], tris[3 * t + 1], tris[3 * t + 2]};
        const double* rs = rest5 + 5 * t;
        double xa[3][3];
        for (int a = 0; a < 3; ++a)
            for (int k = 0; k < 3; ++k) xa[a][k] = x[3 * static_cast<std::int64_t>(ids[a]) + k];
        double F[6];
        for (int j = 0; j < 2; ++j)
            for (int k = 0; k < 3; ++k) F[3 * j + k] = (xa[1][k] - xa[0][k]) * rs[2 * j] + (xa[2][k] - xa[0][k]) * rs[2 * j + 1];
        const double a_t = rs[4] * m.thickness;
        double val = 0, dF[6] = {0, 0, 0, 0, 0, 0}, H6[36];
        for (int k = 0; k < 36; ++k) H6[k] = 0;
        for (int dir = 0; dir < 2; ++dir) {  // fbw_membrane (membrane.hpp:54-75)
            const double scale = m.stretch * a_t;
            const double* f = F + 3 * dir;
            const double I5v = f[0] * f[0] + f[1] * f[1] + f[2] * f[2];
            const double sq = sqrt(I5v);
            val += scale * (sq - 1) * (sq - 1);
            for (int k = 0; k < 3; ++k) dF[3 * dir + k] += 2 * scale * (1 - 1 / sq) * f[k];
            const double e1 = 2 * scale;
            double e23 = 2 * scale * (1 - 1 / sq);
            if (project && e23 < 0) e23 = 0;
            for (int c = 0; c < 3; ++c)
                for (int r = 0; r < 3; ++r)
                    H6[6 * (3 * dir + c) + 3 * dir + r] += (r == c ? e23 : 0.0) + (e1 - e23) * (f[r] / sq) * (f[c] / sq);
        }
        for (int dir = 0; dir < 2; ++dir) {  // cubic_strain_limit (:87-102)
            const double scale = m.strain_limit * a_t;
            const double* f = F + 3 * dir;
            const double I5v = f[0] * f[0] + f[1] * f[1] + f[2] * f[2];
            if (I5v <= 1.0) continue;
            const double sq = sqrt(I5v);
            val += scale * (sq - 1) * (sq - 1) * (sq - 1);
            for (int k = 0; k < 3; ++k) dF[3 * dir + k] += scale * (3 * (sq - 1) * (sq - 1) / sq) * f[k];
            const double e1 = 6 * (sq - 1), e23 = 3 * (1 / sq + sq - 2);
            for (int c = 0; c < 3; ++c)
                for (int r = 0; r < 3; ++r)
                    H6[6 * (3 * dir + c) + 3 * dir + r] += scale * ((r == c ? e23 : 0.0) + ((e1 - e23) / I5v) * f[r] * f[c]);
        }
        {  // shear_energy (:105-121)
            const double scale = m.shear_fraction * m.stretch * a_t;
            const double I6 = F[0] * F[3] + F[1] * F[4] + F[2] * F[5];
            val += scale * I6 * I6;
            for (int k = 0; k < 3; ++k) {
                dF[k] += 2 * scale * I6 * F[3 + k];
                dF[3 + k] += 2 * scale * I6 * F[k];
            }
            const double g[6] = {F[3], F[4], F[5], F[0], F[1], F[2]};
            double S[36];
            for (int c = 0; c < 6; ++c)
                for (int r = 0; r < 6; ++r)
                    S[6 * c + r] = 2 * scale * (g[r] * g[c] + I6 * ((r < 3) != (c < 3) && r % 3 == c % 3 ? 1.0 : 0.0));
            if (project) project_sym<6>(S);
            for (int k = 0; k < 36; ++k) H6[k] += S[k];
        }
        e += val;
        double C[3][2];
        for (int j = 0; j < 2; ++j) {
            C[0][j] = -rs[2 * j] - rs[2 * j + 1];
            C[1][j] = rs[2 * j];
            C[2][j] = rs[2 * j + 1];
        }
        if (grad)
            for (int a = 0; a < 3; ++a)
                for (int k = 0; k < 3; ++k)
                    red_add_f64(grad + 3 * static_cast<std::int64_t>(ids[a]) + k, dt2 * (C[a][0] * dF[k] + C[a][1] * dF[3 + k]));
        if (!keys) continue;
        int q = 0;
        for (int a = 0; a < 3; ++a)
            for (int b = a; b < 3; ++b, ++q) {
                double h[9];
                for (int c = 0; c < 3; ++c)
                    for (int r = 0; r < 3; ++r) {
                        double v = 0;
                        for (int j = 0; j < 2; ++j)
                            for (int l = 0; l < 2; ++l) v += C[a][j] * C[b][l] * H6[6 * (3 * l + c) + 3 * j + r];
                        h[3 * c + r] = v;
                    }
                const bool flip = ids[a] > ids[b];
                const std::uint32_t r0 = static_cast<std::uint32_t>(flip ? ids[b] : ids[a]);
                const std::uint32_t c0 = static_cast<std::uint32_t>(flip ? ids[a] : ids[b]);
                keys[6 * t + q] = (static_cast<std::uint64_t>(r0) << 32) | c0;
                double* o = vals + 9 * (6 * t + q);
                for (int c = 0; c < 3; ++c)
                    for (int r = 0; r < 3; ++r) o[3 * c + r] = dt2 * (flip ? h[3 * r + c] : h[3 * c + r]);
            }
    }
    block_sum_atomic(dt2 * e, value);
}

// hinge bending (energy/bending.hpp:11-75): k w (theta - rest)^2 with the
// dihedral angle by second-order duals; PSD projection in the complement of
// the translations (the angle is translation invariant); scatter12, 10 blocks
struct HingeWork {
    D12 e[3], n1[3], n2[3], t[3];
    D12 a, b, c, d, t0, t1;
};
__global__ void __launch_bounds__(64) k_shell_hinges(std::int64_t n_h, const std::int32_t* __restrict__ hinges,
                                                     const double* __restrict__ rest2, const double* __restrict__ x,
                                                     double kb, double dt2, int project, std::uint64_t* __restrict__ keys,
                                                     double* __restrict__ vals, double* __restrict__ grad,
                                                     double* __restrict__ value, HingeWork* __restrict__ work) {
    const std::int64_t tid = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x;
    HingeWork& W = work[tid];
    double en = 0;
    for (std::int64_t h = tid; h < n_h; h += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        const int ids[4] = {hinges[4 * h], hinges[4 * h + 1], hinges[4 * h + 2], hinges[4 * h + 3]};
        double xs[12];
        for (int a = 0; a < 4; ++a)
            for (int k = 0; k < 3; ++k) xs[3 * a + k] = x[3 * static_cast<std::int64_t>(ids[a]) + k];
        // dihedral_angle_g: e = x1 - x0, n1 = e x (x2 - x0), n2 = (x3 - x0) x e,
        // s = ((n1 x n2) . e) / sqrt(|e|^2), c = n1 . n2, atan2(s, c)
        d_vdiff(W.e, xs, 1, 0);
        d_vdiff(W.t, xs, 2, 0);
        d_cross(W.n1, W.e, W.t, W.t0, W.t1);
        d_vdiff(W.t, xs, 3, 0);
        d_cross(W.n2, W.t, W.e, W.t0, W.t1);
        d_cross(W.t, W.n1, W.n2, W.t0, W.t1);
        d_dot(W.a, W.t, W.e, W.t0, W.t1);   // (n1 x n2) . e
        d_norm2(W.b, W.e, W.t0, W.t1);      // |e|^2
        d_sqrt(W.b, W.b);
        d_div(W.c, W.a, W.b, W.t0);         // s
        d_dot(W.d, W.n1, W.n2, W.t0, W.t1); // c
        d_atan2(W.a, W.c, W.d);             // theta
        W.a.v += -rest2[2 * h];             // theta - rest
        d_mul(W.b, W.a, W.a);
        d_scale(W.c, W.b, kb * rest2[2 * h + 1]);
        const D12& E = W.c;
        en += E.v;
        if (grad)
            for (int a = 0; a < 4; ++a)
                for (int k = 0; k < 3; ++k) red_add_f64(grad + 3 * static_cast<std::int64_t>(ids[a]) + k, dt2 * E.g[3 * a + k]);
        if (!keys) continue;
        double H[144];
        for (int j = 0; j < 12; ++j)
            for (int i = 0; i < 12; ++i) H[12 * j + i] = E.h[hp(i, j)];
        if (project) {
            double M[81];
            reduce_translation(H, M);
            if (!psd9(M)) {
                project9(M);
                lift_translation(M, H);
            }
        }
        int q = 0;
        for (int a = 0; a < 4; ++a)
            for (int b = a; b < 4; ++b, ++q) {
                const bool flip = ids[a] > ids[b];
                const std::uint32_t r0 = static_cast<std::uint32_t>(flip ? ids[b] : ids[a]);
                const std::uint32_t c0 = static_cast<std::uint32_t>(flip ? ids[a] : ids[b]);
                keys[10 * h + q] = (static_cast<std::uint64_t>(r0) << 32) | c0;
                double* o = vals + 9 * (10 * h + q);
                for (int c = 0; c < 3; ++c)
                    for (int r = 0; r < 3; ++r)
                        o[3 * c + r] = dt2 * (flip ? H[12 * (3 * b + r) + 3 * a + c] : H[12 * (3 * b + c) + 3 * a + r]);
            }
    }
    block_sum_atomic(dt2 * en, value);
}

// pinned slots: zero gradient (incremental_potential.hpp:253-254)
__global__ void k_fem_pin_grad(std::int32_t n, const std::uint8_t* __restrict__ pinned, double* __restrict__ grad) {
    for (std::int64_t v = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; v < n;
         v += static_cast<std::int64_t>(gridDim.x) * blockDim.x)
        if (pinned[v]) grad[3 * v] = grad[3 * v + 1] = grad[3 * v + 2] = 0.0;
}

}  // namespace

// The stream (n_verts + 10 n_tets + 20 n_bodies entries), the gradient
// (3 (n_verts + 4 n_bodies)) and the value (one device double) of inertia,
// every solid mesh and the affine bodies. d_keys / d_vals null: the value
// (and, with d_grad, the gradient) only — IncrementalPotential::value for
// the line search (incremental_potential.hpp:61-131, raw stencils: the
// projection does not change values).
void fem_emit(Ctx& c, const FemDesc& d, std::uint64_t* d_keys, double* d_vals, double* d_grad, double* d_value) {
    cudaStream_t st = c.stream;
    ADIPC_CUDA(cudaMemsetAsync(d_value, 0, sizeof(double), st));
    if (d.n_verts > 0) {
        k_fem_inertia<<<grid_for(d.n_verts, 256, 8), 256, 0, st>>>(d.n_verts, d.x, d.x_tilde, d.mass, d_keys, d_vals,
                                                                 d_grad, d_value);
        ADIPC_LAUNCH_CHECK();
    }
    // stream layout (incremental_potential.hpp:170-249): vertex inertia, body
    // inertia tiles, the meshes in scene order (solid: 10 blocks per tet;
    // shell: 6 per membrane triangle, then 10 per hinge), body orthogonality
    const std::int64_t nb = d.n_bodies;
    std::int64_t off = d.n_verts + 10 * nb;
    if (nb > 0) {
        k_body_inertia<<<grid_for(nb, 128, 8), 128, 0, st>>>(d.n_bodies, d.n_verts, d.q, d.q_tilde, d.reduced_mass,
                                                             d_keys ? d_keys + d.n_verts : nullptr,
                                                             d_vals ? d_vals + 9 * d.n_verts : nullptr, d_grad, d_value);
        ADIPC_LAUNCH_CHECK();
    }
    auto solid = [&](int m) {
        const std::int64_t t0 = d.tet_begin[m], nt = d.tet_begin[m + 1] - t0;
        if (nt > 0) {
            // indefinite stencils are projected by k_fem_project from a list
            // (capacity: every stencil of the mesh)
            const bool defer = d.project && d_keys;
            if (defer) {
                c.fem_defer_m.reserve(static_cast<std::size_t>(nt) * 45);
                c.fem_defer_t.reserve(static_cast<std::size_t>(nt));
                c.fem_defer_n.reserve(1);
                ADIPC_CUDA(cudaMemsetAsync(c.fem_defer_n.p, 0, sizeof(unsigned long long), st));
            }
            k_fem_tets<<<grid_for(nt, kFemThreads, 16), kFemThreads, 0, st>>>(
                nt, d.tets + 4 * t0, d.rest_inv9 + 9 * t0, d.rest_volume + t0, d.x, d.mu[m], d.lambda[m], d.dt2,
                d.project, d_keys ? d_keys + off : nullptr, d_vals ? d_vals + 9 * off : nullptr, d_grad, d_value,
                defer ? c.fem_defer_m.p : nullptr, defer ? c.fem_defer_t.p : nullptr,
                defer ? c.fem_defer_n.p : nullptr);
            ADIPC_LAUNCH_CHECK();
            if (defer) {
                const std::size_t smem = sizeof(double) * (81 + 18) * kProjThreads;
                ADIPC_CUDA(cudaFuncSetAttribute(k_fem_project, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                static_cast<int>(smem)));
                int sms = kSMs, occ = 0;
                cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c.device);
                ADIPC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_fem_project, kProjThreads, smem));
                k_fem_project<<<sms * std::max(occ, 1), kProjThreads, smem, st>>>(
                    c.fem_defer_n.p, c.fem_defer_m.p, c.fem_defer_t.p, d.tets + 4 * t0, d.dt2, d_keys + off,
                    d_vals + 9 * off);
                ADIPC_LAUNCH_CHECK();
            }
        }
        off += 10 * nt;
    };
    auto shell = [&](int m) {
        const ShellParams sp{d.shell_material[5 * m], d.shell_material[5 * m + 1], d.shell_material[5 * m + 2],
                             d.shell_material[5 * m + 3], d.shell_material[5 * m + 4]};
        const std::int64_t t0 = d.tri_begin[m], ntr = d.tri_begin[m + 1] - t0;
        if (ntr > 0) {
            k_shell_tris<<<grid_for(ntr, 128, 16), 128, 0, st>>>(ntr, d.tris + 3 * t0, d.tri_rest + 5 * t0, d.x, sp, d.dt2,
                                                                  d.project, d_keys ? d_keys + off : nullptr,
                                                                  d_vals ? d_vals + 9 * off : nullptr, d_grad, d_value);
            ADIPC_LAUNCH_CHECK();
        }
        off += 6 * ntr;
        const std::int64_t h0 = d.hinge_begin[m], nh = d.hinge_begin[m + 1] - h0;
        if (nh > 0) {
            const int grid = static_cast<int>(std::min<std::int64_t>(ceil_div(nh, 64), kSMs * 4));
            c.hinge_work.reserve(static_cast<std::size_t>(grid) * 64 * sizeof(HingeWork));
            k_shell_hinges<<<grid, 64, 0, st>>>(nh, d.hinges + 4 * h0, d.hinge_rest + 2 * h0, d.x, sp.bending, d.dt2,
                                                d.project, d_keys ? d_keys + off : nullptr,
                                                d_vals ? d_vals + 9 * off : nullptr, d_grad, d_value,
                                                reinterpret_cast<HingeWork*>(c.hinge_work.p));
            ADIPC_LAUNCH_CHECK();
        }
        off += 10 * nh;
    };
    if (d.n_kinds == 0) {
        for (int m = 0; m < d.n_meshes; ++m) solid(m);
    } else {
        int si = 0, hi = 0;
        for (int i = 0; i < d.n_kinds; ++i) {
            if (d.mesh_kind[i] == 0)
                solid(si++);
            else
                shell(hi++);
        }
    }
    const std::int64_t orth0 = off;
    if (nb > 0) {
        k_body_orth<<<grid_for(nb, 128, 8), 128, 0, st>>>(d.n_bodies, d.n_verts, d.q, d.body_kappa, d.body_volume,
                                                          d.dt2, d.project, d_keys ? d_keys + orth0 : nullptr,
                                                          d_vals ? d_vals + 9 * orth0 : nullptr, d_grad, d_value);
        ADIPC_LAUNCH_CHECK();
    }
    const std::int32_t n_slots = d.n_verts + 4 * d.n_bodies;
    if (d_grad && d.pinned && n_slots > 0) {
        k_fem_pin_grad<<<grid_for(n_slots, 256, 8), 256, 0, st>>>(n_slots, d.pinned, d_grad);
        ADIPC_LAUNCH_CHECK();
    }
}

}  // namespace adipc_gpu
