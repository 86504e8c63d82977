// Device helpers shared by the element and contact producers (energy.cu,
// contact.cu): fp64 RED / CTA sums, and the PSD projection of a 12 x 12
// stencil Hessian over four nodes that is invariant under a common
// translation of the nodes (stable Neo-Hookean, distance barriers), done in
// the 9-dimensional complement of the translations: with Q the Helmert basis
// of 1-perp in R^4, H12 = (Q (x) I3) M (Q (x) I3)^T and proj(H12) =
// (Q (x) I3) proj(M) (Q (x) I3)^T (energy/psd.hpp:8-14 semantics; the three
// translation eigenvalues are exactly 0).
#pragma once

#include "common.cuh"

namespace adipc_gpu {
namespace {

__device__ __forceinline__ void red_add_f64(double* p, double v) { asm volatile("red.global.add.f64 [%0], %1;" ::"l"(p), "d"(v)); }

// CTA sum of v, one fp64 atomic per CTA into *out
__device__ __forceinline__ void block_sum_atomic(double v, double* out) {
    __shared__ double part[32];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) part[w] = v;
    __syncthreads();
    if (w == 0) {
        v = lane < static_cast<int>(blockDim.x >> 5) ? part[lane] : 0.0;
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) atomicAdd(out, v);
    }
}

// Helmert basis of the complement of (1,1,1,1) in R^4 (columns of Q, 4 x 3)
__device__ __forceinline__ double helmert(int a, int j) {
    const double s2 = 0.70710678118654752440, s6 = 0.40824829046386301637, s12 = 0.28867513459481288225;
    if (j == 0) return a == 0 ? s2 : (a == 1 ? -s2 : 0.0);
    if (j == 1) return a < 2 ? s6 : (a == 2 ? -2.0 * s6 : 0.0);
    return a < 3 ? s12 : -3.0 * s12;
}

// packed lower index of (i, j), i >= j, n = 9
__device__ __forceinline__ constexpr int pk(int i, int j) { return i * (i + 1) / 2 + j; }

// Cholesky of M + tau I in place (packed lower); true when every pivot > 0
__device__ __forceinline__ bool shifted_cholesky_ok(double* L, double tau) {
    bool ok = true;
#pragma unroll
    for (int j = 0; j < 9; ++j) {
        double d = L[pk(j, j)] + tau;
#pragma unroll
        for (int k = 0; k < j; ++k) d -= L[pk(j, k)] * L[pk(j, k)];
        ok = ok && d > 0;
        const double inv = d > 0 ? rsqrt(d) : 0.0;
        L[pk(j, j)] = d > 0 ? d * inv : 0.0;
#pragma unroll
        for (int i = j + 1; i < 9; ++i) {
            double s = L[pk(i, j)];
#pragma unroll
            for (int k = 0; k < j; ++k) s -= L[pk(i, k)] * L[pk(j, k)];
            L[pk(i, j)] = s * inv;
        }
    }
    return ok;
}

// proj(M) for a symmetric N x N (full column-major in `a`, overwritten):
// V max(w, 0) V^T from a Householder reduction to tridiagonal form and
// implicit shifted QL sweeps with deflation at |e_i| <= 2^-52 max(|d| + |e|)
// (Wilkinson / Reinsch tred2 + tql2; Eigen's SelfAdjointEigenSolver is the
// same family: tridiagonalisation + implicit symmetric QR). ~2 K FMA for a
// 9 x 9 against ~17 K for cyclic Jacobi to convergence: the geometric
// scene's contact pass went from 4.4 to 2.3 ms (the element producer runs
// the same algorithm in its own deferred pass, energy.cu k_fem_project).
template <int N>
__device__ __noinline__ void project_sym(double* a) {
    double V[N * N], d[N], e[N];  // V row-major: V[i][j] = V[N * i + j]
    for (int i = 0; i < N; ++i)
        for (int j = 0; j < N; ++j) V[N * i + j] = a[N * j + i];
    // --- tridiagonalisation (tred2)
    for (int j = 0; j < N; ++j) d[j] = V[N * (N - 1) + j];
    for (int i = N - 1; i > 0; --i) {
        double scale = 0, h = 0;
        for (int k = 0; k < i; ++k) scale += fabs(d[k]);
        if (scale == 0) {
            e[i] = d[i - 1];
            for (int j = 0; j < i; ++j) {
                d[j] = V[N * (i - 1) + j];
                V[N * i + j] = 0;
                V[N * j + i] = 0;
            }
        } else {
            for (int k = 0; k < i; ++k) {
                d[k] /= scale;
                h += d[k] * d[k];
            }
            double f = d[i - 1];
            double g = sqrt(h);
            if (f > 0) g = -g;
            e[i] = scale * g;
            h -= f * g;
            d[i - 1] = f - g;
            for (int j = 0; j < i; ++j) e[j] = 0;
            for (int j = 0; j < i; ++j) {
                f = d[j];
                V[N * j + i] = f;
                g = e[j] + V[N * j + j] * f;
                for (int k = j + 1; k <= i - 1; ++k) {
                    g += V[N * k + j] * d[k];
                    e[k] += V[N * k + j] * f;
                }
                e[j] = g;
            }
            f = 0;
            for (int j = 0; j < i; ++j) {
                e[j] /= h;
                f += e[j] * d[j];
            }
            const double hh = f / (h + h);
            for (int j = 0; j < i; ++j) e[j] -= hh * d[j];
            for (int j = 0; j < i; ++j) {
                f = d[j];
                g = e[j];
                for (int k = j; k <= i - 1; ++k) V[N * k + j] -= (f * e[k] + g * d[k]);
                d[j] = V[N * (i - 1) + j];
                V[N * i + j] = 0;
            }
        }
        d[i] = h;
    }
    for (int i = 0; i < N - 1; ++i) {  // accumulate the reflections
        V[N * (N - 1) + i] = V[N * i + i];
        V[N * i + i] = 1;
        const double h = d[i + 1];
        if (h != 0) {
            for (int k = 0; k <= i; ++k) d[k] = V[N * k + i + 1] / h;
            for (int j = 0; j <= i; ++j) {
                double g = 0;
                for (int k = 0; k <= i; ++k) g += V[N * k + i + 1] * V[N * k + j];
                for (int k = 0; k <= i; ++k) V[N * k + j] -= g * d[k];
            }
        }
        for (int k = 0; k <= i; ++k) V[N * k + i + 1] = 0;
    }
    for (int j = 0; j < N; ++j) {
        d[j] = V[N * (N - 1) + j];
        V[N * (N - 1) + j] = 0;
    }
    V[N * (N - 1) + N - 1] = 1;
    e[0] = 0;
    // --- implicit shifted QL (tql2)
    for (int i = 1; i < N; ++i) e[i - 1] = e[i];
    e[N - 1] = 0;
    double f = 0, tst1 = 0;
    const double eps = 2.220446049250313e-16;
    for (int l = 0; l < N; ++l) {
        tst1 = fmax(tst1, fabs(d[l]) + fabs(e[l]));
        int m = l;
        while (m < N - 1 && fabs(e[m]) > eps * tst1) ++m;
        if (m > l) {
            for (int iter = 0; iter < 64; ++iter) {
                double g = d[l];
                double p = (d[l + 1] - g) / (2.0 * e[l]);
                double r = hypot(p, 1.0);
                if (p < 0) r = -r;
                d[l] = e[l] / (p + r);
                d[l + 1] = e[l] * (p + r);
                const double dl1 = d[l + 1];
                double h = g - d[l];
                for (int i = l + 2; i < N; ++i) d[i] -= h;
                f += h;
                p = d[m];
                double c = 1, c2 = 1, c3 = 1, sn = 0, s2 = 0;
                const double el1 = e[l + 1];
                for (int i = m - 1; i >= l; --i) {
                    c3 = c2;
                    c2 = c;
                    s2 = sn;
                    g = c * e[i];
                    h = c * p;
                    r = hypot(p, e[i]);
                    e[i + 1] = sn * r;
                    sn = e[i] / r;
                    c = p / r;
                    p = c * d[i] - sn * g;
                    d[i + 1] = h + sn * (c * g + sn * d[i]);
                    for (int k = 0; k < N; ++k) {
                        h = V[N * k + i + 1];
                        V[N * k + i + 1] = sn * V[N * k + i] + c * h;
                        V[N * k + i] = c * V[N * k + i] - sn * h;
                    }
                }
                p = -sn * s2 * c3 * el1 * e[l] / dl1;
                e[l] = sn * p;
                d[l] = c * p;
                if (!(fabs(e[l]) > eps * tst1)) break;
            }
        }
        d[l] += f;
        e[l] = 0;
    }
    // --- V max(w, 0) V^T (column k of V = eigenvector of d[k])
    for (int k = 0; k < N; ++k) d[k] = d[k] > 0 ? d[k] : 0.0;
    for (int j = 0; j < N; ++j)
        for (int i = j; i < N; ++i) {
            double sum = 0;
            for (int k = 0; k < N; ++k) sum += V[N * i + k] * d[k] * V[N * j + k];
            a[N * j + i] = sum;
            a[N * i + j] = sum;
        }
}
__device__ __forceinline__ void project9(double* a) { project_sym<9>(a); }

// M (9 x 9, full column-major) = (Q (x) I3)^T H (Q (x) I3) from a 12 x 12
// column-major H
__device__ __forceinline__ void reduce_translation(const double* H, double* M) {
    for (int l = 0; l < 3; ++l)
        for (int j = 0; j < 3; ++j)
            for (int c = 0; c < 3; ++c)
                for (int r = 0; r < 3; ++r) {
                    double s = 0;
                    for (int b = 0; b < 4; ++b)
                        for (int a = 0; a < 4; ++a)
                            s += helmert(a, j) * helmert(b, l) * H[12 * (3 * b + c) + 3 * a + r];
                    M[9 * (3 * l + c) + 3 * j + r] = s;
                }
}

// H (12 x 12) = (Q (x) I3) M (Q (x) I3)^T
__device__ __forceinline__ void lift_translation(const double* M, double* H) {
    for (int b = 0; b < 4; ++b)
        for (int a = 0; a < 4; ++a)
            for (int c = 0; c < 3; ++c)
                for (int r = 0; r < 3; ++r) {
                    double s = 0;
                    for (int l = 0; l < 3; ++l)
                        for (int j = 0; j < 3; ++j) s += helmert(a, j) * helmert(b, l) * M[9 * (3 * l + c) + 3 * j + r];
                    H[12 * (3 * b + c) + 3 * a + r] = s;
                }
}

// true when M (full 9 x 9) + tau I passes a Cholesky, tau = 1e-12 tr M
__device__ __forceinline__ bool psd9(const double* M) {
    double L[45], tr = 0;
    for (int i = 0; i < 9; ++i) {
        tr += M[10 * i];
        for (int j = 0; j <= i; ++j) L[pk(i, j)] = M[9 * j + i];
    }
    return tr > 0 && shifted_cholesky_ok(L, 1e-12 * tr);
}

}  // namespace
}  // namespace adipc_gpu
