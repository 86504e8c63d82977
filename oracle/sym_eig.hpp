// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// Symmetric eigen-decomposition behind the PSD projection of
// energy/psd.hpp:8-14, standing in for Eigen 3.4's SelfAdjointEigenSolver,
// which is not in the image. Same algorithm family as Eigen's: Householder
// reduction to tridiagonal form, then implicit shifted QL sweeps with
// deflation at |e_i| <= 2^-52 max(|d| + |e|) (Wilkinson / Reinsch, Handbook
// for Automatic Computation II, tred2 + tql2; Golub & Van Loan §8.3) — the
// cost of one 12 x 12 is a few microseconds, as with Eigen, so CPU timings of
// the producers are not inflated. Eigenvalues ascending with their
// eigenvectors as columns, as Eigen returns them; they and the projection
// agree with Eigen's to rounding (the reference's tests pin the projection
// to 1e-10 / 1e-12). Sizes above 16 (unused by the path) fall back to cyclic
// Jacobi. Shared by oracle.hpp (the restatement) and eigen_shim/Eigen/Dense
// (the reference's own psd.hpp compiled into oracle/_ref).
#pragma once

#include <algorithm>
#include <cmath>
#include <numeric>
#include <vector>

namespace oracle_eig {

// cyclic Jacobi (Golub & Van Loan §8.5) for n > 16: threshold rule, an
// off-diagonal entry below 1e-17 of the Frobenius norm is zeroed, not rotated
inline void sym_eig_jacobi(int n, const double* A, double* w, double* V) {
    std::vector<double> a(A, A + static_cast<std::size_t>(n) * n), v(static_cast<std::size_t>(n) * n, 0.0);
    auto at = [n](std::vector<double>& m, int i, int j) -> double& { return m[static_cast<std::size_t>(j) * n + i]; };
    for (int i = 0; i < n; ++i) at(v, i, i) = 1.0;
    double tot = 0;  // ||A||_F^2, invariant under the rotations
    for (std::size_t k = 0; k < a.size(); ++k) tot += a[k] * a[k];
    const double negligible = 1e-34 * tot;
    for (int sweep = 0; sweep < 64; ++sweep) {
        bool rotated = false;
        for (int p = 0; p < n - 1; ++p)
            for (int q = p + 1; q < n; ++q) {
                const double apq = at(a, p, q);
                if (apq == 0.0) continue;
                if (apq * apq <= negligible) {
                    at(a, p, q) = at(a, q, p) = 0.0;
                    continue;
                }
                rotated = true;
                const double theta = (at(a, q, q) - at(a, p, p)) / (2.0 * apq);
                const double t = (theta >= 0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
                const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
                for (int k = 0; k < n; ++k) {  // A <- A J (columns p, q)
                    const double kp = at(a, k, p), kq = at(a, k, q);
                    at(a, k, p) = c * kp - s * kq;
                    at(a, k, q) = s * kp + c * kq;
                }
                for (int k = 0; k < n; ++k) {  // A <- J^T A (rows p, q)
                    const double pk = at(a, p, k), qk = at(a, q, k);
                    at(a, p, k) = c * pk - s * qk;
                    at(a, q, k) = s * pk + c * qk;
                }
                for (int k = 0; k < n; ++k) {  // V <- V J
                    const double kp = at(v, k, p), kq = at(v, k, q);
                    at(v, k, p) = c * kp - s * kq;
                    at(v, k, q) = s * kp + c * kq;
                }
            }
        if (!rotated) break;
    }
    std::vector<int> ord(n);
    std::iota(ord.begin(), ord.end(), 0);
    std::stable_sort(ord.begin(), ord.end(), [&](int x, int y) { return at(a, x, x) < at(a, y, y); });
    for (int k = 0; k < n; ++k) {
        w[k] = at(a, ord[k], ord[k]);
        for (int i = 0; i < n; ++i) V[static_cast<std::size_t>(k) * n + i] = at(v, i, ord[k]);
    }
}

// Householder tridiagonalisation of the symmetric V (n x n, row-major,
// overwritten by the accumulated orthogonal transform): diagonal d, the
// sub-diagonal in e[1..n-1].
inline void tridiagonalize(int n, double* V, double* d, double* e) {
    auto v = [n, V](int i, int j) -> double& { return V[i * n + j]; };
    for (int j = 0; j < n; ++j) d[j] = v(n - 1, j);
    for (int i = n - 1; i > 0; --i) {
        double scale = 0, h = 0;
        for (int k = 0; k < i; ++k) scale += std::fabs(d[k]);
        if (scale == 0) {
            e[i] = d[i - 1];
            for (int j = 0; j < i; ++j) {
                d[j] = v(i - 1, j);
                v(i, j) = 0;
                v(j, i) = 0;
            }
        } else {
            for (int k = 0; k < i; ++k) {
                d[k] /= scale;
                h += d[k] * d[k];
            }
            double f = d[i - 1];
            double g = std::sqrt(h);
            if (f > 0) g = -g;
            e[i] = scale * g;
            h -= f * g;
            d[i - 1] = f - g;
            for (int j = 0; j < i; ++j) e[j] = 0;
            for (int j = 0; j < i; ++j) {
                f = d[j];
                v(j, i) = f;
                g = e[j] + v(j, j) * f;
                for (int k = j + 1; k <= i - 1; ++k) {
                    g += v(k, j) * d[k];
                    e[k] += v(k, j) * f;
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
                for (int k = j; k <= i - 1; ++k) v(k, j) -= (f * e[k] + g * d[k]);
                d[j] = v(i - 1, j);
                v(i, j) = 0;
            }
        }
        d[i] = h;
    }
    for (int i = 0; i < n - 1; ++i) {  // accumulate the reflections
        v(n - 1, i) = v(i, i);
        v(i, i) = 1;
        const double h = d[i + 1];
        if (h != 0) {
            for (int k = 0; k <= i; ++k) d[k] = v(k, i + 1) / h;
            for (int j = 0; j <= i; ++j) {
                double g = 0;
                for (int k = 0; k <= i; ++k) g += v(k, i + 1) * v(k, j);
                for (int k = 0; k <= i; ++k) v(k, j) -= g * d[k];
            }
        }
        for (int k = 0; k <= i; ++k) v(k, i + 1) = 0;
    }
    for (int j = 0; j < n; ++j) {
        d[j] = v(n - 1, j);
        v(n - 1, j) = 0;
    }
    v(n - 1, n - 1) = 1;
    e[0] = 0;
}

// implicit shifted QL on the tridiagonal (d, e), rotations applied to V
inline void tridiagonal_ql(int n, double* V, double* d, double* e) {
    auto v = [n, V](int i, int j) -> double& { return V[i * n + j]; };
    for (int i = 1; i < n; ++i) e[i - 1] = e[i];
    e[n - 1] = 0;
    double f = 0, tst1 = 0;
    const double eps = std::ldexp(1.0, -52);
    for (int l = 0; l < n; ++l) {
        tst1 = std::max(tst1, std::fabs(d[l]) + std::fabs(e[l]));
        int m = l;
        while (m < n - 1 && std::fabs(e[m]) > eps * tst1) ++m;
        if (m > l) {
            for (int iter = 0; iter < 64; ++iter) {
                double g = d[l];
                double p = (d[l + 1] - g) / (2.0 * e[l]);
                double r = std::hypot(p, 1.0);
                if (p < 0) r = -r;
                d[l] = e[l] / (p + r);
                d[l + 1] = e[l] * (p + r);
                const double dl1 = d[l + 1];
                double h = g - d[l];
                for (int i = l + 2; i < n; ++i) d[i] -= h;
                f += h;
                p = d[m];
                double c = 1, c2 = 1, c3 = 1, s = 0, s2 = 0;
                const double el1 = e[l + 1];
                for (int i = m - 1; i >= l; --i) {
                    c3 = c2;
                    c2 = c;
                    s2 = s;
                    g = c * e[i];
                    h = c * p;
                    r = std::hypot(p, e[i]);
                    e[i + 1] = s * r;
                    s = e[i] / r;
                    c = p / r;
                    p = c * d[i] - s * g;
                    d[i + 1] = h + s * (c * g + s * d[i]);
                    for (int k = 0; k < n; ++k) {
                        h = v(k, i + 1);
                        v(k, i + 1) = s * v(k, i) + c * h;
                        v(k, i) = c * v(k, i) - s * h;
                    }
                }
                p = -s * s2 * c3 * el1 * e[l] / dl1;
                e[l] = s * p;
                d[l] = c * p;
                if (!(std::fabs(e[l]) > eps * tst1)) break;
            }
        }
        d[l] += f;
        e[l] = 0;
    }
}

// A: n x n column-major symmetric (read only). w: n eigenvalues ascending.
// V: n x n column-major, column k = eigenvector of w[k].
inline void sym_eig(int n, const double* A, double* w, double* V) {
    if (n > 16 || n < 1) {
        sym_eig_jacobi(n, A, w, V);
        return;
    }
    double Q[256], d[16], e[16];
    for (int i = 0; i < n; ++i)  // symmetric: row-major copy of the lower triangle mirrored
        for (int j = 0; j < n; ++j) Q[i * n + j] = A[(i >= j ? j * n + i : i * n + j)];
    tridiagonalize(n, Q, d, e);
    tridiagonal_ql(n, Q, d, e);
    int ord[16];  // stable insertion sort (no heap: the producers call this from every thread)
    for (int k = 0; k < n; ++k) {
        int j = k;
        while (j > 0 && d[ord[j - 1]] > d[k]) {
            ord[j] = ord[j - 1];
            --j;
        }
        ord[j] = k;
    }
    for (int k = 0; k < n; ++k) {
        w[k] = d[ord[k]];
        for (int i = 0; i < n; ++i) V[static_cast<std::size_t>(k) * n + i] = Q[i * n + ord[k]];
    }
}

// energy/psd.hpp:8-14: V max(w, 0) V^T, in Eigen's evaluation order
// ((V * diag) * V^T, inner index ascending).
inline void project_psd(int n, const double* M, double* out) {
    double ws[16], Vs[256], VDs[256];
    std::vector<double> wh, Vh, VDh;
    double *w = ws, *V = Vs, *VD = VDs;
    if (n > 16) {
        wh.resize(n);
        Vh.resize(static_cast<std::size_t>(n) * n);
        VDh.resize(static_cast<std::size_t>(n) * n);
        w = wh.data();
        V = Vh.data();
        VD = VDh.data();
    }
    sym_eig(n, M, w, V);
    for (int k = 0; k < n; ++k) {
        const double d = std::max(w[k], 0.0);
        for (int i = 0; i < n; ++i) VD[static_cast<std::size_t>(k) * n + i] = V[static_cast<std::size_t>(k) * n + i] * d;
    }
    for (int j = 0; j < n; ++j)
        for (int i = 0; i < n; ++i) {
            double s = 0;
            for (int k = 0; k < n; ++k) s += VD[static_cast<std::size_t>(k) * n + i] * V[static_cast<std::size_t>(k) * n + j];
            out[static_cast<std::size_t>(j) * n + i] = s;
        }
}

}  // namespace oracle_eig
