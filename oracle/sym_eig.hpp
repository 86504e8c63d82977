// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// Symmetric eigen-decomposition behind the PSD projection of
// energy/psd.hpp:8-14, standing in for Eigen 3.4's SelfAdjointEigenSolver
// (Householder tridiagonalisation + implicit symmetric QR), which is not in
// the image: cyclic Jacobi rotations (Golub & Van Loan, Matrix Computations
// §8.5), swept until the off-diagonal Frobenius norm is below 1e-16 of the
// whole; eigenvalues ascending with their eigenvectors as columns, as Eigen
// returns them. Eigenvalues and the projection agree with Eigen's to
// rounding (the reference's tests pin the projection to 1e-10 / 1e-12).
// Shared by oracle.hpp (the restatement) and eigen_shim/Eigen/Dense (the
// reference's own psd.hpp compiled into oracle/_ref).
#pragma once

#include <algorithm>
#include <cmath>
#include <numeric>
#include <vector>

namespace oracle_eig {

// A: n x n column-major symmetric (read only). w: n eigenvalues ascending.
// V: n x n column-major, column k = eigenvector of w[k].
inline void sym_eig(int n, const double* A, double* w, double* V) {
    std::vector<double> a(A, A + static_cast<std::size_t>(n) * n), v(static_cast<std::size_t>(n) * n, 0.0);
    auto at = [n](std::vector<double>& m, int i, int j) -> double& { return m[static_cast<std::size_t>(j) * n + i]; };
    for (int i = 0; i < n; ++i) at(v, i, i) = 1.0;
    for (int sweep = 0; sweep < 64; ++sweep) {
        double off = 0, tot = 0;
        for (int j = 0; j < n; ++j)
            for (int i = 0; i < n; ++i) {
                const double x = at(a, i, j) * at(a, i, j);
                tot += x;
                if (i != j) off += x;
            }
        if (off <= 1e-32 * tot) break;
        for (int p = 0; p < n - 1; ++p)
            for (int q = p + 1; q < n; ++q) {
                const double apq = at(a, p, q);
                if (apq == 0.0) continue;
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
    }
    std::vector<int> ord(n);
    std::iota(ord.begin(), ord.end(), 0);
    std::stable_sort(ord.begin(), ord.end(), [&](int x, int y) { return at(a, x, x) < at(a, y, y); });
    for (int k = 0; k < n; ++k) {
        w[k] = at(a, ord[k], ord[k]);
        for (int i = 0; i < n; ++i) V[static_cast<std::size_t>(k) * n + i] = at(v, i, ord[k]);
    }
}

// energy/psd.hpp:8-14: V max(w, 0) V^T, in Eigen's evaluation order
// ((V * diag) * V^T, inner index ascending).
inline void project_psd(int n, const double* M, double* out) {
    std::vector<double> w(n), V(static_cast<std::size_t>(n) * n), VD(static_cast<std::size_t>(n) * n);
    sym_eig(n, M, w.data(), V.data());
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
