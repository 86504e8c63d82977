// Closed-form first and second derivatives of the per-feature squared
// distances of contact/distance.hpp:111-223 (point-point, point-edge, and the
// plane / line form h^2 / |n|^2 of point-triangle interiors and edge-edge
// interiors). The reference differentiates these with second-order duals
// over all 12 stencil coordinates (core/dual2.hpp); here each distance is a
// function of at most three difference vectors e_p = x[plus_p] - x[minus_p]
// and its gradient / Hessian are written in that 9-dimensional feature space
// by the product and quotient rules, then mapped to the 12 stencil
// coordinates by the 0 / +-1 selection (H12 = S^T Hf S). Values use the
// duals' exact operation order (bitwise the same squared distance); the
// derivatives agree with the duals' to rounding.
//
// Compiles as CUDA (device) and as host C++ (tests/cpp/dist_derivs_check.cpp).
#pragma once

#ifdef __CUDACC__
#define ADIPC_HD __host__ __device__ __forceinline__
#else
#define ADIPC_HD inline
#endif

namespace adipc_gpu {

struct FeatDerivs {
    int nvec;               // difference vectors in use (1..3)
    int plus[3], minus[3];  // stencil node indices (0..3) of e_p = x[plus] - x[minus]
    double v;               // squared distance
    double g[9];            // d v / d e (3 nvec)
    double H[81];           // 9 x 9 column-major over (e_0, e_1, e_2); 3 nvec x 3 nvec used
};

namespace fd {

ADIPC_HD void diff(const double* x, int a, int b, double* e) {
    for (int k = 0; k < 3; ++k) e[k] = x[3 * a + k] - x[3 * b + k];
}
ADIPC_HD void cross(const double* a, const double* b, double* r) {  // d_cross's order
    r[0] = a[1] * b[2] - a[2] * b[1];
    r[1] = a[2] * b[0] - a[0] * b[2];
    r[2] = a[0] * b[1] - a[1] * b[0];
}
ADIPC_HD double dot(const double* a, const double* b) { return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2]; }
// K = [a]x, 3 x 3 row-major: K v = a x v
ADIPC_HD void skew(const double* a, double* K) {
    K[0] = 0;
    K[1] = -a[2];
    K[2] = a[1];
    K[3] = a[2];
    K[4] = 0;
    K[5] = -a[0];
    K[6] = -a[1];
    K[7] = a[0];
    K[8] = 0;
}
// H block (p, q) += s * M (M 3 x 3 row-major: row = component of e_p)
ADIPC_HD void add_block(double* H, int p, int q, const double* M, double s) {
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) H[9 * (3 * q + j) + 3 * p + i] += s * M[3 * i + j];
}
// block (p, q) += s M and block (q, p) += s M^T
ADIPC_HD void add_sym_pair(double* H, int p, int q, const double* M, double s) {
    add_block(H, p, q, M, s);
    double T[9];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) T[3 * j + i] = M[3 * i + j];
    add_block(H, q, p, T, s);
}
// A^T B for 3 x 3 row-major
ADIPC_HD void mtm(const double* A, const double* B, double* C) {
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) C[3 * i + j] = A[i] * B[j] + A[3 + i] * B[3 + j] + A[6 + i] * B[6 + j];
}

}  // namespace fd

// |x_a - x_b|^2 (distance.hpp:111-114)
ADIPC_HD void feat_pp(const double* x, int a, int b, FeatDerivs& f) {
    f.nvec = 1;
    f.plus[0] = a;
    f.minus[0] = b;
    double u[3];
    fd::diff(x, a, b, u);
    f.v = (u[0] * u[0] + u[1] * u[1]) + u[2] * u[2];
    for (int k = 0; k < 81; ++k) f.H[k] = 0;
    for (int k = 0; k < 3; ++k) {
        f.g[k] = 2 * u[k];
        f.H[9 * k + k] = 2;
    }
}

// |w x d|^2 / |d|^2 with d = x_e1 - x_e0, w = x_p - x_e0 (distance.hpp:116-123);
// features e_0 = w, e_1 = d
ADIPC_HD void feat_pe(const double* x, int p, int e0, int e1, FeatDerivs& f) {
    f.nvec = 2;
    f.plus[0] = p;
    f.minus[0] = e0;
    f.plus[1] = e1;
    f.minus[1] = e0;
    double w[3], d[3], n[3];
    fd::diff(x, e1, e0, d);
    fd::diff(x, p, e0, w);
    fd::cross(w, d, n);
    const double A = (n[0] * n[0] + n[1] * n[1]) + n[2] * n[2];
    const double B = (d[0] * d[0] + d[1] * d[1]) + d[2] * d[2];
    // n = w x d: dn/dw = -[d]x, dn/dd = [w]x
    double Kd[9], Kw[9], Kn[9], M[9];
    fd::skew(d, Kd);
    fd::skew(w, Kw);
    fd::skew(n, Kn);
    // f = A / B, B = |d|^2 (dB/dd = 2 d, d2B/dd2 = 2 I): the quotient rule
    // accumulated straight into f (no Hessian temporaries)
    double gA[6], gB[6], t[3];
    fd::cross(d, n, t);  // dA/dw = 2 d x n
    for (int k = 0; k < 3; ++k) gA[k] = 2 * t[k];
    fd::cross(n, w, t);  // dA/dd = 2 n x w
    for (int k = 0; k < 3; ++k) gA[3 + k] = 2 * t[k];
    for (int k = 0; k < 3; ++k) {
        gB[k] = 0;
        gB[3 + k] = 2 * d[k];
    }
    const double ib = 1.0 / B, ib2 = ib * ib, ib3 = ib2 * ib;
    for (int i = 0; i < 6; ++i) f.g[i] = gA[i] * ib - A * gB[i] * ib2;
    for (int j = 0; j < 6; ++j)
        for (int i = 0; i < 6; ++i)
            f.H[9 * j + i] = -(gA[i] * gB[j] + gB[i] * gA[j]) * ib2 + 2.0 * A * gB[i] * gB[j] * ib3;
    fd::mtm(Kd, Kd, M);  // d2A/dw2 = 2 [d]x^T [d]x
    fd::add_block(f.H, 0, 0, M, 2 * ib);
    fd::mtm(Kw, Kw, M);  // d2A/dd2 = 2 [w]x^T [w]x
    fd::add_block(f.H, 1, 1, M, 2 * ib);
    fd::mtm(Kd, Kw, M);  // d2A/dw dd = -2 [d]x^T [w]x - 2 [n]x
    for (int k = 0; k < 9; ++k) M[k] = -M[k] - Kn[k];
    fd::add_sym_pair(f.H, 0, 1, M, 2 * ib);
    for (int k = 0; k < 3; ++k) f.H[9 * (3 + k) + 3 + k] -= 2 * A * ib2;  // - A d2B/dd2 / B^2
    f.v = A * (1.0 / B);  // the duals divide as a * (1 / b)
}

// h^2 / |n|^2 with n = (x_q1 - x_q0) x (x_r1 - x_r0), h = (x_o - x_base) . n
// (distance.hpp:125-140: triangle plane and line-line forms); features
// e_0 = u = q1 - q0, e_1 = w = r1 - r0, e_2 = c = o - base
ADIPC_HD void feat_hn(const double* x, int q0, int q1, int r0, int r1, int o, int base, FeatDerivs& f) {
    f.nvec = 3;
    f.plus[0] = q1;
    f.minus[0] = q0;
    f.plus[1] = r1;
    f.minus[1] = r0;
    f.plus[2] = o;
    f.minus[2] = base;
    double u[3], w[3], c[3], n[3];
    fd::diff(x, q1, q0, u);
    fd::diff(x, r1, r0, w);
    fd::cross(u, w, n);
    fd::diff(x, o, base, c);
    const double h = fd::dot(c, n);
    const double a = h * h;
    const double N = (n[0] * n[0] + n[1] * n[1]) + n[2] * n[2];
    double Ku[9], Kw[9], Kc[9], Kn[9], M[9], t[3];  // [.]x matrices, row-major
    fd::skew(u, Ku);
    fd::skew(w, Kw);
    fd::skew(c, Kc);
    fd::skew(n, Kn);
    // h = c . (u x w): dh/du = w x c, dh/dw = c x u, dh/dc = n;
    // d2h/du dw = -[c]x, d2h/dc du = -[w]x, d2h/dc dw = [u]x
    double gh[9];
    fd::cross(w, c, t);
    for (int k = 0; k < 3; ++k) gh[k] = t[k];
    fd::cross(c, u, t);
    for (int k = 0; k < 3; ++k) gh[3 + k] = t[k];
    for (int k = 0; k < 3; ++k) gh[6 + k] = n[k];
    // N = |u x w|^2: dN/du = 2 w x n, dN/dw = 2 n x u
    double gN[9];
    fd::cross(w, n, t);
    for (int k = 0; k < 3; ++k) gN[k] = 2 * t[k];
    fd::cross(n, u, t);
    for (int k = 0; k < 3; ++k) gN[3 + k] = 2 * t[k];
    for (int k = 0; k < 3; ++k) gN[6 + k] = 0;
    // f = a / N with a = h^2 (da = 2 h dh, d2a = 2 dh dh^T + 2 h d2h): the
    // quotient rule accumulated straight into f
    const double ib = 1.0 / N, ib2 = ib * ib, ib3 = ib2 * ib;
    for (int i = 0; i < 9; ++i) f.g[i] = 2 * h * gh[i] * ib - a * gN[i] * ib2;
    for (int j = 0; j < 9; ++j)
        for (int i = 0; i < 9; ++i)
            f.H[9 * j + i] = 2 * gh[i] * gh[j] * ib - (2 * h * gh[i] * gN[j] + gN[i] * 2 * h * gh[j]) * ib2 +
                             2.0 * a * gN[i] * gN[j] * ib3;
    // 2 h d2h / N: d2h/du dw = -[c]x, d2h/dc du = -[w]x, d2h/dc dw = [u]x
    for (int k = 0; k < 9; ++k) M[k] = -Kc[k];
    fd::add_sym_pair(f.H, 0, 1, M, 2 * h * ib);
    for (int k = 0; k < 9; ++k) M[k] = -Kw[k];
    fd::add_sym_pair(f.H, 2, 0, M, 2 * h * ib);
    fd::add_sym_pair(f.H, 2, 1, Ku, 2 * h * ib);
    // - a d2N / N^2: d2N/du2 = 2 [w]x^T [w]x, d2N/dw2 = 2 [u]x^T [u]x,
    // d2N/du dw = -2 [w]x^T [u]x - 2 [n]x
    const double sN = -2 * a * ib2;
    fd::mtm(Kw, Kw, M);
    fd::add_block(f.H, 0, 0, M, sN);
    fd::mtm(Ku, Ku, M);
    fd::add_block(f.H, 1, 1, M, sN);
    fd::mtm(Kw, Ku, M);
    for (int k = 0; k < 9; ++k) M[k] = -M[k] - Kn[k];
    fd::add_sym_pair(f.H, 0, 1, M, sN);
    f.v = a * (1.0 / N);
}

// feature -> stencil: g12 = S^T g, H12 = S^T (b2 g g^T + b1 Hf) S scaled
// later by the caller; coefficient of node a in e_p
ADIPC_HD double feat_coef(const FeatDerivs& f, int p, int a) {
    return (f.plus[p] == a ? 1.0 : 0.0) - (f.minus[p] == a ? 1.0 : 0.0);
}
ADIPC_HD void feat_grad12(const FeatDerivs& f, double* g12) {
    for (int a = 0; a < 4; ++a)
        for (int i = 0; i < 3; ++i) {
            double s = 0;
            for (int p = 0; p < f.nvec; ++p) s += feat_coef(f, p, a) * f.g[3 * p + i];
            g12[3 * a + i] = s;
        }
}
// H12 (12 x 12 column-major) = S^T Hf S for a 9 x 9 feature-space matrix Hf
ADIPC_HD void feat_lift(const FeatDerivs& f, const double* Hf, double* H12) {
    double C[4][3];
    for (int a = 0; a < 4; ++a)
        for (int p = 0; p < 3; ++p) C[a][p] = p < f.nvec ? feat_coef(f, p, a) : 0.0;
    for (int b = 0; b < 4; ++b)
        for (int j = 0; j < 3; ++j)
            for (int a = 0; a < 4; ++a)
                for (int i = 0; i < 3; ++i) {
                    double s = 0;
                    for (int q = 0; q < f.nvec; ++q) {
                        if (C[b][q] == 0) continue;
                        double t = 0;
                        for (int p = 0; p < f.nvec; ++p)
                            if (C[a][p] != 0) t += C[a][p] * Hf[9 * (3 * q + j) + 3 * p + i];
                        s += C[b][q] * t;
                    }
                    H12[12 * (3 * b + j) + 3 * a + i] = s;
                }
}

// the feature of a classified stencil (kind 0: PT, 1: EE; region as in
// classify_pt / classify_ee), stencil coordinates x[12]
ADIPC_HD void feature_derivs(int kind, int region, const double* x, FeatDerivs& f) {
    if (kind == 0) {
        switch (region) {
            case 0: feat_pp(x, 0, 1, f); break;
            case 1: feat_pp(x, 0, 2, f); break;
            case 2: feat_pp(x, 0, 3, f); break;
            case 3: feat_pe(x, 0, 1, 2, f); break;
            case 4: feat_pe(x, 0, 2, 3, f); break;
            case 5: feat_pe(x, 0, 3, 1, f); break;
            default: feat_hn(x, 1, 2, 1, 3, 0, 1, f); break;
        }
        return;
    }
    switch (region) {
        case 0: feat_pp(x, 0, 2, f); break;
        case 1: feat_pp(x, 0, 3, f); break;
        case 2: feat_pp(x, 1, 2, f); break;
        case 3: feat_pp(x, 1, 3, f); break;
        case 4: feat_pe(x, 0, 2, 3, f); break;
        case 5: feat_pe(x, 1, 2, 3, f); break;
        case 6: feat_pe(x, 2, 0, 1, f); break;
        case 7: feat_pe(x, 3, 0, 1, f); break;
        default: feat_hn(x, 0, 1, 2, 3, 2, 0, f); break;
    }
}

}  // namespace adipc_gpu
