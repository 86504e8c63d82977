// Second-order forward-mode duals over 12 variables (core/dual2.hpp's
// algebra: value, gradient, symmetric Hessian packed upper), in per-thread
// scratch; shared by the contact producer (distance derivatives) and the
// hinge-bending producer (dihedral angle).
#pragma once

#include "common.cuh"

namespace adipc_gpu {
namespace {

// core/dual2.hpp with N = 12, Hessian packed upper (j >= i at j (j+1)/2 + i)
struct D12 {
    double v;
    double g[12];
    double h[78];
};
__device__ __forceinline__ int hp(int i, int j) { return i <= j ? j * (j + 1) / 2 + i : i * (i + 1) / 2 + j; }

__device__ void d_sub(D12& r, const D12& a, const D12& b) {
    r.v = a.v - b.v;
    for (int i = 0; i < 12; ++i) r.g[i] = a.g[i] - b.g[i];
    for (int i = 0; i < 78; ++i) r.h[i] = a.h[i] - b.h[i];
}
__device__ void d_add(D12& r, const D12& a, const D12& b) {
    r.v = a.v + b.v;
    for (int i = 0; i < 12; ++i) r.g[i] = a.g[i] + b.g[i];
    for (int i = 0; i < 78; ++i) r.h[i] = a.h[i] + b.h[i];
}
// r = a b (r may not alias a or b)
__device__ void d_mul(D12& r, const D12& a, const D12& b) {
    r.v = a.v * b.v;
    for (int i = 0; i < 12; ++i) r.g[i] = a.g[i] * b.v + b.g[i] * a.v;
    for (int j = 0; j < 12; ++j)
        for (int i = 0; i <= j; ++i)
            r.h[hp(i, j)] = a.h[hp(i, j)] * b.v + b.h[hp(i, j)] * a.v + a.g[i] * b.g[j] + b.g[i] * a.g[j];
}
// r = a / b = a * inverse(b) (dual2.hpp:64-75)
__device__ void d_div(D12& r, const D12& a, const D12& b, D12& tmp) {
    const double iv = 1.0 / b.v;
    tmp.v = iv;
    for (int i = 0; i < 12; ++i) tmp.g[i] = -b.g[i] * (iv * iv);
    const double c = 2 * iv * iv * iv;
    for (int j = 0; j < 12; ++j)
        for (int i = 0; i <= j; ++i) tmp.h[hp(i, j)] = -b.h[hp(i, j)] * (iv * iv) + (c * b.g[i]) * b.g[j];
    d_mul(r, a, tmp);
}
// r = |a|^2 = a0 a0 + a1 a1 + a2 a2
__device__ void d_norm2(D12& r, const D12* a, D12& t0, D12& t1) {
    d_mul(t0, a[0], a[0]);
    d_mul(t1, a[1], a[1]);
    d_add(r, t0, t1);
    d_mul(t0, a[2], a[2]);
    d_add(t1, r, t0);
    r = t1;
}
// r = a . b
__device__ void d_dot(D12& r, const D12* a, const D12* b, D12& t0, D12& t1) {
    d_mul(t0, a[0], b[0]);
    d_mul(t1, a[1], b[1]);
    d_add(r, t0, t1);
    d_mul(t0, a[2], b[2]);
    d_add(t1, r, t0);
    r = t1;
}
// r = a x b
__device__ void d_cross(D12* r, const D12* a, const D12* b, D12& t0, D12& t1) {
    const int i1[3] = {1, 2, 0}, i2[3] = {2, 0, 1};
    for (int k = 0; k < 3; ++k) {
        d_mul(t0, a[i1[k]], b[i2[k]]);
        d_mul(t1, a[i2[k]], b[i1[k]]);
        d_sub(r[k], t0, t1);
    }
}

// dual of (xa - xb) with xa, xb the AD variables ka, kb (dual_point + gsub)
__device__ void d_diff(D12& r, double xa, int ka, double xb, int kb) {
    r.v = xa - xb;
    for (int i = 0; i < 12; ++i) r.g[i] = (i == ka ? 1.0 : 0.0) - (i == kb ? 1.0 : 0.0);
    for (int i = 0; i < 78; ++i) r.h[i] = 0.0;
}
// the 3-vector dual (pa - pb) of stencil points a, b (coordinates x[.], variables 3 a + k)
__device__ void d_vdiff(D12* r, const double* x, int a, int b) {
    for (int k = 0; k < 3; ++k) d_diff(r[k], x[3 * a + k], 3 * a + k, x[3 * b + k], 3 * b + k);
}

// r = a s (dual2.hpp:48-53)
__device__ void d_scale(D12& r, const D12& a, double s) {
    r.v = a.v * s;
    for (int i = 0; i < 12; ++i) r.g[i] = a.g[i] * s;
    for (int i = 0; i < 78; ++i) r.h[i] = a.h[i] * s;
}
// r = sqrt(a) (dual2.hpp:80-86); r may alias a
__device__ void d_sqrt(D12& r, const D12& a) {
    const double s = sqrt(a.v), av = a.v;
    for (int j = 0; j < 12; ++j)
        for (int i = 0; i <= j; ++i) r.h[hp(i, j)] = a.h[hp(i, j)] / (2 * s) - a.g[i] * a.g[j] / (4 * av * s);
    for (int i = 0; i < 12; ++i) r.g[i] = a.g[i] / (2 * s);
    r.v = s;
}
// r = atan2(y, x) (dual2.hpp:89-101); r may not alias y or x
__device__ void d_atan2(D12& r, const D12& y, const D12& x) {
    const double r2 = x.v * x.v + y.v * y.v;
    r.v = atan2(y.v, x.v);
    for (int i = 0; i < 12; ++i) r.g[i] = (x.v * y.g[i] - y.v * x.g[i]) / r2;
    const double c1 = y.v * y.v - x.v * x.v, c2 = 2 * x.v * y.v;
    for (int j = 0; j < 12; ++j)
        for (int i = 0; i <= j; ++i) {
            const double gxgy = x.g[i] * y.g[j] + x.g[j] * y.g[i];
            const double dd = x.g[i] * x.g[j] - y.g[i] * y.g[j];
            r.h[hp(i, j)] = (c1 * gxgy + c2 * dd) / (r2 * r2) + (x.v * y.h[hp(i, j)] - y.v * x.h[hp(i, j)]) / r2;
        }
}

}  // namespace
}  // namespace adipc_gpu
