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
// cyclic Jacobi (oracle/sym_eig.hpp's rotations) with the threshold rule — an
// off-diagonal entry below 1e-17 of the Frobenius norm (rounding level) is
// zeroed instead of rotated and the sweeps end once one rotates nothing —
// then V max(w, 0) V^T
template <int N>
__device__ __noinline__ void project_sym(double* a) {
    double v[N * N];
    for (int k = 0; k < N * N; ++k) v[k] = (k % (N + 1) == 0) ? 1.0 : 0.0;
    double tot = 0;  // ||a||_F^2, invariant under the rotations
    for (int k = 0; k < N * N; ++k) tot += a[k] * a[k];
    const double negligible = 1e-34 * tot;
    for (int sweep = 0; sweep < 64; ++sweep) {
        bool rotated = false;
        for (int p = 0; p < N - 1; ++p)
            for (int q = p + 1; q < N; ++q) {
                const double apq = a[N * q + p];
                if (apq == 0.0) continue;
                if (apq * apq <= negligible) {
                    a[N * q + p] = a[N * p + q] = 0.0;
                    continue;
                }
                rotated = true;
                const double theta = (a[N * q + q] - a[N * p + p]) / (2.0 * apq);
                const double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
                const double c = rsqrt(t * t + 1.0), s = t * c;
                for (int k = 0; k < N; ++k) {
                    const double kp = a[N * p + k], kq = a[N * q + k];
                    a[N * p + k] = c * kp - s * kq;
                    a[N * q + k] = s * kp + c * kq;
                }
                for (int k = 0; k < N; ++k) {
                    const double pk_ = a[N * k + p], qk = a[N * k + q];
                    a[N * k + p] = c * pk_ - s * qk;
                    a[N * k + q] = s * pk_ + c * qk;
                }
                for (int k = 0; k < N; ++k) {
                    const double kp = v[N * p + k], kq = v[N * q + k];
                    v[N * p + k] = c * kp - s * kq;
                    v[N * q + k] = s * kp + c * kq;
                }
            }
        if (!rotated) break;
    }
    double w[N];
    for (int k = 0; k < N; ++k) w[k] = a[(N + 1) * k] > 0 ? a[(N + 1) * k] : 0.0;
    for (int j = 0; j < N; ++j)
        for (int i = 0; i < N; ++i) {
            double s = 0;
            for (int k = 0; k < N; ++k) s += v[N * k + i] * w[k] * v[N * k + j];
            a[N * j + i] = s;
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
