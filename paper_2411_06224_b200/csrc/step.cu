// The step after the solve, on the device: what
// TimeStepper does with the PCG direction before the line search
// (adipc/solver/newton.hpp:257-290). Vectors are in the reference's block
// numbering: FEM vertices first, then 4 blocks (12 dofs: p, then the rows of
// A) per affine body (DofMap, abd_reduce.hpp:11-27).
#include <cstring>

#include "context.hpp"

namespace adipc_gpu {

namespace {

// IEEE ordering of non-negative doubles = ordering of their bit patterns
__device__ __forceinline__ void atomic_max_nonneg(unsigned long long* slot, double v) {
    atomicMax(slot, static_cast<unsigned long long>(__double_as_longlong(v)));
}

// step_inf_norm (newton.hpp:257-270): max over FEM vertices of |d_i| and over
// bodies of |d_p| + |d_A|_F max|xbar|
__global__ void k_step_inf_norm(const double* __restrict__ d, std::int32_t n_fem, std::int32_t n_bodies,
                                const double* __restrict__ max_xbar, unsigned long long* __restrict__ out) {
    double worst = 0;
    for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x;
         i < static_cast<std::int64_t>(n_fem) + n_bodies; i += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        double v;
        if (i < n_fem) {
            const double* s = d + 3 * i;
            v = sqrt(__dadd_rn(__dadd_rn(__dmul_rn(s[0], s[0]), __dmul_rn(s[1], s[1])), __dmul_rn(s[2], s[2])));
        } else {
            const std::int64_t b = i - n_fem;
            const double* s = d + 3 * (static_cast<std::int64_t>(n_fem) + 4 * b);
            double p2 = 0, a2 = 0;
            for (int k = 0; k < 3; ++k) p2 = __dadd_rn(p2, __dmul_rn(s[k], s[k]));
            for (int k = 3; k < 12; ++k) a2 = __dadd_rn(a2, __dmul_rn(s[k], s[k]));
            v = __dadd_rn(sqrt(p2), __dmul_rn(sqrt(a2), max_xbar[b]));
        }
        worst = v > worst ? v : worst;  // std::max(worst, v): a NaN v is ignored
    }
    for (int o = 16; o > 0; o >>= 1) {
        const double w = __shfl_xor_sync(0xffffffffu, worst, o);
        worst = w > worst ? w : worst;
    }
    if ((threadIdx.x & 31) == 0) atomic_max_nonneg(out, worst);
}

// apply_direction (newton.hpp:283-290): out = s + alpha d over every block
// (x of the FEM vertices, q of the bodies), each component as x + alpha * d
__global__ void k_apply_direction(const double* __restrict__ s, const double* __restrict__ d, double alpha,
                                  std::int64_t n, double* __restrict__ out) {
    for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<std::int64_t>(gridDim.x) * blockDim.x)
        out[i] = __dadd_rn(s[i], __dmul_rn(alpha, d[i]));
}

// node_displacements (newton.hpp:272-281): FEM nodes copy their block; an
// affine-body node n moves by J(n) d_body, J the 3x12 column-major jacobian
__global__ void k_node_displacements(const double* __restrict__ d, std::int32_t n_fem, std::int32_t n_abd,
                                     const std::int32_t* __restrict__ abd_body, const double* __restrict__ jac36,
                                     double* __restrict__ out) {
    for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x;
         i < static_cast<std::int64_t>(n_fem) + n_abd; i += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        if (i < n_fem) {
            for (int k = 0; k < 3; ++k) out[3 * i + k] = d[3 * i + k];
        } else {
            const std::int64_t a = i - n_fem;
            const double* J = jac36 + 36 * a;
            const double* q = d + 3 * (static_cast<std::int64_t>(n_fem) + 4 * static_cast<std::int64_t>(abd_body[a]));
            for (int r = 0; r < 3; ++r) {
                double acc = 0;
                for (int c = 0; c < 12; ++c) acc = __dadd_rn(acc, __dmul_rn(J[3 * c + r], q[c]));
                out[3 * i + r] = acc;
            }
        }
    }
}

// contact_node_positions (scene.hpp:112-120): FEM vertices copy x; an
// affine-body node is affine_point(q, x_bar) = A x_bar + p (core/types.hpp:
// 34-40) in that operation order — not J q, whose sum order differs in the
// last bit (a friction base position feeds dx = x - base at 1e-5 scale).
// x_bar_k is the node Jacobian's (0, 3 + k) entry.
__global__ void k_contact_positions(const double* __restrict__ st, std::int32_t n_fem, std::int32_t n_abd,
                                    const std::int32_t* __restrict__ abd_body, const double* __restrict__ jac36,
                                    double* __restrict__ out) {
    for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x;
         i < static_cast<std::int64_t>(n_fem) + n_abd; i += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        if (i < n_fem) {
            for (int k = 0; k < 3; ++k) out[3 * i + k] = st[3 * i + k];
        } else {
            const std::int64_t a = i - n_fem;
            const double* J = jac36 + 36 * a;
            const double x0 = J[9], x1 = J[12], x2 = J[15];
            const double* q = st + 3 * (static_cast<std::int64_t>(n_fem) + 4 * static_cast<std::int64_t>(abd_body[a]));
            for (int r = 0; r < 3; ++r) {
                const double* Ar = q + 3 + 3 * r;
                out[3 * i + r] = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(Ar[0], x0), __dmul_rn(Ar[1], x1)),
                                                     __dmul_rn(Ar[2], x2)),
                                           q[r]);
            }
        }
    }
}

// assemble_contact's gradient lift (incremental_potential.hpp:395-403): a FEM
// node's contact gradient adds to its slot, an affine-body node's through
// J^T to its body's 12 dofs (fp64 RED); pinned slots receive nothing (the
// reference zeroes them right after, :253-254)
__global__ void k_lift_node_grad(const double* __restrict__ g, std::int32_t n_fem, std::int32_t n_abd,
                                 const std::int32_t* __restrict__ abd_body, const double* __restrict__ jac36,
                                 const std::uint8_t* __restrict__ pinned, double* __restrict__ grad) {
    for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x;
         i < static_cast<std::int64_t>(n_fem) + n_abd; i += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        const double g0 = g[3 * i], g1 = g[3 * i + 1], g2 = g[3 * i + 2];
        if (g0 * g0 + g1 * g1 + g2 * g2 == 0) continue;
        if (i < n_fem) {
            if (pinned && pinned[i]) continue;
            atomicAdd(grad + 3 * i, g0);
            atomicAdd(grad + 3 * i + 1, g1);
            atomicAdd(grad + 3 * i + 2, g2);
        } else {
            const std::int64_t a = i - n_fem;
            const double* J = jac36 + 36 * a;
            const std::int64_t base = static_cast<std::int64_t>(n_fem) + 4 * static_cast<std::int64_t>(abd_body[a]);
            double* q = grad + 3 * base;
            for (int c = 0; c < 12; ++c)
                if (!pinned || !pinned[base + c / 3])
                    atomicAdd(q + c, J[3 * c] * g0 + J[3 * c + 1] * g1 + J[3 * c + 2] * g2);
        }
    }
}

}  // namespace

void lift_node_grad(Ctx& c, const double* d_node_grad, std::int32_t n_fem, std::int32_t n_abd,
                    const std::int32_t* d_abd_body, const double* d_jac36, const std::uint8_t* d_pinned,
                    double* d_grad) {
    const std::int64_t n = static_cast<std::int64_t>(n_fem) + n_abd;
    if (n <= 0) return;
    k_lift_node_grad<<<grid_for(n, 256, 16), 256, 0, c.stream>>>(d_node_grad, n_fem, n_abd, d_abd_body, d_jac36,
                                                                d_pinned, d_grad);
    ADIPC_LAUNCH_CHECK();
}

void contact_positions(Ctx& c, const double* d_state, std::int32_t n_fem, std::int32_t n_abd,
                       const std::int32_t* d_abd_body, const double* d_jac36, double* d_out) {
    const std::int64_t n = static_cast<std::int64_t>(n_fem) + n_abd;
    if (n <= 0) return;
    k_contact_positions<<<grid_for(n, 256, 16), 256, 0, c.stream>>>(d_state, n_fem, n_abd, d_abd_body, d_jac36, d_out);
    ADIPC_LAUNCH_CHECK();
}

double step_inf_norm(Ctx& c, const double* d_dir, std::int32_t n_fem, std::int32_t n_bodies,
                     const double* d_max_xbar) {
    c.step_max.reserve(1);
    unsigned long long* slot = c.step_max.p;
    ADIPC_CUDA(cudaMemsetAsync(slot, 0, sizeof(unsigned long long), c.stream));
    const std::int64_t n = static_cast<std::int64_t>(n_fem) + n_bodies;
    if (n > 0) {
        k_step_inf_norm<<<grid_for(n, 256, 8), 256, 0, c.stream>>>(d_dir, n_fem, n_bodies, d_max_xbar, slot);
        ADIPC_LAUNCH_CHECK();
    }
    unsigned long long bits = 0;
    ADIPC_CUDA(cudaMemcpyAsync(&bits, slot, sizeof(bits), cudaMemcpyDeviceToHost, c.stream));
    ADIPC_CUDA(cudaStreamSynchronize(c.stream));
    double v;
    std::memcpy(&v, &bits, sizeof(v));
    return v;
}

void apply_direction(Ctx& c, const double* d_state, const double* d_dir, double alpha, std::int64_t n,
                     double* d_out) {
    if (n <= 0) return;
    k_apply_direction<<<grid_for(n, 256, 16), 256, 0, c.stream>>>(d_state, d_dir, alpha, n, d_out);
    ADIPC_LAUNCH_CHECK();
}

void node_displacements(Ctx& c, const double* d_dir, std::int32_t n_fem, std::int32_t n_abd,
                        const std::int32_t* d_abd_body, const double* d_jac36, double* d_out) {
    const std::int64_t n = static_cast<std::int64_t>(n_fem) + n_abd;
    if (n <= 0) return;
    k_node_displacements<<<grid_for(n, 256, 16), 256, 0, c.stream>>>(d_dir, n_fem, n_abd, d_abd_body, d_jac36,
                                                                    d_out);
    ADIPC_LAUNCH_CHECK();
}

}  // namespace adipc_gpu
