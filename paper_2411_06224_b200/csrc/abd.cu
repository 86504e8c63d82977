// Two-level affine-body Hessian reduction on B200 (replaces
// two_level_abd_reduce, sparse/abd_reduce.hpp:32-74, called at
// solver/incremental_potential.hpp:392-393; paper Sec. 4.2 / Alg. 2-3).
//   level 1: the contact node-pair stream is sorted + reduced with the same
//            device sort/segment path as the global assembly (bitwise equal to
//            the reference's deterministic mode);
//   then:    one thread per unique node pair pushes the merged 3x3 block
//            through the body Jacobians and emits its 1 / 4 / 10 / 16 tiles
//            (block_split.hpp:10-33 with emit()'s canonicalisation) at a
//            scanned offset, so the tile stream has exactly the reference's
//            order (which the level-2 deterministic sums depend on).
// Products use explicit round-to-nearest mul/add in the reference's
// evaluation order (left-associated J^T C J, inner index ascending), so tiles
// match the oracle bit for bit.
#include "context.hpp"
#include "scan.cuh"

namespace adipc_gpu {

namespace {

struct Map {
    std::int32_t n_fem, n_bodies, n_abd;
    const std::int32_t* body;  // abd node -> body
    const double* jac;         // 36 doubles per abd node, 3x12 column-major
    __device__ bool is_fem(std::int32_t v) const { return v < n_fem; }
    __device__ std::int32_t body_of(std::int32_t v) const { return body[v - n_fem]; }
    __device__ std::int32_t base(std::int32_t b) const { return n_fem + 4 * b; }
    // J(r, c) of node v
    __device__ double J(std::int32_t v, int r, int c) const { return jac[36 * static_cast<std::int64_t>(v - n_fem) + 3 * c + r]; }
};

__device__ __forceinline__ double mac3(double a0, double b0, double a1, double b1, double a2, double b2) {
    // ((a0 b0 + a1 b1) + a2 b2), no contraction
    return __dadd_rn(__dadd_rn(__dmul_rn(a0, b0), __dmul_rn(a1, b1)), __dmul_rn(a2, b2));
}

// Output writer with emit() canonicalisation (block_coo.hpp:38-46).
__device__ __forceinline__ void emit(std::int32_t r, std::int32_t c, const double* t /*3x3 col-major*/,
                                     std::uint64_t* ok, double* ov, std::int64_t pos) {
    if (r <= c) {
        ok[pos] = (static_cast<std::uint64_t>(static_cast<std::uint32_t>(r)) << 32) | static_cast<std::uint32_t>(c);
        for (int k = 0; k < 9; ++k) ov[9 * pos + k] = t[k];
    } else {
        ok[pos] = (static_cast<std::uint64_t>(static_cast<std::uint32_t>(c)) << 32) | static_cast<std::uint32_t>(r);
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) ov[9 * pos + 3 * j + i] = t[3 * i + j];
    }
}

__device__ __forceinline__ int tile_count(const Map& m, std::int32_t i, std::int32_t j) {
    const bool fi = m.is_fem(i), fj = m.is_fem(j);
    if (fi && fj) return 1;
    if (fi != fj) return 4;
    return m.body_of(i) != m.body_of(j) ? 16 : 10;
}

__global__ void k_abd_count(const std::uint32_t* __restrict__ rows, const std::uint32_t* __restrict__ cols,
                            std::int64_t U, Map m, std::int32_t* __restrict__ cnt) {
    for (std::int64_t e = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; e < U;
         e += static_cast<std::int64_t>(gridDim.x) * blockDim.x)
        cnt[e] = tile_count(m, static_cast<std::int32_t>(rows[e]), static_cast<std::int32_t>(cols[e]));
}

// K tile (ti, tj) of J_i^T C J_j (12x12), computed as in (J_i^T C) J_j.
__device__ __forceinline__ void jtcj_tile(const Map& m, std::int32_t i, std::int32_t j, const double* C, int ti, int tj,
                                          double* out) {
    // JtC rows 3ti..3ti+2: JtC(a, k) = sum_m J_i(m, 3ti+a) C(m, k)
    double jtc[9];  // [a][k] row-major small
    for (int a = 0; a < 3; ++a)
        for (int k = 0; k < 3; ++k)
            jtc[3 * a + k] = mac3(m.J(i, 0, 3 * ti + a), C[3 * k + 0], m.J(i, 1, 3 * ti + a), C[3 * k + 1],
                                  m.J(i, 2, 3 * ti + a), C[3 * k + 2]);
    // (J^T C) J is an Eigen GEMM (12x3 * 3x12: accumulators start at zero),
    // so a -0.0 entry comes out +0.0: the trailing + 0.0 reproduces that
    for (int b = 0; b < 3; ++b)
        for (int a = 0; a < 3; ++a)
            out[3 * b + a] = __dadd_rn(mac3(jtc[3 * a + 0], m.J(j, 0, 3 * tj + b), jtc[3 * a + 1],
                                            m.J(j, 1, 3 * tj + b), jtc[3 * a + 2], m.J(j, 2, 3 * tj + b)),
                                       0.0);
}

__global__ void k_abd_emit(const std::uint32_t* __restrict__ rows, const std::uint32_t* __restrict__ cols,
                           const double* __restrict__ blocks, std::int64_t U, Map m, const std::int64_t* __restrict__ off,
                           std::uint64_t* __restrict__ ok, double* __restrict__ ov) {
    for (std::int64_t e = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; e < U;
         e += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        const std::int32_t i = static_cast<std::int32_t>(rows[e]), j = static_cast<std::int32_t>(cols[e]);
        double C[9];
        for (int k = 0; k < 9; ++k) C[k] = blocks[blk(e, k)];
        std::int64_t pos = off[e];
        const bool fi = m.is_fem(i), fj = m.is_fem(j);
        double t[9];
        if (fi && fj) {
            emit(i, j, C, ok, ov, pos);
        } else if (fi && !fj) {  // split_3x12(i, base(bj), C J_j)
            const std::int32_t cb = m.base(m.body_of(j));
            for (int tt = 0; tt < 4; ++tt) {
                for (int b = 0; b < 3; ++b)
                    for (int a = 0; a < 3; ++a)
                        t[3 * b + a] = mac3(C[a], m.J(j, 0, 3 * tt + b), C[3 + a], m.J(j, 1, 3 * tt + b), C[6 + a],
                                            m.J(j, 2, 3 * tt + b));
                emit(i, cb + tt, t, ok, ov, pos++);
            }
        } else if (!fi && fj) {  // split_12x3(base(bi), j, J_i^T C) — unreachable for canonical keys
            const std::int32_t rb = m.base(m.body_of(i));
            for (int tt = 0; tt < 4; ++tt) {
                for (int b = 0; b < 3; ++b)
                    for (int a = 0; a < 3; ++a)
                        t[3 * b + a] = mac3(m.J(i, 0, 3 * tt + a), C[3 * b], m.J(i, 1, 3 * tt + a), C[3 * b + 1],
                                            m.J(i, 2, 3 * tt + a), C[3 * b + 2]);
                emit(rb + tt, j, t, ok, ov, pos++);
            }
        } else {
            const std::int32_t bi = m.body_of(i), bj = m.body_of(j);
            if (bi != bj) {  // split_12x12
                for (int ti = 0; ti < 4; ++ti)
                    for (int tj = 0; tj < 4; ++tj) {
                        jtcj_tile(m, i, j, C, ti, tj, t);
                        emit(m.base(bi) + ti, m.base(bj) + tj, t, ok, ov, pos++);
                    }
            } else if (i == j) {  // split_sym_12x12(J^T C J)
                for (int ti = 0; ti < 4; ++ti)
                    for (int tj = ti; tj < 4; ++tj) {
                        jtcj_tile(m, i, j, C, ti, tj, t);
                        emit(m.base(bi) + ti, m.base(bi) + tj, t, ok, ov, pos++);
                    }
            } else {  // split_sym_12x12(K + K^T)
                double u[9];
                for (int ti = 0; ti < 4; ++ti)
                    for (int tj = ti; tj < 4; ++tj) {
                        jtcj_tile(m, i, j, C, ti, tj, t);
                        jtcj_tile(m, i, j, C, tj, ti, u);
                        double s[9];
                        for (int b = 0; b < 3; ++b)
                            for (int a = 0; a < 3; ++a) s[3 * b + a] = __dadd_rn(t[3 * b + a], u[3 * a + b]);
                        emit(m.base(bi) + ti, m.base(bi) + tj, s, ok, ov, pos++);
                    }
            }
        }
    }
}

}  // namespace

// LEVEL 1 + tile emission into `ok` / `ov` (reserved here to the exact tile
// count when `grow`; otherwise out_cap bounds it). Scratch lives in the
// context (reused across Newton iterations, freed with it).
static std::int64_t two_level_impl(Ctx& c, const std::uint64_t* d_keys, const double* d_vals, std::int64_t Tn,
                                   std::int32_t n_fem, std::int32_t n_bodies, std::int32_t n_abd,
                                   const std::int32_t* d_body, const double* d_jac36, DBuf<std::uint64_t>* grow_k,
                                   DBuf<double>* grow_v, std::uint64_t* d_out_keys, double* d_out_vals,
                                   std::int64_t out_cap) {
    cudaStream_t st = c.stream;
    DeviceMatrix& merged = c.abd_l1;
    const std::int32_t n_nodes = n_fem + n_abd;
    sort_reduce(c, d_keys, d_vals, Tn, n_nodes, merged);  // LEVEL 1 (abd_reduce.hpp:35-37)
    const std::int64_t U = merged.U;
    if (U == 0) return 0;
    Map m{n_fem, n_bodies, n_abd, d_body, d_jac36};
    c.abd_cnt.reserve(U);
    c.abd_off.reserve(U + 1);
    k_abd_count<<<grid_for(U, 256, 16), 256, 0, st>>>(merged.rows.p, merged.cols.p, U, m, c.abd_cnt.p);
    ADIPC_LAUNCH_CHECK();
    exclusive_scan(c.abd_cnt.p, U, c.abd_off.p, c.scan_scratch, st);
    std::int64_t total = 0;
    ADIPC_CUDA(cudaMemcpyAsync(&total, c.abd_off.p + U, sizeof(total), cudaMemcpyDeviceToHost, st));
    ADIPC_CUDA(cudaStreamSynchronize(st));
    if (grow_k) {
        grow_k->reserve(static_cast<std::size_t>(total));
        grow_v->reserve(9 * static_cast<std::size_t>(total));
        d_out_keys = grow_k->p;
        d_out_vals = grow_v->p;
    } else if (total > out_cap) {
        throw StatusError(kInvalidArgument, "two_level_abd_reduce: output capacity too small");
    }
    k_abd_emit<<<grid_for(U, 128, 16), 128, 0, st>>>(merged.rows.p, merged.cols.p, merged.blocks.p, U, m,
                                                      c.abd_off.p, d_out_keys, d_out_vals);
    ADIPC_LAUNCH_CHECK();
    return total;
}

std::int64_t two_level_abd_reduce(Ctx& c, const std::uint64_t* d_keys, const double* d_vals, std::int64_t Tn,
                                  std::int32_t n_fem, std::int32_t n_bodies, std::int32_t n_abd,
                                  const std::int32_t* d_body, const double* d_jac36, std::uint64_t* d_out_keys,
                                  double* d_out_vals, std::int64_t out_cap) {
    const std::int64_t total = two_level_impl(c, d_keys, d_vals, Tn, n_fem, n_bodies, n_abd, d_body, d_jac36, nullptr,
                                              nullptr, d_out_keys, d_out_vals, out_cap);
    ADIPC_CUDA(cudaStreamSynchronize(c.stream));
    return total;
}

// The device fast path of assemble_contact (incremental_potential.hpp:
// 392-394 then 253-257): the reduced tiles stay on the device in the
// context's tile buffers and are appended to the DOF stream as its second
// segment — filter_pinned, sort and reduce read both segments in place.
std::int64_t assemble_contact(Ctx& c, const std::uint64_t* d_keys, const double* d_vals, std::int64_t T,
                              const std::uint64_t* d_nkeys, const double* d_nvals, std::int64_t Tn,
                              std::int32_t n_fem, std::int32_t n_bodies, std::int32_t n_abd, const std::int32_t* d_body,
                              const double* d_jac36, std::int32_t n, const std::uint8_t* d_pinned,
                              cudaEvent_t vals_ready) {
    std::int64_t Tt = 0;
    if (Tn > 0)
        Tt = two_level_impl(c, d_nkeys, d_nvals, Tn, n_fem, n_bodies, n_abd, d_body, d_jac36, &c.tile_keys,
                            &c.tile_vals, nullptr, nullptr, 0);
    if (d_pinned)
        assemble_filtered(c, d_keys, d_vals, T, n, d_pinned, vals_ready, c.tile_keys.p, c.tile_vals.p, Tt);
    else
        assemble_filtered(c, d_keys, d_vals, T, n, nullptr, vals_ready, c.tile_keys.p, c.tile_vals.p, Tt);
    return Tt;
}

}  // namespace adipc_gpu
