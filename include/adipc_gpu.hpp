// adipc_gpu.hpp — C++ shim over the C-ABI (adipc_gpu.h) with the reference's
// own signatures, for dropping the B200 path into the reference `adipc`
// sources. Include it AFTER the adipc headers; it needs
// the reference's types (Eigen-based Mat3 / VecX, BlockTripletStream,
// SortedSymBlockCoo, MasHierarchy, Preconditioner, PcgResult).
//
// Memory layout: with Eigen, std::vector<Mat3> is 9 contiguous column-major
// doubles per block and VecX 3n contiguous doubles, exactly the C-ABI's
// layout, so every call passes the vectors' storage straight through. When a
// matrix type carries more than its coefficients (sizeof(Mat3) != 72, e.g.
// the Eigen subset the tests compile the reference with), the blocks are
// packed into / unpacked from a contiguous buffer instead.
#pragma once

#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "adipc_gpu.h"

namespace adipc::gpu {

// N contiguous doubles per element (zero-copy when the type is exactly that)
template <int N, class M>
const double* flat_in(const std::vector<M>& v, std::vector<double>& tmp) {
    if (v.empty()) return nullptr;
    if constexpr (sizeof(M) == N * sizeof(double)) {
        return v[0].data();
    } else {
        tmp.resize(v.size() * N);
        for (std::size_t i = 0; i < v.size(); ++i) std::memcpy(tmp.data() + N * i, v[i].data(), N * sizeof(double));
        return tmp.data();
    }
}
template <int N, class M>
double* flat_out(std::vector<M>& v, std::vector<double>& tmp) {
    if (v.empty()) return nullptr;
    if constexpr (sizeof(M) == N * sizeof(double)) {
        return v[0].data();
    } else {
        tmp.resize(v.size() * N);
        return tmp.data();
    }
}
template <int N, class M>
void flat_back(std::vector<M>& v, const std::vector<double>& tmp) {
    if constexpr (sizeof(M) != N * sizeof(double))
        for (std::size_t i = 0; i < v.size(); ++i) std::memcpy(v[i].data(), tmp.data() + N * i, N * sizeof(double));
}

inline void check(int rc, const adipc_gpu_ctx* ctx) {
    if (rc == ADIPC_OK) return;
    const std::string msg = adipc_gpu_last_error(ctx);
    if (rc == ADIPC_INVALID_ARGUMENT) throw std::invalid_argument(msg);   // e.g. reduction.hpp:34
    throw std::runtime_error(msg);                                         // mas.hpp:74-77, CUDA
}

// One device context per scene (TimeStepper owns one; not thread-safe).
class Context {
public:
    explicit Context(int device = 0) { check(adipc_gpu_create(device, &ctx_), nullptr); }
    ~Context() { adipc_gpu_destroy(ctx_); }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
    adipc_gpu_ctx* get() const { return ctx_; }

private:
    adipc_gpu_ctx* ctx_ = nullptr;
};

// sort_stream + fast_hash_reduction (incremental_potential.hpp:256-257) in one
// call; the result stays on the device for the preconditioner and PCG, and is
// copied back into `hess` for host consumers (bitwise equal to the reference's
// deterministic mode).
inline void assemble(Context& c, const BlockTripletStream& s, Index n_block_rows, SortedSymBlockCoo& hess,
                     bool copy_back = true) {
    int64_t U = 0;
    std::vector<double> in, out;
    check(adipc_gpu_assemble(c.get(), s.keys.data(), flat_in<9>(s.values, in), static_cast<int64_t>(s.size()),
                             n_block_rows, 1, &U),
          c.get());
    hess.n_block_rows = n_block_rows;
    if (!copy_back) return;
    hess.rows.resize(U);
    hess.cols.resize(U);
    hess.blocks.resize(U);
    check(adipc_gpu_copy_matrix(c.get(), reinterpret_cast<uint32_t*>(hess.rows.data()),
                                reinterpret_cast<uint32_t*>(hess.cols.data()), flat_out<9>(hess.blocks, out)),
          c.get());
    flat_back<9>(hess.blocks, out);
}

// block_coo.hpp:106 (stable, in place)
inline void sort_stream(Context& c, BlockTripletStream& s) {
    std::vector<double> tmp;
    double* v = flat_out<9>(s.values, tmp);
    if constexpr (sizeof(s.values[0]) != 9 * sizeof(double))
        for (std::size_t i = 0; i < s.values.size(); ++i) std::memcpy(v + 9 * i, s.values[i].data(), 9 * sizeof(double));
    check(adipc_gpu_sort_stream(c.get(), s.keys.data(), v, static_cast<int64_t>(s.size())), c.get());
    flat_back<9>(s.values, tmp);
}

// abd_reduce.hpp:32 — same DofMap, same tile order
inline BlockTripletStream two_level_abd_reduce(Context& c, const BlockTripletStream& node_pairs, const DofMap& map) {
    BlockTripletStream out;
    const int64_t cap = 16 * static_cast<int64_t>(node_pairs.size());
    out.keys.resize(cap);
    out.values.resize(cap);
    int64_t n = 0;
    std::vector<double> vin, jin, vout;
    check(adipc_gpu_two_level_abd_reduce(
              c.get(), node_pairs.keys.data(), flat_in<9>(node_pairs.values, vin),
              static_cast<int64_t>(node_pairs.size()), map.n_fem_nodes, map.n_bodies,
              static_cast<int32_t>(map.abd_node_body.size()), map.abd_node_body.data(),
              flat_in<36>(map.abd_node_jacobian, jin), out.keys.data(), flat_out<9>(out.values, vout), cap, &n),
          c.get());
    flat_back<9>(out.values, vout);
    out.keys.resize(n);
    out.values.resize(n);
    return out;
}

// MasPreconditioner / BlockJacobiPreconditioner as the plugin (mas.hpp:12-15):
// apply() runs on the device matrix of the context.
class GpuPreconditioner : public Preconditioner {
public:
    explicit GpuPreconditioner(Context& c) : c_(c) {}
    // TimeStepper ctor, newton.hpp:66-68
    void set_level0(const Partition& l0, int max_levels) {
        check(adipc_gpu_set_level0_partition(c_.get(), l0.part_of.data(), static_cast<int32_t>(l0.part_of.size()),
                                             l0.n_parts, l0.capacity, max_levels),
              c_.get());
    }
    // build_preconditioner, newton.hpp:243-255 (MAS: block_edges +
    // build_hierarchy + MasPreconditioner::build on the device matrix)
    void build_mas() { check(adipc_gpu_build_preconditioner(c_.get(), ADIPC_PRECOND_MAS), c_.get()); }
    void build_jacobi() { check(adipc_gpu_build_preconditioner(c_.get(), ADIPC_PRECOND_JACOBI), c_.get()); }
    void apply(const VecX& r, VecX& z) const override {
        z.resize(r.size());
        check(adipc_gpu_precond_apply(c_.get(), r.data(), z.data()), c_.get());
    }
    Context& context() const { return c_; }

private:
    Context& c_;
};

// pcg.hpp:34 — same arguments and PcgResult; A must be the context's matrix.
inline PcgResult pcg_solve(GpuPreconditioner& M, const VecX& b, Real rel_tol, int restart, int max_iters, VecX& x) {
    PcgResult out;
    x.resize(b.size());
    int iters = 0, conv = 0;
    double rel = 0;
    check(adipc_gpu_pcg(M.context().get(), b.data(), rel_tol, restart, max_iters, x.data(), &iters, &rel, &conv),
          M.context().get());
    out.iters = iters;
    out.rel_residual = rel;
    out.converged = conv != 0;
    return out;
}

// pcg.hpp:34 with the reference's own signature, so the newton.hpp:129-131
// call site only gains the namespace: `gpu::pcg_solve(hess_, rhs,
// gpu_precond_, cfg.pcg_rel_tol, cfg.pcg_restart, cfg.max_pcg, pol_, dir_)`.
// M must be a GpuPreconditioner (std::invalid_argument otherwise: there is
// no host PCG behind this call) and A the matrix assembled into its context
// (same block rows and stored blocks; checked). The device path ignores the
// ExecPolicy except through ADIPC_OPT_DETERMINISTIC on the context.
inline PcgResult pcg_solve(const SortedSymBlockCoo& A, const VecX& b, const Preconditioner& M, Real rel_tol,
                           int restart, int max_iters, const ExecPolicy& /*pol*/, VecX& x) {
    const auto* g = dynamic_cast<const GpuPreconditioner*>(&M);
    if (!g) throw std::invalid_argument("gpu::pcg_solve: the preconditioner is not a GpuPreconditioner");
    int32_t n = 0;
    int64_t U = 0;
    check(adipc_gpu_matrix_info(g->context().get(), &n, &U), g->context().get());
    if (n != A.n_block_rows || (!A.rows.empty() && static_cast<int64_t>(A.rows.size()) != U))
        throw std::invalid_argument("gpu::pcg_solve: A is not the matrix assembled on the device");
    return pcg_solve(const_cast<GpuPreconditioner&>(*g), b, rel_tol, restart, max_iters, x);
}

}  // namespace adipc::gpu
