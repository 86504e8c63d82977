// TEST INFRASTRUCTURE — the drop-in boundary exercised from C++.
//
// A host program written against the REFERENCE's own headers (compiled in
// place from /root/reference/proj/include with the Eigen subset of
// oracle/eigen_shim, as oracle/_ref) that runs the same linear solve twice:
//   * through the reference's CPU path: sort_stream + fast_hash_reduction
//     (incremental_potential.hpp:256-257), block_edges + build_hierarchy +
//     MasPreconditioner::build (newton.hpp:243-255), pcg_solve
//     (newton.hpp:129-131);
//   * through include/adipc_gpu.hpp — the C++ shim with the reference's
//     signatures over the C ABI — on the B200.
// It prints one JSON line and exits 0 iff the parity contract holds:
// assembled matrix bitwise equal to the reference's deterministic mode, MAS
// apply within 1e-10, PCG iteration counts within +-2 %, solutions within
// 1e-5 relative L2. Built by `make -C oracle shim` into oracle/_ref (needs
// /root/reference); run by tests/test_gpu_shim.py on a GPU box.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>

#include "adipc/precond/hierarchy.hpp"
#include "adipc/precond/mas.hpp"
#include "adipc/precond/partition.hpp"
#include "adipc/solver/pcg.hpp"
#include "adipc/sparse/abd_reduce.hpp"
#include "adipc/sparse/block_coo.hpp"
#include "adipc/sparse/reduction.hpp"
// the shim needs the reference's types in scope
using namespace adipc;
#include "adipc_gpu.hpp"

namespace {

double rel_l2(const VecX& a, const VecX& b) {
    double num = 0, den = 0;
    for (long i = 0; i < a.size(); ++i) {
        num += (a[i] - b[i]) * (a[i] - b[i]);
        den += b[i] * b[i];
    }
    return std::sqrt(num / (den > 0 ? den : 1.0));
}

}  // namespace

int main(int argc, char** argv) {
    const int G = argc > 1 ? std::atoi(argv[1]) : 16;  // G^3 block rows
    const Index n = G * G * G;
    std::mt19937 rng(7);
    std::uniform_real_distribution<double> uw(0.5, 2.0), up(-0.3, 0.3);
    auto id = [G](int i, int j, int k) { return static_cast<Index>((k * G + j) * G + i); };

    // A = sum over grid edges e=(a,b) of w_e (e_a - e_b)(e_a - e_b)^T (x) M_e + 0.05 I,
    // M_e SPD: the edge terms emitted as separate triplets (duplicates on
    // the diagonal exercise the reduction's emission-order sums)
    BlockTripletStream stream;
    std::vector<std::pair<Index, Index>> rest_edges;
    for (Index v = 0; v < n; ++v) stream.emit(v, v, 0.05 * Mat3::Identity());
    for (int k = 0; k < G; ++k)
        for (int j = 0; j < G; ++j)
            for (int i = 0; i < G; ++i) {
                const Index a = id(i, j, k);
                const Index nb[3] = {i + 1 < G ? id(i + 1, j, k) : -1, j + 1 < G ? id(i, j + 1, k) : -1,
                                     k + 1 < G ? id(i, j, k + 1) : -1};
                for (const Index b : nb) {
                    if (b < 0) continue;
                    Mat3 B;
                    for (int r = 0; r < 3; ++r)
                        for (int c = 0; c < 3; ++c) B(r, c) = up(rng);
                    const Mat3 M = (B * B.transpose() + Mat3::Identity()) * uw(rng);
                    stream.emit(a, a, M);
                    stream.emit(b, b, M);
                    stream.emit(b, a, -M);  // canonicalised by emit (transpose when swapped)
                    rest_edges.emplace_back(a, b);
                }
            }
    VecX rhs(3 * n);
    std::normal_distribution<double> nd(0.0, 1.0);
    for (long i = 0; i < rhs.size(); ++i) rhs[i] = nd(rng);

    // ---- reference CPU path ----
    ExecPolicy det;
    det.deterministic = true;
    BlockTripletStream sorted = stream;
    sort_stream(sorted, det);
    const SortedSymBlockCoo A = fast_hash_reduction(sorted, n, det);
    const Partition l0 = partition_block_graph(n, rest_edges, 16);
    const MasHierarchy h = build_hierarchy(l0, block_edges(A), 4);
    MasPreconditioner M;
    M.build(A, h);
    VecX x_cpu;
    const PcgResult r_cpu = pcg_solve(A, rhs, M, 1e-8, 250, 10000, det, x_cpu);
    VecX z_cpu;
    M.apply(rhs, z_cpu);

    // ---- B200 path through the shim ----
    gpu::Context ctx(0);
    SortedSymBlockCoo Ag;
    gpu::assemble(ctx, stream, n, Ag);  // copies the device matrix back for the check
    bool bitwise = Ag.rows == A.rows && Ag.cols == A.cols && Ag.blocks.size() == A.blocks.size();
    for (std::size_t e = 0; bitwise && e < A.blocks.size(); ++e)
        bitwise = std::memcmp(Ag.blocks[e].data(), A.blocks[e].data(), 9 * sizeof(double)) == 0;
    gpu::GpuPreconditioner gm(ctx);
    gm.set_level0(l0, 4);
    gm.build_mas();
    VecX z_gpu;
    gm.apply(rhs, z_gpu);
    VecX x_gpu;
    const PcgResult r_gpu = gpu::pcg_solve(Ag, rhs, gm, 1e-8, 250, 10000, det, x_gpu);  // the reference signature

    const double dz = rel_l2(z_gpu, z_cpu), dx = rel_l2(x_gpu, x_cpu);
    const int di = std::abs(r_gpu.iters - r_cpu.iters);
    const bool ok = bitwise && dz <= 1e-10 && di <= std::max(1.0, 0.02 * r_cpu.iters) && dx <= 1e-5 &&
                    r_gpu.converged && r_cpu.converged;
    std::printf(
        "{\"n_block_rows\": %d, \"blocks\": %zu, \"assembly_bitwise\": %s, \"levels\": %d, \"apply_rel_l2\": %.3e, "
        "\"iters_reference\": %d, \"iters_gpu\": %d, \"x_rel_l2\": %.3e, \"ok\": %s}\n",
        n, A.rows.size(), bitwise ? "true" : "false", h.n_levels(), dz, r_cpu.iters, r_gpu.iters, dx,
        ok ? "true" : "false");
    return ok ? 0 : 1;
}
