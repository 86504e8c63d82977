// Fused PCG (replaces pcg_solve, solver/pcg.hpp:34-88) over the device
// matrix and preconditioner of a context. One iteration is 2 + L launches,
// each of which is also a grid-wide dependency point of the algorithm:
//   1. SRBK SpMV  Ap = A p  with p.Ap fused (last CTA finishes the dot)
//   2. update pass (one warp per level-0 subdomain): alpha = rho / p.Ap,
//      x += alpha p, r -= alpha Ap, restriction of r to level 1
//   3. level-0 dense solves || coarse chain (levels 1..L-1, each solving and
//      restricting to the next) on a high-priority side stream
//   4. prolongation z = z0 + sum_l P_l y_l, rho' = r.z, convergence test,
//      p = z + (rho'/rho) p, Ap cleared for the next SpMV, iteration index
//      advanced on the device.
// Scalars (alpha, beta, dots, stop test, iteration index) never leave the
// device, so an iteration's launch sequence is identical every time: it is
// captured once per solve as a CUDA graph (plus a restart variant) and
// replayed. The host polls the done flag asynchronously, one chunk behind the
// chunk it is enqueuing, so the GPU never drains between chunks; every kernel
// returns immediately once the done flag is set, so over-issued iterations
// are near-free. Termination semantics follow pcg.hpp exactly: x0 = 0, zero
// rhs -> 0 iterations, !(rho0 > 0) -> not converged, !(pAp > 0) ->
// iters = k-1, residual recomputed as b - A x every `restart` iterations, stop
// when r.z <= tol^2 r0.z0.
#include <algorithm>
#include <cmath>

#include "mas_kernels.cuh"

namespace adipc_gpu {

int level_grid(const Ctx& c, int l);
int slot_grid(const Ctx& c);
int jacobi_grid(const Ctx& c);
template <int kMode, bool kSolve>
void launch_level(Ctx& c, int l, const double* r_in, double* z, const PcgArgs& a, double* partials, unsigned* ticket,
                  double* dot_out, cudaStream_t st, bool restrict_next);
template <int kFinal>
void launch_final(Ctx& c, double* z, double* p, double* ap, const PcgArgs& a);
template <int kMode>
void launch_jacobi(Ctx& c, const double* r_in, double* z, const PcgArgs& a, double* partials, unsigned* ticket,
                   double* dot_out);
// solve_order.cu
bool so_supported(const Ctx& c);
int so_partials(const Ctx& c);
template <int kMode>
void launch_update_so(Ctx& c, const PcgArgs& a);
void launch_precond_so(Ctx& c, const double* r, double* z, const int* flags, double* partials, unsigned* ticket,
                       double* dot);
template <int kFinal>
void launch_final_so(Ctx& c, double* z, double* p, double* ap, const PcgArgs& a);
void clear_restrict_so(Ctx& c);

namespace {

__global__ void k_dot_self(const double* __restrict__ v, std::int64_t n, double* partials, unsigned* ticket,
                           double* out) {
    double s = 0;
    for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<std::int64_t>(gridDim.x) * blockDim.x)
        s += v[i] * v[i];
    grid_sum_last_block(s, partials, ticket, out);
}

// x += alpha p ahead of a restart SpMV (pcg.hpp:67-71)
__global__ void k_x_update(std::int64_t n3, PcgArgs a) {
    if (a.flags[F_DONE]) return;
    double alpha;
    if (!pcg_alpha(a, alpha)) return;
    for (std::int64_t g = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; g < n3;
         g += static_cast<std::int64_t>(gridDim.x) * blockDim.x)
        a.x[g] += alpha * a.p[g];
}

__global__ void k_zero(double* __restrict__ v, std::int64_t n, const int* __restrict__ flags) {
    if (flags && flags[F_DONE]) return;
    for (std::int64_t g = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; g < n;
         g += static_cast<std::int64_t>(gridDim.x) * blockDim.x)
        v[g] = 0;
}

struct GraphExec {
    cudaGraphExec_t exec = nullptr;
    long long kernels = 0;
    ~GraphExec() {
        if (exec) cudaGraphExecDestroy(exec);
    }
};

}  // namespace

static PcgOut pcg_impl(Ctx& c, const double* d_b, double rel_tol, int restart, int max_iters, double* d_x) {
    PcgOut out;
    cudaStream_t st = c.stream;
    const std::int32_t n = c.A.n;
    const std::int64_t n3 = 3 * static_cast<std::int64_t>(n);
    if (c.pkind == kNone) throw StatusError(kInvalidArgument, "no preconditioner built");
    const bool mas = c.pkind == kMas;
    const int n_levels = mas ? static_cast<int>(c.levels.size()) : 0;
    PcgWork& w = c.w;
    w.r.reserve(n3);
    w.p.reserve(n3);
    w.ap.reserve(n3);
    w.z.reserve(n3);
    w.tmp.reserve(n3);
    int pmax = std::max({spmv_grid(c, c.S()), slot_grid(c), kSMs * 8, jacobi_grid(c)});
    for (int l = 0; l < n_levels; ++l) pmax = std::max(pmax, level_grid(c, l));
    // solve-order iteration kernels (solve_order.cu)
    const bool so = c.so_kernels && so_supported(c);
    if (so) pmax = std::max(pmax, so_partials(c));
    prepare_spmv(c, c.S());  // deterministic mode: column index, before any graph capture
    w.partials.reserve(static_cast<std::size_t>(pmax) * T_COUNT);
    w.tickets.reserve(T_COUNT);
    w.scal.reserve(S_COUNT);
    w.flags.reserve(F_COUNT);
    if (!c.h_flags) ADIPC_CUDA(cudaMallocHost(&c.h_flags, 2 * F_COUNT * sizeof(int)));
    double* part = w.partials.p;
    auto partials_of = [&](int t) { return part + static_cast<std::size_t>(t) * pmax; };
    ADIPC_CUDA(cudaMemsetAsync(w.tickets.p, 0, sizeof(unsigned) * T_COUNT, st));
    int h_flags0[F_COUNT] = {0};
    h_flags0[F_K] = 0;  // advanced to 1 by the first iteration's SpMV
    ADIPC_CUDA(cudaMemcpyAsync(w.flags.p, h_flags0, sizeof(h_flags0), cudaMemcpyHostToDevice, st));
    double h_scal[S_COUNT] = {0};
    h_scal[S_STOP] = rel_tol * rel_tol;
    ADIPC_CUDA(cudaMemcpyAsync(w.scal.p, h_scal, sizeof(h_scal), cudaMemcpyHostToDevice, st));

    cudaEvent_t e0, e1;
    ADIPC_CUDA(cudaEventCreate(&e0));
    ADIPC_CUDA(cudaEventCreate(&e1));
    ADIPC_CUDA(cudaEventRecord(e0, st));

    // zero right hand side -> converged in 0 iterations, x = 0 (pcg.hpp:38-42)
    k_dot_self<<<grid_for(n3, 256, 8), 256, 0, st>>>(d_b, n3, partials_of(T_BB), w.tickets.p + T_BB, w.scal.p + S_BB);
    ADIPC_LAUNCH_CHECK();
    double bb = 0;
    ADIPC_CUDA(cudaMemcpyAsync(&bb, w.scal.p + S_BB, sizeof(double), cudaMemcpyDeviceToHost, st));
    ADIPC_CUDA(cudaStreamSynchronize(st));
    if (bb == 0) {
        ADIPC_CUDA(cudaMemsetAsync(d_x, 0, sizeof(double) * n3, st));
        ADIPC_CUDA(cudaStreamSynchronize(st));
        out.converged = 1;
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        c.ms_pcg = 0;
        c.last_iters = 0;
        return out;
    }

    PcgArgs a{};
    a.x = d_x;
    a.r = w.r.p;
    a.p = w.p.p;
    a.ap = w.ap.p;
    a.b = d_b;
    a.scal = w.scal.p;
    a.flags = w.flags.p;
    // MAS preconditioner application inside the iteration: after the update
    // pass (x, r and the level-1 restriction), the level-0 solve runs on the
    // solve stream while the latency-bound coarse chain (levels 1..L-1, each
    // restricting to the next) runs concurrently on a high-priority side
    // stream; the prolongation/p-update kernel joins both.
    if (mas && !c.side) {
        int lo = 0, hi = 0;
        ADIPC_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        ADIPC_CUDA(cudaStreamCreateWithPriority(&c.side, cudaStreamNonBlocking, hi));
        ADIPC_CUDA(cudaEventCreateWithFlags(&c.ev_fork, cudaEventDisableTiming));
        ADIPC_CUDA(cudaEventCreateWithFlags(&c.ev_join, cudaEventDisableTiming));
    }
    auto mas_apply = [&](const PcgArgs& aa) {
        ADIPC_CUDA(cudaEventRecord(c.ev_fork, st));
        ADIPC_CUDA(cudaStreamWaitEvent(c.side, c.ev_fork, 0));
        for (int l = 1; l < n_levels; ++l)
            launch_level<M_COARSE, true>(c, l, nullptr, nullptr, aa, partials_of(T_LEVEL + l),
                                         w.tickets.p + T_LEVEL + l, w.scal.p + S_RZ + l, c.side, true);
        launch_level<M_APPLY, true>(c, 0, w.r.p, w.z.p, aa, partials_of(T_LEVEL), w.tickets.p + T_LEVEL,
                                    w.scal.p + S_RZ, st, false);
        ADIPC_CUDA(cudaEventRecord(c.ev_join, c.side));
        ADIPC_CUDA(cudaStreamWaitEvent(st, c.ev_join, 0));
    };
    // r = b, z = M r, p = z, rho0 = r.z (pcg.hpp:51-57)
    if (mas) {
        launch_level<M_INIT, false>(c, 0, nullptr, nullptr, a, nullptr, nullptr, nullptr, st, true);
        mas_apply(a);
    } else {
        launch_jacobi<M_INIT>(c, nullptr, w.z.p, a, partials_of(T_LEVEL), w.tickets.p + T_LEVEL, w.scal.p + S_RZ);
    }
    launch_final<F_PCG_INIT>(c, w.z.p, w.p.p, w.ap.p, a);
    if (so) clear_restrict_so(c);

    // optional per-kernel-class timing (ADIPC_OPT_PROFILE): events bracket the
    // SpMV, update, preconditioner and prolongation/p-update launches of every
    // iteration; iterations are then launched directly instead of as graphs.
    const bool prof = c.profile;
    const int chunk = 16;
    if (prof) {
        if (c.prof_events.empty()) {
            c.prof_events.resize(static_cast<std::size_t>(chunk) * 5);
            for (auto& e : c.prof_events) ADIPC_CUDA(cudaEventCreate(&e));
        }
        for (int q = 0; q < 4; ++q) c.prof_ms[q] = 0;
        c.prof_iters = 0;
    }
    auto mark = [&](int slot, int q) {
        if (prof) ADIPC_CUDA(cudaEventRecord(c.prof_events[5 * slot + q], st));
    };
    // one iteration's launch sequence (restart variant: x += alpha p, r = b - A x)
    auto iteration = [&](bool is_restart, int slot) {
        mark(slot, 0);
        spmv_launch(c, c.S(), w.p.p, w.ap.p, false, w.flags.p, partials_of(T_SPMV), w.tickets.p + T_SPMV,
                    w.scal.p + S_PAP);
        mark(slot, 1);
        if (is_restart) {
            k_x_update<<<slot_grid(c), 256, 0, st>>>(n3, a);
            ADIPC_LAUNCH_CHECK();
            k_zero<<<slot_grid(c), 256, 0, st>>>(w.tmp.p, n3, w.flags.p);
            ADIPC_LAUNCH_CHECK();
            spmv_launch(c, c.S(), d_x, w.tmp.p, false, w.flags.p, nullptr, nullptr, nullptr);
            PcgArgs ar = a;
            ar.ap = w.tmp.p;
            if (so)
                launch_update_so<M_RESTART>(c, ar);
            else if (mas)
                launch_level<M_RESTART, false>(c, 0, nullptr, nullptr, ar, nullptr, nullptr, nullptr, st, true);
            else
                launch_jacobi<M_RESTART>(c, nullptr, w.z.p, ar, partials_of(T_LEVEL), w.tickets.p + T_LEVEL,
                                         w.scal.p + S_RZ);
        } else {
            if (so)
                launch_update_so<M_UPDATE>(c, a);
            else if (mas)
                launch_level<M_UPDATE, false>(c, 0, nullptr, nullptr, a, nullptr, nullptr, nullptr, st, true);
            else
                launch_jacobi<M_UPDATE>(c, nullptr, w.z.p, a, partials_of(T_LEVEL), w.tickets.p + T_LEVEL,
                                        w.scal.p + S_RZ);
        }
        mark(slot, 2);
        if (so)
            launch_precond_so(c, w.r.p, w.z.p, w.flags.p, partials_of(T_LEVEL), w.tickets.p + T_LEVEL,
                              w.scal.p + S_RZ);
        else if (mas)
            mas_apply(a);
        mark(slot, 3);
        if (so)
            launch_final_so<F_PCG_STEP>(c, w.z.p, w.p.p, w.ap.p, a);
        else
            launch_final<F_PCG_STEP>(c, w.z.p, w.p.p, w.ap.p, a);
        mark(slot, 4);
    };
    // capture the two iteration variants as graphs (non-profiled runs)
    GraphExec g_norm, g_rest;
    if (!prof) {
        auto capture = [&](bool is_restart, GraphExec& g) {
            cudaGraph_t graph;
            // kernels recorded into the graph are counted when the graph is
            // replayed (kernel_launches() reports kernels actually executed)
            CaptureCount& cc = capture_count();
            cc.active = true;
            cc.n = 0;
            ADIPC_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
            try {
                iteration(is_restart, 0);
            } catch (...) {
                cc.active = false;
                cudaStreamEndCapture(st, &graph);
                throw;
            }
            cc.active = false;
            ADIPC_CUDA(cudaStreamEndCapture(st, &graph));
            ADIPC_CUDA(cudaGraphInstantiate(&g.exec, graph, 0));
            ADIPC_CUDA(cudaGraphDestroy(graph));
            g.kernels = cc.n;
        };
        capture(false, g_norm);
        if (restart > 0 && restart <= max_iters) capture(true, g_rest);
    }

    // chunks of iterations; the done flag of chunk i is checked while chunk
    // i+1 is already queued (h_flags double-buffered in pinned memory)
    int* hf[2] = {c.h_flags, c.h_flags + F_COUNT};
    if (!c.ev_chunk[0])
        for (auto& e : c.ev_chunk) ADIPC_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    int k = 1, ci = 0;
    bool done = false;
    while (!done && k <= max_iters) {
        const int kbeg = k, kend = std::min(max_iters, k + chunk - 1);
        for (; k <= kend; ++k) {
            const bool is_restart = restart > 0 && k % restart == 0;
            if (prof)
                iteration(is_restart, k - kbeg);
            else {
                GraphExec& g = is_restart ? g_rest : g_norm;
                ADIPC_CUDA(cudaGraphLaunch(g.exec, st));
                launch_counter() += g.kernels;
            }
        }
        ADIPC_CUDA(cudaMemcpyAsync(hf[ci & 1], w.flags.p, F_COUNT * sizeof(int), cudaMemcpyDeviceToHost, st));
        ADIPC_CUDA(cudaEventRecord(c.ev_chunk[ci & 1], st));
        if (prof) {  // profiling: synchronous per chunk (events are reused)
            ADIPC_CUDA(cudaEventSynchronize(c.ev_chunk[ci & 1]));
            const int* f = hf[ci & 1];
            const int last = f[F_DONE] ? std::min(kend, std::max(f[F_ITERS], kbeg)) : kend;
            for (int kk = kbeg; kk <= last; ++kk) {
                for (int q = 0; q < 4; ++q) {
                    float ms = 0;
                    ADIPC_CUDA(cudaEventElapsedTime(&ms, c.prof_events[5 * (kk - kbeg) + q],
                                                    c.prof_events[5 * (kk - kbeg) + q + 1]));
                    c.prof_ms[q] += ms;
                }
                ++c.prof_iters;
            }
            done = f[F_DONE] != 0;
        } else if (ci > 0) {  // check the previous chunk while this one runs
            ADIPC_CUDA(cudaEventSynchronize(c.ev_chunk[(ci - 1) & 1]));
            done = hf[(ci - 1) & 1][F_DONE] != 0;
        }
        ++ci;
    }
    ADIPC_CUDA(cudaEventRecord(e1, st));
    int h_final[F_COUNT];
    ADIPC_CUDA(cudaMemcpyAsync(h_final, w.flags.p, sizeof(h_final), cudaMemcpyDeviceToHost, st));
    ADIPC_CUDA(cudaMemcpyAsync(h_scal, w.scal.p, sizeof(h_scal), cudaMemcpyDeviceToHost, st));
    ADIPC_CUDA(cudaStreamSynchronize(st));
    ADIPC_CUDA(cudaEventElapsedTime(&c.ms_pcg, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (h_final[F_DONE]) {
        out.iters = h_final[F_ITERS];
        out.converged = h_final[F_CONVERGED];
        out.rel_residual = h_scal[S_REL];
    } else {  // ran out of iterations (pcg.hpp:86-87)
        out.iters = max_iters;
        out.converged = 0;
        const double rho = h_scal[S_RHO0 + (max_iters & 1)];
        out.rel_residual = std::sqrt(std::fabs(rho) / h_scal[S_RHO_INIT]);
    }
    c.last_iters = out.iters;
    return out;
}

// The MAS solve runs in solve order (Ctx::perm): b is permuted in and x out.
PcgOut pcg(Ctx& c, const double* d_b, double rel_tol, int restart, int max_iters, double* d_x) {
    check_solve_matrix(c);
    if (!(c.pkind == kMas && c.perm_active)) return pcg_impl(c, d_b, rel_tol, restart, max_iters, d_x);
    const std::size_t n3 = 3 * static_cast<std::size_t>(c.A.n);
    c.pv_in.reserve(n3);
    c.pv_out.reserve(n3);
    permute_vec(c, d_b, c.pv_in.p, true);
    const PcgOut o = pcg_impl(c, c.pv_in.p, rel_tol, restart, max_iters, c.pv_out.p);
    permute_vec(c, c.pv_out.p, d_x, false);
    return o;
}

}  // namespace adipc_gpu
