// extern "C" entry points of include/adipc_gpu.h. Each wraps the C++
// implementation in a try/catch that maps exceptions to status codes and
// records the message on the context.
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <vector>

#include "../../include/adipc_gpu.h"
#include "context.hpp"

struct adipc_gpu_ctx {
    adipc_gpu::Ctx c;
};
struct adipc_hierarchy {
    adipc_gpu::host::MasHierarchy h;
};

namespace adipc_gpu {
Ctx* unwrap(adipc_gpu_ctx* c) { return &c->c; }
std::atomic<long long>& launch_counter() {
    static std::atomic<long long> n{0};
    return n;
}
CaptureCount& capture_count() {
    thread_local CaptureCount cc;
    return cc;
}
}  // namespace adipc_gpu

using namespace adipc_gpu;

namespace {

thread_local std::string g_global_err;

template <class F>
int guarded(adipc_gpu_ctx* ctx, F&& f) {
    try {
        if (ctx) ADIPC_CUDA(cudaSetDevice(ctx->c.device));
        f();
        return ADIPC_OK;
    } catch (const StatusError& e) {
        (ctx ? ctx->c.err : g_global_err) = e.what();
        return e.code;
    } catch (const CudaError& e) {
        (ctx ? ctx->c.err : g_global_err) = e.what();
        return ADIPC_CUDA_ERROR;
    } catch (const std::bad_alloc& e) {
        (ctx ? ctx->c.err : g_global_err) = "host allocation failed";
        return ADIPC_CUDA_ERROR;
    } catch (const std::exception& e) {
        (ctx ? ctx->c.err : g_global_err) = e.what();
        return ADIPC_INVALID_ARGUMENT;
    }
}

template <class T>
void h2d(DBuf<T>& d, const T* h, std::size_t n, cudaStream_t st) {
    d.reserve(n);
    if (n) ADIPC_CUDA(cudaMemcpyAsync(d.p, h, n * sizeof(T), cudaMemcpyHostToDevice, st));
}

void sync(Ctx& c) { ADIPC_CUDA(cudaStreamSynchronize(c.stream)); }

}  // namespace

namespace {
// Host-pointer entry points: the keys (and pins) go first on the solve stream;
// the values (9/10 of the bytes) follow on a copy stream and the key filter
// and sort run on the device meanwhile — only the reduction waits for them.
// (From pageable host memory the copies are staged synchronously: still
// correct, without the overlap.)
static cudaEvent_t upload_values(Ctx& c, const double* vals9, std::int64_t T) {
    c.vals.reserve(9 * static_cast<std::size_t>(T));
    if (!c.copy_stream) {
        ADIPC_CUDA(cudaStreamCreateWithFlags(&c.copy_stream, cudaStreamNonBlocking));
        ADIPC_CUDA(cudaEventCreateWithFlags(&c.ev_keys, cudaEventDisableTiming));
        ADIPC_CUDA(cudaEventCreateWithFlags(&c.ev_vals, cudaEventDisableTiming));
    }
    ADIPC_CUDA(cudaEventRecord(c.ev_keys, c.stream));  // after the key upload: keys get the link first
    ADIPC_CUDA(cudaStreamWaitEvent(c.copy_stream, c.ev_keys, 0));
    if (T > 0)
        ADIPC_CUDA(cudaMemcpyAsync(c.vals.p, vals9, sizeof(double) * 9 * static_cast<std::size_t>(T),
                                   cudaMemcpyHostToDevice, c.copy_stream));
    ADIPC_CUDA(cudaEventRecord(c.ev_vals, c.copy_stream));
    return c.ev_vals;
}

template <class F>
static void timed(Ctx& c, F&& work) {
    cudaEvent_t e0, e1;
    ADIPC_CUDA(cudaEventCreate(&e0));
    ADIPC_CUDA(cudaEventCreate(&e1));
    ADIPC_CUDA(cudaEventRecord(e0, c.stream));
    work();
    ADIPC_CUDA(cudaEventRecord(e1, c.stream));
    ADIPC_CUDA(cudaEventSynchronize(e1));
    ADIPC_CUDA(cudaEventElapsedTime(&c.ms_assemble, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
}

}  // namespace

extern "C" {

int adipc_gpu_create(int device, adipc_gpu_ctx** out) {
    if (!out) return ADIPC_INVALID_ARGUMENT;
    *out = nullptr;
    auto* ctx = new adipc_gpu_ctx();
    ctx->c.device = device;
    const int rc = guarded(ctx, [&] {
        int n = 0;
        ADIPC_CUDA(cudaGetDeviceCount(&n));
        if (device < 0 || device >= n) throw StatusError(kInvalidArgument, "no such CUDA device");
        ADIPC_CUDA(cudaSetDevice(device));
        ADIPC_CUDA(cudaStreamCreateWithFlags(&ctx->c.stream, cudaStreamNonBlocking));
        ctx->c.own_stream = true;
    });
    if (rc != ADIPC_OK) {
        g_global_err = ctx->c.err;
        delete ctx;
        return rc;
    }
    *out = ctx;
    return ADIPC_OK;
}

int adipc_gpu_destroy(adipc_gpu_ctx* ctx) {
    if (!ctx) return ADIPC_OK;
    cudaSetDevice(ctx->c.device);
    Ctx& c = ctx->c;
    cudaStreamSynchronize(c.stream);
    c.A.rows.free();
    c.A.cols.free();
    c.A.blocks.free();
    c.A.row_ptr.free();
    c.keys.free();
    c.sorted.free();
    c.merge_scratch.free();
    c.huge_info.free();
    c.huge_work.free();
    c.vals.free();
    c.row_cnt.free();
    c.row_cursor.free();
    c.uniq_cnt.free();
    c.big_rows.free();
    c.row_start.free();
    c.uniq_start.free();
    c.scan_scratch.free();
    c.counters.free();
    c.pinned.free();
    for (DeviceMatrix* m : {&c.abd_l1}) {
        m->rows.free();
        m->cols.free();
        m->blocks.free();
        m->row_ptr.free();
    }
    c.abd_cnt.free();
    c.abd_off.free();
    c.tile_keys.free();
    c.tile_vals.free();
    c.io_keys.free();
    c.io_keys2.free();
    c.io_vals.free();
    c.io_vals2.free();
    c.io_jac.free();
    c.io_body.free();
    c.det_tptr.free();
    c.det_tidx.free();
    c.pin_keep.free();
    c.pin_pos.free();
    c.pin_spos.free();
    c.levels.clear();  // ~DeviceLevel releases the level buffers
    c.jinv.free();
    c.build_status.free();
    c.step_max.free();
    for (auto* b : {&c.l0_part, &c.l0_mem_ptr, &c.l0_members, &c.l0_pos, &c.l1_up, &c.l1_ncomp, &c.l1_cnt, &c.l1_adj})
        b->free();
    c.l1_base.free();
    c.l1_ptr.free();
    c.l1_keys.free();
    for (auto* b : {&c.ag_part, &c.ag_mem_ptr, &c.ag_members, &c.ag_pos, &c.ag_up, &c.ag_ncomp, &c.ag_cnt, &c.ag_adj[0],
                    &c.ag_adj[1]})
        b->free();
    for (auto* b : {&c.ag_base, &c.ag_ptr[0], &c.ag_ptr[1], &c.ag_koff}) b->free();
    c.ag_kcnt.free();
    c.stage.free();
    c.fem_defer_m.free();
    c.fem_defer_t.free();
    c.fem_defer_n.free();
    c.stage_up.free();
    c.graph_deg.free();
    c.graph_adj.free();
    c.graph_ptr.free();
    c.fem_keys.free();
    c.hinge_work.free();
    for (auto* b : {&c.seg_cnt, &c.seg_row, &c.seg_heads}) b->free();
    for (auto* b : {&c.seg_ptr, &c.seg_bounds, &c.seg_u}) b->free();
    c.ct_on.free();
    c.ct_rank.free();
    c.ct_work.free();
    c.ct_scal.free();
    c.bp = BroadState();
    c.fem_vals.free();
    c.fem_value.free();
    c.perm.free();
    c.perm_keys.free();
    c.as_src.free();
    c.perm_vals.free();
    c.pv_in.free();
    c.pv_out.free();
    c.As.rows.free();
    c.As.cols.free();
    c.As.blocks.free();
    c.As.row_ptr.free();
    for (auto* b : {&c.w.x, &c.w.r, &c.w.p, &c.w.ap, &c.w.z, &c.w.b, &c.w.tmp, &c.w.partials, &c.w.scal}) b->free();
    c.w.tickets.free();
    c.w.flags.free();
    for (auto e : c.prof_events) cudaEventDestroy(e);
    if (c.side) cudaStreamDestroy(c.side);
    if (c.copy_stream) cudaStreamDestroy(c.copy_stream);
    if (c.ev_keys) cudaEventDestroy(c.ev_keys);
    if (c.ev_vals) cudaEventDestroy(c.ev_vals);
    if (c.h_flags) cudaFreeHost(c.h_flags);
    for (auto e : c.ev_chunk)
        if (e) cudaEventDestroy(e);
    if (c.ev_fork) cudaEventDestroy(c.ev_fork);
    if (c.ev_join) cudaEventDestroy(c.ev_join);
    if (c.own_stream && c.stream) cudaStreamDestroy(c.stream);
    delete ctx;
    return ADIPC_OK;
}

const char* adipc_gpu_last_error(const adipc_gpu_ctx* ctx) { return ctx ? ctx->c.err.c_str() : g_global_err.c_str(); }

int adipc_gpu_set_stream(adipc_gpu_ctx* ctx, void* stream) {
    return guarded(ctx, [&] {
        Ctx& c = ctx->c;
        ADIPC_CUDA(cudaStreamSynchronize(c.stream));
        if (stream) {
            if (c.own_stream && c.stream) ADIPC_CUDA(cudaStreamDestroy(c.stream));
            c.stream = static_cast<cudaStream_t>(stream);
            c.own_stream = false;
        } else if (!c.own_stream) {
            ADIPC_CUDA(cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking));
            c.own_stream = true;
        }
    });
}

int adipc_gpu_set_option(adipc_gpu_ctx* ctx, int option, int value) {
    return guarded(ctx, [&] {
        if (option == ADIPC_OPT_CACHE_HIERARCHY)
            ctx->c.cache_hierarchy = value != 0;
        else if (option == ADIPC_OPT_PROFILE)
            ctx->c.profile = value != 0;
        else if (option == ADIPC_OPT_PC_PAIRS) {
            if (value < 1 || value > 5) throw StatusError(kInvalidArgument, "pairs per CTA not in 1..5");
            ctx->c.pc_pairs = value;
        } else if (option == ADIPC_OPT_DETERMINISTIC) {
            ctx->c.deterministic = value != 0;
        } else if (option == ADIPC_OPT_SO_KERNELS) {
            ctx->c.so_kernels = value != 0;
        } else if (option == ADIPC_OPT_L0_STAGES) {
            if (value != 2 && value != 3) throw StatusError(kInvalidArgument, "level-0 stages not in {2,3}");
            ctx->c.l0_stages = value;
        } else if (option == ADIPC_OPT_SOLVE_ORDER) {
            ctx->c.solve_order = value != 0;
            ctx->c.hier_version = ~0ull;  // the device levels depend on the numbering
            ctx->c.levels.clear();
            ctx->c.pkind = kNone;
        } else
            throw StatusError(kInvalidArgument, "unknown option");
    });
}

int64_t adipc_gpu_kernel_launches(void) { return launch_counter(); }

int adipc_gpu_pcg_profile(adipc_gpu_ctx* ctx, float* ms4, int* iters) {
    if (!ctx || !ms4) return ADIPC_INVALID_ARGUMENT;
    for (int q = 0; q < 4; ++q) ms4[q] = ctx->c.prof_ms[q];
    if (iters) *iters = ctx->c.prof_iters;
    return ADIPC_OK;
}

int adipc_gpu_last_timings(adipc_gpu_ctx* ctx, float* ms4) {
    if (!ctx || !ms4) return ADIPC_INVALID_ARGUMENT;
    ms4[0] = ctx->c.ms_assemble;
    ms4[1] = ctx->c.ms_build;
    ms4[2] = ctx->c.ms_build_host;
    ms4[3] = ctx->c.ms_pcg;
    return ADIPC_OK;
}

// ---- assembly (helpers: upload_values, timed above the extern block) -----------
int adipc_gpu_assemble(adipc_gpu_ctx* ctx, const uint64_t* keys, const double* vals9, int64_t T, int32_t n,
                       int det, int64_t* n_unique) {
    return guarded(ctx, [&] {
        Ctx& c = ctx->c;
        if (T < 0 || n < 0) throw StatusError(kInvalidArgument, "negative size");
        h2d(c.keys, keys, static_cast<std::size_t>(T), c.stream);
        cudaEvent_t ready = upload_values(c, vals9, T);
        timed(c, [&] { assemble(c, c.keys.p, c.vals.p, T, n, det, ready); });
        if (n_unique) *n_unique = c.A.U;
    });
}

int adipc_gpu_assemble_device(adipc_gpu_ctx* ctx, const uint64_t* d_keys, const double* d_vals9, int64_t T, int32_t n,
                              int det, int64_t* n_unique) {
    return guarded(ctx, [&] {
        Ctx& c = ctx->c;
        if (T < 0 || n < 0) throw StatusError(kInvalidArgument, "negative size");
        timed(c, [&] { assemble(c, d_keys, d_vals9, T, n, det); });
        if (n_unique) *n_unique = c.A.U;
    });
}

// filter_pinned + sort_stream + fast_hash_reduction in one call
// (incremental_potential.hpp:255-257): the raw stream crosses PCIe once and
// the values are never moved on the device (assemble_filtered, assemble.cu).
int adipc_gpu_assemble_filtered(adipc_gpu_ctx* ctx, const uint64_t* keys, const double* vals9, int64_t T,
                                int32_t n, const uint8_t* pinned, int det, int64_t* n_unique) {
    (void)det;  // the device path is always the bitwise-deterministic order
    return guarded(ctx, [&] {
        Ctx& c = ctx->c;
        if (T < 0 || n < 0) throw StatusError(kInvalidArgument, "negative size");
        h2d(c.keys, keys, static_cast<std::size_t>(T), c.stream);
        h2d(c.pinned, pinned, static_cast<std::size_t>(n), c.stream);
        cudaEvent_t ready = upload_values(c, vals9, T);
        timed(c, [&] { assemble_filtered(c, c.keys.p, c.vals.p, T, n, c.pinned.p, ready); });
        if (n_unique) *n_unique = c.A.U;
    });
}

int adipc_gpu_assemble_filtered_device(adipc_gpu_ctx* ctx, const uint64_t* d_keys, const double* d_vals9, int64_t T,
                                       int32_t n, const uint8_t* d_pinned, int det, int64_t* n_unique) {
    (void)det;
    return guarded(ctx, [&] {
        Ctx& c = ctx->c;
        if (T < 0 || n < 0) throw StatusError(kInvalidArgument, "negative size");
        timed(c, [&] { assemble_filtered(c, d_keys, d_vals9, T, n, d_pinned); });
        if (n_unique) *n_unique = c.A.U;
    });
}


// ---- element-Hessian producer (energy.cu) ---------------------
static FemDesc fem_desc(const adipc_fem_desc* d) {
    if (!d) throw StatusError(kInvalidArgument, "null adipc_fem_desc");
    if (d->n_verts < 0 || d->n_meshes < 0) throw StatusError(kInvalidArgument, "negative size");
    if (d->n_verts > 0 && (!d->x || !d->x_tilde || !d->mass)) throw StatusError(kInvalidArgument, "missing x / x_tilde / mass");
    if (d->n_meshes > 0 && (!d->tet_begin || !d->mu || !d->lambda))
        throw StatusError(kInvalidArgument, "missing tet_begin / mu / lambda");
    for (int m = 0; m < d->n_meshes; ++m)
        if (d->tet_begin[m + 1] < d->tet_begin[m] || d->tet_begin[0] != 0)
            throw StatusError(kInvalidArgument, "tet_begin must start at 0 and not decrease");
    if (d->n_meshes > 0 && d->tet_begin[d->n_meshes] > 0 && (!d->tets || !d->rest_inv9 || !d->rest_volume))
        throw StatusError(kInvalidArgument, "missing tets / rest data");
    FemDesc f;
    f.n_verts = d->n_verts;
    f.x = d->x;
    f.x_tilde = d->x_tilde;
    f.mass = d->mass;
    f.n_meshes = d->n_meshes;
    f.tet_begin = d->tet_begin;
    f.mu = d->mu;
    f.lambda = d->lambda;
    f.tets = d->tets;
    f.rest_inv9 = d->rest_inv9;
    f.rest_volume = d->rest_volume;
    f.dt2 = d->dt2;
    f.project = d->project;
    f.pinned = d->pinned;
    if (d->n_bodies < 0) throw StatusError(kInvalidArgument, "negative size");
    if (d->n_bodies > 0 && (!d->q || !d->q_tilde || !d->reduced_mass || !d->body_kappa || !d->body_volume))
        throw StatusError(kInvalidArgument, "missing body arrays");
    f.n_bodies = d->n_bodies;
    f.q = d->q;
    f.q_tilde = d->q_tilde;
    f.reduced_mass = d->reduced_mass;
    f.body_kappa = d->body_kappa;
    f.body_volume = d->body_volume;
    if (d->n_shells < 0 || d->n_kinds < 0) throw StatusError(kInvalidArgument, "negative size");
    if (d->n_shells > 0 && (!d->tri_begin || !d->hinge_begin || !d->shell_material))
        throw StatusError(kInvalidArgument, "missing shell ranges / material");
    if (d->n_shells > 0 && ((d->tri_begin[d->n_shells] > 0 && (!d->tris || !d->tri_rest)) ||
                            (d->hinge_begin[d->n_shells] > 0 && (!d->hinges || !d->hinge_rest))))
        throw StatusError(kInvalidArgument, "missing shell arrays");
    if (d->n_kinds > 0) {
        if (!d->mesh_kind) throw StatusError(kInvalidArgument, "missing mesh_kind");
        int ns = 0, nm = 0;
        for (int i = 0; i < d->n_kinds; ++i) (d->mesh_kind[i] ? ns : nm) += 1;
        if (ns != d->n_shells || nm != d->n_meshes) throw StatusError(kInvalidArgument, "mesh_kind does not match the meshes");
    } else if (d->n_shells > 0) {
        throw StatusError(kInvalidArgument, "shells need the scene's mesh order (mesh_kind)");
    }
    f.n_shells = d->n_shells;
    f.tri_begin = d->tri_begin;
    f.tris = d->tris;
    f.tri_rest = d->tri_rest;
    f.hinge_begin = d->hinge_begin;
    f.hinges = d->hinges;
    f.hinge_rest = d->hinge_rest;
    f.shell_material = d->shell_material;
    f.n_kinds = d->n_kinds;
    f.mesh_kind = d->mesh_kind;
    return f;
}

static std::int64_t fem_stream_len(const adipc_fem_desc* d) {
    return static_cast<std::int64_t>(d->n_verts) + 10 * (d->n_meshes > 0 ? d->tet_begin[d->n_meshes] : 0) +
           20 * static_cast<std::int64_t>(d->n_bodies) + (d->n_shells > 0 ? 6 * d->tri_begin[d->n_shells] +
                                                           10 * d->hinge_begin[d->n_shells] : 0);
}

int adipc_gpu_fem_emit_device(adipc_gpu_ctx* ctx, const adipc_fem_desc* d, uint64_t* d_keys, double* d_vals9,
                              double* d_grad, double* value) {
    return guarded(ctx, [&] {
        Ctx& c = ctx->c;
        const FemDesc f = fem_desc(d);
        c.fem_value.reserve(1);
        fem_emit(c, f, d_keys, d_vals9, d_grad, c.fem_value.p);
        if (value) ADIPC_CUDA(cudaMemcpyAsync(value, c.fem_value.p, sizeof(double), cudaMemcpyDeviceToHost, c.stream));
        sync(c);
    });
}

int adipc_gpu_fem_value_device(adipc_gpu_ctx* ctx, const adipc_fem_desc* d, double* d_grad, double* value) {
    return guarded(ctx, [&] {
        Ctx& c = ctx->c;
        const FemDesc f = fem_desc(d);
        c.fem_value.reserve(1);
        fem_emit(c, f, nullptr, nullptr, d_grad, c.fem_value.p);
        if (value) ADIPC_CUDA(cudaMemcpyAsync(value, c.fem_value.p, sizeof(double), cudaMemcpyDeviceToHost, c.stream));
        sync(c);
    });
}

int adipc_gpu_fem_assemble_device(adipc_gpu_ctx* ctx, const adipc_fem_desc* d, double* d_grad, double* value,
                                  int64_t* n_unique) {
    return guarded(ctx, [&] {
        Ctx& c = ctx->c;
        const FemDesc f = fem_desc(d);
        const std::int64_t T = fem_stream_len(d);
        c.fem_keys.reserve(static_cast<std::size_t>(std::max<std::int64_t>(T, 1)));
        c.fem_vals.reserve(9 * static_cast<std::size_t>(std::max<std::int64_t>(T, 1)));
        c.fem_value.reserve(1);
        timed(c, [&] {
            fem_emit(c, f, c.fem_keys.p, c.fem_vals.p, d_grad, c.fem_value.p);
            assemble_filtered(c, c.fem_keys.p, c.fem_vals.p, T, d->n_verts + 4 * d->n_bodies, d->pinned);
        });
        if (value) ADIPC_CUDA(cudaMemcpyAsync(value, c.fem_value.p, sizeof(double), cudaMemcpyDeviceToHost, c.stream));
        sync(c);
        if (n_unique) *n_unique = c.A.U;
    });
}


// ---- contact producers (contact.cu) ---------------------------
static ContactDesc contact_desc(const adipc_contact_desc* d) {
    if (!d) throw StatusError(kInvalidArgument, "null adipc_contact_desc");
    if (d->n_nodes < 0 || d->n_pt < 0 || d->n_ee < 0 || d->n_surf_verts < 0 || d->n_friction < 0)
        throw StatusError(kInvalidArgument, "negative size");
    if ((d->n_nodes > 0 && !d->pos) || (d->n_pt > 0 && !d->pt) || (d->n_ee > 0 && !d->ee) ||
        (d->ground && d->n_surf_verts > 0 && !d->surf_verts))
        throw StatusError(kInvalidArgument, "missing contact arrays");
    if (d->n_friction > 0 && (!d->fr_nodes || !d->fr_n_nodes || !d->fr_coeff || !d->fr_t1 || !d->fr_t2 ||
                              !d->fr_lambda || !d->fr_base))
        throw StatusError(kInvalidArgument, "missing friction arrays");
    if (!(d->dhat > 0)) throw StatusError(kInvalidArgument, "dhat must be positive");
    ContactDesc c;
    c.n_nodes = d->n_nodes;
    c.pos = d->pos;
    c.n_pt = d->n_pt;
    c.n_ee = d->n_ee;
    c.pt = d->pt;
    c.ee = d->ee;
    c.dhat = d->dhat;
    c.kappa = d->kappa;
    c.ground = d->ground;
    for (int k = 0; k < 3; ++k) c.ground_normal[k] = d->ground_normal[k];
    c.ground_height = d->ground_height;
    c.n_surf_verts = d->n_surf_verts;
    c.surf_verts = d->surf_verts;
    c.n_friction = d->n_friction;
    c.fr_nodes = d->fr_nodes;
    c.fr_n_nodes = d->fr_n_nodes;
    c.fr_coeff = d->fr_coeff;
    c.fr_t1 = d->fr_t1;
    c.fr_t2 = d->fr_t2;
    c.fr_lambda = d->fr_lambda;
    c.fr_base = d->fr_base;
    c.mu = d->mu;
    c.fr_eps = d->fr_eps;
    return c;
}

int adipc_gpu_contact_emit_device(adipc_gpu_ctx* ctx, const adipc_contact_desc* d, double dt2, int project,
                                  uint64_t* d_node_keys, double* d_node_vals9, int64_t capacity, double* d_node_grad,
                                  double* value, int64_t* n_out) {
    return guarded(ctx, [&] {
        Ctx& c = ctx->c;
        const ContactDesc cd = contact_desc(d);
        c.ct_scal.reserve(2);
        const std::int64_t T = contact_emit(c, cd, dt2, project, d_node_keys, d_node_vals9, capacity, d_node_grad,
                                            c.ct_scal.p);
        if (value) ADIPC_CUDA(cudaMemcpyAsync(value, c.ct_scal.p, sizeof(double), cudaMemcpyDeviceToHost, c.stream));
        sync(c);
        if (n_out) *n_out = T;
    });
}

int adipc_gpu_contact_value_device(adipc_gpu_ctx* ctx, const adipc_contact_desc* d, double dt2, double* value) {
    return guarded(ctx, [&] {
        const double v = contact_value(ctx->c, contact_desc(d), dt2);
        if (value) *value = v;
    });
}

int adipc_gpu_friction_constraints_device(adipc_gpu_ctx* ctx, const adipc_contact_desc* d, int64_t capacity,
                                          int32_t* d_nodes4, int32_t* d_n_nodes, double* d_coeff4, double* d_t1,
                                          double* d_t2, double* d_lambda, int64_t* n_out) {
    return guarded(ctx, [&] {
        if (capacity < 0) throw StatusError(kInvalidArgument, "negative capacity");
        if (capacity > 0 && (!d_nodes4 || !d_n_nodes || !d_coeff4 || !d_t1 || !d_t2 || !d_lambda))
            throw StatusError(kInvalidArgument, "missing output arrays");
        const std::int64_t k = friction_constraints(ctx->c, contact_desc(d), capacity, d_nodes4, d_n_nodes, d_coeff4,
                                                    d_t1, d_t2, d_lambda);
        if (n_out) *n_out = k;
    });
}

int adipc_gpu_ccd_step_device(adipc_gpu_ctx* ctx, const adipc_contact_desc* d, const double* d_disp, double* alpha) {
    return guarded(ctx, [&] {
        if (!d_disp) throw StatusError(kInvalidArgument, "missing displacement");
        const double a = ccd_step(ctx->c, contact_desc(d), d_disp);
        if (alpha) *alpha = a;
    });
}


// ---- broad phase (broad.cu) ----------------------------------------------------
int adipc_gpu_broad_phase_device(adipc_gpu_ctx* ctx, int32_t n_nodes, const double* d_pos, const double* d_disp,
                                 int32_t n_verts, const int32_t* d_verts, int32_t n_edges, const int32_t* d_edges,
                                 int32_t n_tris, const int32_t* d_tris, double inflate, int64_t* n_pt, int64_t* n_ee) {
    return guarded(ctx, [&] {
        if (n_nodes < 0 || n_verts < 0 || n_edges < 0 || n_tris < 0) throw StatusError(kInvalidArgument, "negative size");
        if ((n_nodes > 0 && !d_pos) || (n_verts > 0 && !d_verts) || (n_edges > 0 && !d_edges) || (n_tris > 0 && !d_tris))
            throw StatusError(kInvalidArgument, "missing surface arrays");
        if (!(inflate >= 0)) throw StatusError(kInvalidArgument, "inflate must be non-negative");
        BroadDesc d;
        d.n_nodes = n_nodes;
        d.pos = d_pos;
        d.disp = d_disp;
        d.n_verts = n_verts;
        d.n_edges = n_edges;
        d.n_tris = n_tris;
        d.verts = d_verts;
        d.edges = d_edges;
        d.tris = d_tris;
        d.inflate = inflate;
        std::int64_t a = 0, b = 0;
        broad_phase(ctx->c, d, &a, &b);
        if (n_pt) *n_pt = a;
        if (n_ee) *n_ee = b;
    });
}

int adipc_gpu_broad_phase_copy(adipc_gpu_ctx* ctx, int32_t* pt_pairs, int32_t* pt_stencils, int32_t* ee_pairs,
                               int32_t* ee_stencils) {
    return guarded(ctx, [&] {
        Ctx& c = ctx->c;
        const BroadState& B = c.bp;
        auto cp = [&](int32_t* dst, const int* src, std::int64_t n) {
            if (dst && n > 0) ADIPC_CUDA(cudaMemcpyAsync(dst, src, sizeof(int32_t) * n, cudaMemcpyDefault, c.stream));
        };
        cp(pt_pairs, B.pt_pairs.p, 2 * B.n_pt);
        cp(pt_stencils, B.pt_stencils.p, 4 * B.n_pt);
        cp(ee_pairs, B.ee_pairs.p, 2 * B.n_ee);
        cp(ee_stencils, B.ee_stencils.p, 4 * B.n_ee);
        sync(c);
    });
}

int adipc_gpu_matrix_info(adipc_gpu_ctx* ctx, int32_t* n, int64_t* U) {
    return guarded(ctx, [&] {
        if (n) *n = ctx->c.A.n;
        if (U) *U = ctx->c.A.U;
    });
}

int adipc_gpu_copy_matrix(adipc_gpu_ctx* ctx, uint32_t* rows, uint32_t* cols, double* blocks9) {
    return guarded(ctx, [&] {
        Ctx& c = ctx->c;
        const std::int64_t U = c.A.U;
        if (U == 0) return;
        if (rows) ADIPC_CUDA(cudaMemcpyAsync(rows, c.A.rows.p, 4 * U, cudaMemcpyDeviceToHost, c.stream));
        if (cols) ADIPC_CUDA(cudaMemcpyAsync(cols, c.A.cols.p, 4 * U, cudaMemcpyDeviceToHost, c.stream));
        if (blocks9) {
            c.vals.reserve(9 * U);
            blocks_soa_to_aos(c, c.A.blocks.p, c.vals.p, U);
            ADIPC_CUDA(cudaMemcpyAsync(blocks9, c.vals.p, 72 * U, cudaMemcpyDeviceToHost, c.stream));
        }
        sync(c);
    });
}

// Binary capture of the context's matrix (SPEC.md "External Interfaces":
// binary or text triplet file for offline oracle checks): little-endian
// "ADIPCMAT" magic, u32 version 1, i32 n_block_rows, i64 U, then rows u32[U],
// cols u32[U], blocks f64[U][9] (column-major 3x3, the reference's Mat3).
int adipc_gpu_dump_matrix_binary(adipc_gpu_ctx* ctx, const char* path) {
    return guarded(ctx, [&] {
        Ctx& c = ctx->c;
        if (!path) throw StatusError(kInvalidArgument, "dump_matrix_binary: null path");
        const std::int64_t U = c.A.U;
        std::vector<std::uint32_t> rows(static_cast<std::size_t>(U)), cols(static_cast<std::size_t>(U));
        std::vector<double> b(9 * static_cast<std::size_t>(U));
        if (U > 0) {
            ADIPC_CUDA(cudaMemcpyAsync(rows.data(), c.A.rows.p, 4 * U, cudaMemcpyDeviceToHost, c.stream));
            ADIPC_CUDA(cudaMemcpyAsync(cols.data(), c.A.cols.p, 4 * U, cudaMemcpyDeviceToHost, c.stream));
            c.vals.reserve(9 * U);
            blocks_soa_to_aos(c, c.A.blocks.p, c.vals.p, U);
            ADIPC_CUDA(cudaMemcpyAsync(b.data(), c.vals.p, 72 * U, cudaMemcpyDeviceToHost, c.stream));
            sync(c);
        }
        std::ofstream os(path, std::ios::binary);
        if (!os) throw StatusError(kInvalidArgument, std::string("dump_matrix_binary: cannot open ") + path);
        const std::uint32_t version = 1;
        const std::int32_t n = c.A.n;
        os.write("ADIPCMAT", 8);
        os.write(reinterpret_cast<const char*>(&version), 4);
        os.write(reinterpret_cast<const char*>(&n), 4);
        os.write(reinterpret_cast<const char*>(&U), 8);
        os.write(reinterpret_cast<const char*>(rows.data()), 4 * U);
        os.write(reinterpret_cast<const char*>(cols.data()), 4 * U);
        os.write(reinterpret_cast<const char*>(b.data()), 72 * U);
        if (!os) throw StatusError(kInvalidArgument, std::string("dump_matrix_binary: write failed: ") + path);
    });
}

// ---- the step after the solve (newton.hpp:257-290), device pointers ----------
int adipc_gpu_step_inf_norm_device(adipc_gpu_ctx* ctx, const double* d_dir, int32_t n_fem, int32_t n_bodies,
                                   const double* d_max_xbar, double* out) {
    return guarded(ctx, [&] {
        if (n_fem < 0 || n_bodies < 0 || !out || (n_bodies > 0 && !d_max_xbar))
            throw StatusError(kInvalidArgument, "step_inf_norm: bad arguments");
        *out = step_inf_norm(ctx->c, d_dir, n_fem, n_bodies, d_max_xbar);
    });
}

int adipc_gpu_apply_direction_device(adipc_gpu_ctx* ctx, const double* d_state, const double* d_dir, double alpha,
                                     int64_t n_dofs, double* d_out) {
    return guarded(ctx, [&] {
        if (n_dofs < 0) throw StatusError(kInvalidArgument, "apply_direction: negative size");
        apply_direction(ctx->c, d_state, d_dir, alpha, n_dofs, d_out);
        sync(ctx->c);
    });
}

int adipc_gpu_lift_node_grad_device(adipc_gpu_ctx* ctx, const double* d_node_grad, int32_t n_fem, int32_t n_abd,
                                    const int32_t* d_abd_node_body, const double* d_abd_node_jacobian36,
                                    const uint8_t* d_pinned, double* d_grad) {
    return guarded(ctx, [&] {
        if (n_fem < 0 || n_abd < 0) throw StatusError(kInvalidArgument, "negative size");
        if ((n_fem + n_abd > 0 && (!d_node_grad || !d_grad)) || (n_abd > 0 && (!d_abd_node_body || !d_abd_node_jacobian36)))
            throw StatusError(kInvalidArgument, "missing arrays");
        lift_node_grad(ctx->c, d_node_grad, n_fem, n_abd, d_abd_node_body, d_abd_node_jacobian36, d_pinned, d_grad);
        sync(ctx->c);
    });
}

int adipc_gpu_contact_positions_device(adipc_gpu_ctx* ctx, const double* d_state, int32_t n_fem, int32_t n_abd,
                                       const int32_t* d_abd_node_body, const double* d_abd_node_jacobian36,
                                       double* d_out) {
    return guarded(ctx, [&] {
        if (n_fem < 0 || n_abd < 0) throw StatusError(kInvalidArgument, "contact_positions: negative size");
        if (n_abd > 0 && (!d_abd_node_body || !d_abd_node_jacobian36))
            throw StatusError(kInvalidArgument, "contact_positions: missing body arrays");
        contact_positions(ctx->c, d_state, n_fem, n_abd, d_abd_node_body, d_abd_node_jacobian36, d_out);
        sync(ctx->c);
    });
}

int adipc_gpu_node_displacements_device(adipc_gpu_ctx* ctx, const double* d_dir, int32_t n_fem, int32_t n_abd,
                                        const int32_t* d_abd_node_body, const double* d_abd_jacobian36,
                                        double* d_out) {
    return guarded(ctx, [&] {
        if (n_fem < 0 || n_abd < 0) throw StatusError(kInvalidArgument, "node_displacements: negative size");
        node_displacements(ctx->c, d_dir, n_fem, n_abd, d_abd_node_body, d_abd_jacobian36, d_out);
        sync(ctx->c);
    });
}

// dump_block_coo (srbk_spmv.hpp:52-60) of the context's matrix — the CLI's
// --dump-hessian text: "n U", then per block "row col" and the 9 values
// row-major, default-formatted doubles
int adipc_gpu_dump_block_coo(adipc_gpu_ctx* ctx, const char* path) {
    return guarded(ctx, [&] {
        Ctx& c = ctx->c;
        if (!path) throw StatusError(kInvalidArgument, "dump_block_coo: null path");
        const std::int64_t U = c.A.U;
        std::vector<std::uint32_t> rows(static_cast<std::size_t>(U)), cols(static_cast<std::size_t>(U));
        std::vector<double> b(9 * static_cast<std::size_t>(U));
        if (U > 0) {
            ADIPC_CUDA(cudaMemcpyAsync(rows.data(), c.A.rows.p, 4 * U, cudaMemcpyDeviceToHost, c.stream));
            ADIPC_CUDA(cudaMemcpyAsync(cols.data(), c.A.cols.p, 4 * U, cudaMemcpyDeviceToHost, c.stream));
            c.vals.reserve(9 * U);
            blocks_soa_to_aos(c, c.A.blocks.p, c.vals.p, U);
            ADIPC_CUDA(cudaMemcpyAsync(b.data(), c.vals.p, 72 * U, cudaMemcpyDeviceToHost, c.stream));
            sync(c);
        }
        std::ofstream os(path);
        if (!os) throw StatusError(kInvalidArgument, std::string("dump_block_coo: cannot open ") + path);
        os << c.A.n << " " << U << "\n";
        for (std::int64_t e = 0; e < U; ++e) {
            os << rows[e] << " " << cols[e];
            const double* m = b.data() + 9 * e;  // column-major block
            for (int i = 0; i < 3; ++i)
                for (int k = 0; k < 3; ++k) os << " " << m[3 * k + i];
            os << "\n";
        }
        if (!os) throw StatusError(kInvalidArgument, std::string("dump_block_coo: write failed: ") + path);
    });
}

int adipc_gpu_set_matrix(adipc_gpu_ctx* ctx, int32_t n, int64_t U, const uint32_t* rows, const uint32_t* cols,
                         const double* blocks9) {
    return guarded(ctx, [&] {
        if (n < 0 || U < 0) throw StatusError(kInvalidArgument, "negative size");
        upload_matrix(ctx->c, n, U, rows, cols, blocks9, true);
        sync(ctx->c);
    });
}

int adipc_gpu_set_matrix_device(adipc_gpu_ctx* ctx, int32_t n, int64_t U, const uint32_t* rows, const uint32_t* cols,
                                const double* blocks9) {
    return guarded(ctx, [&] {
        if (n < 0 || U < 0) throw StatusError(kInvalidArgument, "negative size");
        upload_matrix(ctx->c, n, U, rows, cols, blocks9, false);
        sync(ctx->c);
    });
}

int adipc_gpu_sort_stream(adipc_gpu_ctx* ctx, uint64_t* keys, double* vals9, int64_t T) {
    return guarded(ctx, [&] {
        Ctx& c = ctx->c;
        if (T <= 0) return;
        h2d(c.keys, keys, static_cast<std::size_t>(T), c.stream);
        h2d(c.vals, vals9, 9 * static_cast<std::size_t>(T), c.stream);
        DBuf<std::uint64_t> ok;
        DBuf<double> ov;
        ok.reserve(T);
        ov.reserve(9 * T);
        sort_stream(c, c.keys.p, c.vals.p, T, ok.p, ov.p);
        ADIPC_CUDA(cudaMemcpyAsync(keys, ok.p, 8 * T, cudaMemcpyDeviceToHost, c.stream));
        ADIPC_CUDA(cudaMemcpyAsync(vals9, ov.p, 72 * T, cudaMemcpyDeviceToHost, c.stream));
        sync(c);
        ok.free();
        ov.free();
    });
}

int adipc_gpu_segment_reduce(adipc_gpu_ctx* ctx, const int32_t* O, int64_t nO, const double* V, int64_t nV, int width,
                             int32_t n_segments, int /*deterministic*/, double* R) {
    return guarded(ctx, [&] {
        Ctx& c = ctx->c;
        if (nO != nV) throw StatusError(kInvalidArgument, "segment map size mismatch");
        if (n_segments < 0) throw StatusError(kInvalidArgument, "negative segment count");
        DBuf<std::int32_t> dO;
        DBuf<double> dV, dR;
        h2d(dO, O, static_cast<std::size_t>(nO), c.stream);
        h2d(dV, V, static_cast<std::size_t>(nV) * width, c.stream);
        dR.reserve(static_cast<std::size_t>(n_segments) * width);
        segment_reduce(c, dO.p, nO, dV.p, width, n_segments, dR.p);
        if (n_segments)
            ADIPC_CUDA(cudaMemcpyAsync(R, dR.p, sizeof(double) * width * n_segments, cudaMemcpyDeviceToHost, c.stream));
        sync(c);
        dO.free();
        dV.free();
        dR.free();
    });
}

int adipc_gpu_two_level_abd_reduce(adipc_gpu_ctx* ctx, const uint64_t* keys, const double* vals9, int64_t Tn,
                                   int32_t n_fem, int32_t n_bodies, int32_t n_abd, const int32_t* body,
                                   const double* jac36, uint64_t* out_keys, double* out_vals9, int64_t out_cap,
                                   int64_t* n_out) {
    return guarded(ctx, [&] {
        Ctx& c = ctx->c;
        if (Tn < 0 || n_fem < 0 || n_bodies < 0 || n_abd < 0 || out_cap < 0)
            throw StatusError(kInvalidArgument, "negative size");
        h2d(c.io_keys, keys, static_cast<std::size_t>(Tn), c.stream);
        h2d(c.io_vals, vals9, 9 * static_cast<std::size_t>(Tn), c.stream);
        h2d(c.io_body, body, static_cast<std::size_t>(n_abd), c.stream);
        h2d(c.io_jac, jac36, 36 * static_cast<std::size_t>(n_abd), c.stream);
        c.io_keys2.reserve(static_cast<std::size_t>(std::max<std::int64_t>(out_cap, 1)));
        c.io_vals2.reserve(9 * static_cast<std::size_t>(std::max<std::int64_t>(out_cap, 1)));
        const std::int64_t n = two_level_abd_reduce(c, c.io_keys.p, c.io_vals.p, Tn, n_fem, n_bodies, n_abd,
                                                    c.io_body.p, c.io_jac.p, c.io_keys2.p, c.io_vals2.p, out_cap);
        if (n) {
            ADIPC_CUDA(cudaMemcpyAsync(out_keys, c.io_keys2.p, 8 * n, cudaMemcpyDeviceToHost, c.stream));
            ADIPC_CUDA(cudaMemcpyAsync(out_vals9, c.io_vals2.p, 72 * n, cudaMemcpyDeviceToHost, c.stream));
        }
        sync(c);
        if (n_out) *n_out = n;
    });
}

// two_level_abd_reduce + stream_.append + filter_pinned + sort_stream +
// fast_hash_reduction in one call (incremental_potential.hpp:392-394 and
// 253-257): the reduced contact tiles never leave the device.
int adipc_gpu_assemble_contact(adipc_gpu_ctx* ctx, const uint64_t* keys, const double* vals9, int64_t T,
                               const uint64_t* node_keys, const double* node_vals9, int64_t Tn, int32_t n_fem,
                               int32_t n_bodies, int32_t n_abd, const int32_t* body, const double* jac36, int32_t n,
                               const uint8_t* pinned, int64_t* n_unique, int64_t* n_tiles) {
    return guarded(ctx, [&] {
        Ctx& c = ctx->c;
        if (T < 0 || Tn < 0 || n < 0 || n_fem < 0 || n_bodies < 0 || n_abd < 0)
            throw StatusError(kInvalidArgument, "negative size");
        h2d(c.keys, keys, static_cast<std::size_t>(T), c.stream);
        if (pinned) h2d(c.pinned, pinned, static_cast<std::size_t>(n), c.stream);
        h2d(c.io_keys, node_keys, static_cast<std::size_t>(Tn), c.stream);
        h2d(c.io_vals, node_vals9, 9 * static_cast<std::size_t>(Tn), c.stream);
        h2d(c.io_body, body, static_cast<std::size_t>(n_abd), c.stream);
        h2d(c.io_jac, jac36, 36 * static_cast<std::size_t>(n_abd), c.stream);
        cudaEvent_t ready = upload_values(c, vals9, T);
        std::int64_t tiles = 0;
        timed(c, [&] {
            tiles = assemble_contact(c, c.keys.p, c.vals.p, T, c.io_keys.p, c.io_vals.p, Tn, n_fem, n_bodies, n_abd,
                                     c.io_body.p, c.io_jac.p, n, pinned ? c.pinned.p : nullptr, ready);
        });
        if (n_unique) *n_unique = c.A.U;
        if (n_tiles) *n_tiles = tiles;
    });
}

int adipc_gpu_assemble_contact_device(adipc_gpu_ctx* ctx, const uint64_t* d_keys, const double* d_vals9, int64_t T,
                                      const uint64_t* d_node_keys, const double* d_node_vals9, int64_t Tn,
                                      int32_t n_fem, int32_t n_bodies, int32_t n_abd, const int32_t* d_body,
                                      const double* d_jac36, int32_t n, const uint8_t* d_pinned, int64_t* n_unique,
                                      int64_t* n_tiles) {
    return guarded(ctx, [&] {
        Ctx& c = ctx->c;
        if (T < 0 || Tn < 0 || n < 0 || n_fem < 0 || n_bodies < 0 || n_abd < 0)
            throw StatusError(kInvalidArgument, "negative size");
        std::int64_t tiles = 0;
        timed(c, [&] {
            tiles = assemble_contact(c, d_keys, d_vals9, T, d_node_keys, d_node_vals9, Tn, n_fem, n_bodies, n_abd,
                                     d_body, d_jac36, n, d_pinned);
        });
        if (n_unique) *n_unique = c.A.U;
        if (n_tiles) *n_tiles = tiles;
    });
}

int adipc_gpu_filter_pinned(adipc_gpu_ctx* ctx, const uint64_t* keys, const double* vals9, int64_t T,
                            const uint8_t* pinned, int32_t n_slots, uint64_t* out_keys, double* out_vals9,
                            int64_t* n_out) {
    return guarded(ctx, [&] {
        Ctx& c = ctx->c;
        DBuf<std::uint64_t> dk, ok;
        DBuf<double> dv, ov;
        DBuf<std::uint8_t> dp;
        h2d(dk, keys, static_cast<std::size_t>(T), c.stream);
        h2d(dv, vals9, 9 * static_cast<std::size_t>(T), c.stream);
        h2d(dp, pinned, static_cast<std::size_t>(n_slots), c.stream);
        ok.reserve(static_cast<std::size_t>(T + n_slots));
        ov.reserve(9 * static_cast<std::size_t>(T + n_slots));
        const std::int64_t n = filter_pinned(c, dk.p, dv.p, T, dp.p, n_slots, ok.p, ov.p);
        if (n) {
            ADIPC_CUDA(cudaMemcpyAsync(out_keys, ok.p, 8 * n, cudaMemcpyDeviceToHost, c.stream));
            ADIPC_CUDA(cudaMemcpyAsync(out_vals9, ov.p, 72 * n, cudaMemcpyDeviceToHost, c.stream));
        }
        sync(c);
        if (n_out) *n_out = n;
        for (auto* b : {&dk, &ok}) b->free();
        for (auto* b : {&dv, &ov}) b->free();
        dp.free();
    });
}

int adipc_gpu_filter_pinned_device(adipc_gpu_ctx* ctx, const uint64_t* keys, const double* vals9, int64_t T,
                                   const uint8_t* pinned, int32_t n_slots, uint64_t* out_keys, double* out_vals9,
                                   int64_t* n_out) {
    return guarded(ctx, [&] {
        const std::int64_t n = filter_pinned(ctx->c, keys, vals9, T, pinned, n_slots, out_keys, out_vals9);
        if (n_out) *n_out = n;
    });
}

// ---- SpMV ---------------------------------------------------------------------------
int adipc_gpu_spmv(adipc_gpu_ctx* ctx, const double* x, double* y) {
    return guarded(ctx, [&] {
        Ctx& c = ctx->c;
        const std::size_t n3 = 3 * static_cast<std::size_t>(c.A.n);
        h2d(c.io_vals, x, n3, c.stream);
        c.io_vals2.reserve(n3);
        spmv(c, c.io_vals.p, c.io_vals2.p);
        if (n3) ADIPC_CUDA(cudaMemcpyAsync(y, c.io_vals2.p, 8 * n3, cudaMemcpyDeviceToHost, c.stream));
        sync(c);
    });
}

int adipc_gpu_spmv_device(adipc_gpu_ctx* ctx, const double* d_x, double* d_y) {
    return guarded(ctx, [&] {
        spmv(ctx->c, d_x, d_y);
        sync(ctx->c);
    });
}

// ---- partition / hierarchy ---------------------------------------------------------------
int32_t adipc_subdomain_count(int32_t v, int32_t n, int32_t n_o) { return host::subdomain_count(v, n, n_o); }

int32_t adipc_chunk_partition(int32_t v, int32_t capacity, int32_t* part_of) {
    const host::Partition p = host::chunk_partition(v, capacity);
    if (v > 0) std::memcpy(part_of, p.part_of.data(), 4 * static_cast<std::size_t>(v));
    return p.n_parts;
}

int32_t adipc_partition_block_graph(int32_t v, const int32_t* pairs, int64_t n_edges, int32_t capacity,
                                    int32_t* part_of) {
    const host::Partition p = host::partition_block_graph(v, pairs, static_cast<std::size_t>(n_edges), capacity);
    if (v > 0) std::memcpy(part_of, p.part_of.data(), 4 * static_cast<std::size_t>(v));
    return p.n_parts;
}

adipc_hierarchy* adipc_build_hierarchy(const int32_t* part_of, int32_t n_slots, int32_t n_parts, int32_t capacity,
                                       const int32_t* pairs, int64_t n_edges, int32_t max_levels) {
    host::Partition l0;
    l0.part_of.assign(part_of, part_of + n_slots);
    l0.n_parts = n_parts;
    l0.capacity = capacity;
    auto* h = new adipc_hierarchy();
    h->h = host::build_hierarchy(l0, pairs, static_cast<std::size_t>(n_edges), max_levels);
    return h;
}

int adipc_hierarchy_n_levels(const adipc_hierarchy* h) { return h ? h->h.n_levels() : 0; }

static int level_out(const host::MasHierarchy& h, int level, int32_t* n_nodes, int32_t* n_parts, int32_t* part_of,
                     int32_t* agg) {
    if (level < 0 || level >= h.n_levels()) return ADIPC_INVALID_ARGUMENT;
    const host::Level& L = h.levels[level];
    if (n_nodes) *n_nodes = L.n_nodes;
    if (n_parts) *n_parts = L.n_parts;
    if (part_of && L.n_nodes) std::memcpy(part_of, L.part_of.data(), 4 * static_cast<std::size_t>(L.n_nodes));
    if (agg && !L.agg.empty()) std::memcpy(agg, L.agg.data(), 4 * L.agg.size());
    return ADIPC_OK;
}

int adipc_hierarchy_level(const adipc_hierarchy* h, int level, int32_t* n_nodes, int32_t* n_parts, int32_t* part_of,
                          int32_t* agg) {
    if (!h) return ADIPC_INVALID_ARGUMENT;
    return level_out(h->h, level, n_nodes, n_parts, part_of, agg);
}

void adipc_hierarchy_free(adipc_hierarchy* h) { delete h; }

// ---- preconditioner -----------------------------------------------------------------------
int adipc_gpu_set_level0_partition(adipc_gpu_ctx* ctx, const int32_t* part_of, int32_t n_slots, int32_t n_parts,
                                   int32_t capacity, int32_t max_levels) {
    return guarded(ctx, [&] {
        Ctx& c = ctx->c;
        if (n_slots < 0 || n_parts < 0 || capacity <= 0) throw StatusError(kInvalidArgument, "bad partition sizes");
        for (int32_t i = 0; i < n_slots; ++i)
            if (part_of[i] < 0 || part_of[i] >= n_parts) throw StatusError(kInvalidArgument, "part_of out of range");
        c.l0.part_of.assign(part_of, part_of + n_slots);
        c.l0.n_parts = n_parts;
        c.l0.capacity = capacity;
        ++c.l0_version;
        c.max_levels = max_levels;
        c.have_l0 = true;
        c.hier_version = ~0ull;
        c.levels.clear();
        // the levels are gone: a preconditioner must be rebuilt before use
        c.pkind = kNone;
        c.perm_active = false;
    });
}

int adipc_gpu_build_preconditioner(adipc_gpu_ctx* ctx, int kind) {
    return guarded(ctx, [&] {
        Ctx& c = ctx->c;
        if (kind != ADIPC_PRECOND_MAS && kind != ADIPC_PRECOND_JACOBI)
            throw StatusError(kInvalidArgument, "unknown preconditioner kind");
        cudaEvent_t e0, e1;
        ADIPC_CUDA(cudaEventCreate(&e0));
        ADIPC_CUDA(cudaEventCreate(&e1));
        ADIPC_CUDA(cudaEventRecord(e0, c.stream));
        try {
            build_preconditioner(c, kind == ADIPC_PRECOND_MAS ? kMas : kJacobi);
        } catch (...) {
            cudaEventDestroy(e0);
            cudaEventDestroy(e1);
            throw;
        }
        ADIPC_CUDA(cudaEventRecord(e1, c.stream));
        ADIPC_CUDA(cudaEventSynchronize(e1));
        ADIPC_CUDA(cudaEventElapsedTime(&c.ms_build, e0, e1));
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
    });
}

int adipc_gpu_build_mas(adipc_gpu_ctx* ctx, const adipc_hierarchy* h) {
    return guarded(ctx, [&] {
        Ctx& c = ctx->c;
        if (!h) throw StatusError(kInvalidArgument, "null hierarchy");
        if (h->h.n_slots != c.A.n) throw StatusError(kInvalidArgument, "hierarchy slot count differs from n_block_rows");
        cudaEvent_t e0, e1;
        ADIPC_CUDA(cudaEventCreate(&e0));
        ADIPC_CUDA(cudaEventCreate(&e1));
        ADIPC_CUDA(cudaEventRecord(e0, c.stream));
        try {
            build_mas_from_hierarchy(c, h->h);
        } catch (...) {
            cudaEventDestroy(e0);
            cudaEventDestroy(e1);
            throw;
        }
        ADIPC_CUDA(cudaEventRecord(e1, c.stream));
        ADIPC_CUDA(cudaEventSynchronize(e1));
        ADIPC_CUDA(cudaEventElapsedTime(&c.ms_build, e0, e1));
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
    });
}

int adipc_gpu_precond_n_levels(adipc_gpu_ctx* ctx) {
    if (!ctx) return 0;
    return ctx->c.pkind == kMas ? ctx->c.hier.n_levels() : (ctx->c.pkind == kJacobi ? 1 : 0);
}

int adipc_gpu_precond_level(adipc_gpu_ctx* ctx, int level, int32_t* n_nodes, int32_t* n_parts, int32_t* part_of,
                            int32_t* agg) {
    if (!ctx || ctx->c.pkind != kMas) return ADIPC_INVALID_ARGUMENT;
    return level_out(ctx->c.hier, level, n_nodes, n_parts, part_of, agg);
}

int adipc_gpu_precond_subdomain_inverse(adipc_gpu_ctx* ctx, int level, int32_t sub, int32_t* dim, double* out) {
    return guarded(ctx, [&] {
        Ctx& c = ctx->c;
        if (c.pkind != kMas || level < 0 || level >= static_cast<int>(c.levels.size()))
            throw StatusError(kInvalidArgument, "no such level");
        DeviceLevel& L = *c.levels[level];
        if (sub < 0 || sub >= L.n_parts) throw StatusError(kInvalidArgument, "no such subdomain");
        std::int32_t sp[2];
        std::int64_t off = 0;
        ADIPC_CUDA(cudaMemcpyAsync(sp, L.sub_ptr.p + sub, 8, cudaMemcpyDeviceToHost, c.stream));
        ADIPC_CUDA(cudaMemcpyAsync(&off, L.inv_off.p + sub, 8, cudaMemcpyDeviceToHost, c.stream));
        sync(c);
        const int d = 3 * (sp[1] - sp[0]);
        if (dim) *dim = d;
        if (out && d) {  // unpack the symmetric-packed storage to a full column-major matrix
            std::vector<double> pk(static_cast<std::size_t>(packed_doubles(d)));
            ADIPC_CUDA(cudaMemcpyAsync(pk.data(), L.inv.p + off, 8 * pk.size(), cudaMemcpyDeviceToHost, c.stream));
            sync(c);
            for (int k = 0; k < d; ++k)
                for (int j = 0; j < d; ++j) out[static_cast<std::size_t>(k) * d + j] = pk[packed_idx(j, k)];
        }
    });
}

int adipc_gpu_precond_shifts(adipc_gpu_ctx* ctx, int64_t* shifts) {
    if (!ctx || !shifts) return ADIPC_INVALID_ARGUMENT;
    *shifts = ctx->c.shifts_applied;
    return ADIPC_OK;
}

int adipc_gpu_precond_apply(adipc_gpu_ctx* ctx, const double* r, double* z) {
    return guarded(ctx, [&] {
        Ctx& c = ctx->c;
        const std::size_t n3 = 3 * static_cast<std::size_t>(c.A.n);
        h2d(c.io_vals, r, n3, c.stream);
        c.io_vals2.reserve(n3);
        precond_apply(c, c.io_vals.p, c.io_vals2.p);
        if (n3) ADIPC_CUDA(cudaMemcpyAsync(z, c.io_vals2.p, 8 * n3, cudaMemcpyDeviceToHost, c.stream));
        sync(c);
    });
}

int adipc_gpu_precond_apply_device(adipc_gpu_ctx* ctx, const double* d_r, double* d_z) {
    return guarded(ctx, [&] {
        precond_apply(ctx->c, d_r, d_z);
        sync(ctx->c);
    });
}

// ---- PCG --------------------------------------------------------------------------------------
int adipc_gpu_pcg(adipc_gpu_ctx* ctx, const double* b, double rel_tol, int restart, int max_iters, double* x,
                  int* iters, double* rel_residual, int* converged) {
    return guarded(ctx, [&] {
        Ctx& c = ctx->c;
        const std::size_t n3 = 3 * static_cast<std::size_t>(c.A.n);
        h2d(c.w.b, b, n3, c.stream);
        c.w.x.reserve(n3);
        const PcgOut o = pcg(c, c.w.b.p, rel_tol, restart, max_iters, c.w.x.p);
        if (n3) ADIPC_CUDA(cudaMemcpyAsync(x, c.w.x.p, 8 * n3, cudaMemcpyDeviceToHost, c.stream));
        sync(c);
        if (iters) *iters = o.iters;
        if (rel_residual) *rel_residual = o.rel_residual;
        if (converged) *converged = o.converged;
    });
}

int adipc_gpu_pcg_device(adipc_gpu_ctx* ctx, const double* d_b, double rel_tol, int restart, int max_iters, double* d_x,
                         int* iters, double* rel_residual, int* converged) {
    return guarded(ctx, [&] {
        const PcgOut o = pcg(ctx->c, d_b, rel_tol, restart, max_iters, d_x);
        if (iters) *iters = o.iters;
        if (rel_residual) *rel_residual = o.rel_residual;
        if (converged) *converged = o.converged;
    });
}

}  // extern "C"
