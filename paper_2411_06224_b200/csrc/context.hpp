// Per-scene device context behind the C-ABI (include/adipc_gpu.h). One
// context = one assembled system + its preconditioner + PCG workspace, all
// resident in HBM. Not thread-safe per context; distinct contexts may live on
// distinct host threads and devices (SURVEY.md §8b conventions).
#pragma once

#include <memory>
#include <string>
#include <vector>

#include "common.cuh"
#include "host_precond.hpp"

struct adipc_gpu_ctx;

namespace adipc_gpu {

// Status codes of the C-ABI (adipc_gpu.h).
enum Status : int { kOk = 0, kInvalidArgument = 1, kIndefinite = 2, kCudaError = 3 };

struct StatusError : std::runtime_error {
    int code;
    StatusError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

// Assembled SortedSymBlockCoo (block_coo.hpp:54-61) in HBM.
//   rows/cols u32[U]; blocks in 32-block tiles, SoA inside a tile (blk(),
//   common.cuh): a warp's 32 consecutive blocks are one contiguous 2,304-byte
//   tile read with nine coalesced 256-byte loads (DRAM page locality: one
//   stream per warp instead of nine); the C-ABI converts to / from the
//   reference's AoS Mat3 storage (72 B per block) at the boundary.
//   row_ptr i64[n+1]: CSR offsets of the sorted rows.
struct DeviceMatrix {
    std::int32_t n = 0;
    std::int64_t U = 0;
    DBuf<std::uint32_t> rows, cols;
    DBuf<double> blocks;
    DBuf<std::int64_t> row_ptr;
    std::uint64_t version = 0;  // bumps on every (re)assembly / upload
};

// One MAS level in HBM (mas.hpp:106-113 LevelData, re-laid out for the GPU).
struct DeviceLevel {
    std::int32_t n_nodes = 0, n_parts = 0;
    DBuf<std::int32_t> agg;        // slot -> node (level 0: identity, not stored)
    DBuf<std::int32_t> part_of;    // node -> subdomain
    DBuf<std::int32_t> pos_of;     // node -> position inside its subdomain
    DBuf<std::int32_t> sub_ptr;    // subdomain -> first member node (CSR over sub_nodes)
    DBuf<std::int32_t> sub_nodes;  // members of each subdomain, ascending node id (= pos order)
    DBuf<std::int32_t> up_first;   // subdomain -> first next-level node nested in it
    DBuf<std::int32_t> upc_ptr;    // next-level node -> range of its children (CSR)
    DBuf<std::int32_t> upc_pos;    // children as positions inside this level's subdomain
    DBuf<std::int32_t> upc_node;   // children as this level's node ids (solve order: level 0 = solve slots)
    DBuf<std::int32_t> up_node;    // node -> the next level's node containing it
    DBuf<std::int32_t> anc;        // level >= 2: level-1 node -> this level's node containing it
    // deterministic build (level >= 1): the solve slots of each subdomain in
    // ascending order (CSR), valid for det_version == Ctx::levels_version
    DBuf<std::int64_t> det_ptr;
    DBuf<std::int32_t> det_slots;
    std::uint64_t det_version = ~0ull;
    DBuf<double> rr;               // level >= 1: restricted residual per node (3 per node)
    std::vector<std::int32_t> pos_host;
    DBuf<std::int64_t> inv_off;    // subdomain -> offset of its packed inverse (16-byte aligned)
    DBuf<double> inv;              // explicit inverses, symmetric-packed upper by columns
    DBuf<std::int64_t> dense_off;  // subdomain -> offset of its dense restricted matrix (build scratch)
    DBuf<double> dense;            // restricted matrices R A R^T, packed lower triangle by columns (build scratch)
    std::int64_t dense_doubles = 0;
    std::vector<std::int64_t> inv_off_host;
    DBuf<double> y;                // level >= 1: per-node solution (3 per node)
    std::int64_t inv_doubles = 0;
    int max_fill = 0;
    void release() {
        for (auto* b : {&agg, &part_of, &pos_of, &sub_ptr, &sub_nodes, &up_first, &upc_ptr, &upc_pos, &upc_node,
                        &up_node, &anc})
            b->free();
        for (auto* b : {&rr, &inv, &dense, &y}) b->free();
        det_ptr.free();
        det_slots.free();
        inv_off.free();
        dense_off.free();
    }
    DeviceLevel() = default;
    DeviceLevel(const DeviceLevel&) = delete;
    DeviceLevel& operator=(const DeviceLevel&) = delete;
    ~DeviceLevel() { release(); }
};

enum PrecondKind : int { kNone = 0, kMas = 1, kJacobi = 2 };

// broad phase (broad.cu): primitive boxes, grid entries and their hash
// table, per-query counts / offsets, the candidate pairs and node stencils
struct BpBox {
    double lo[3], hi[3];
};
struct BpEntry {
    int x, y, z, id;
};
struct BroadState {
    DBuf<BpBox> tri_box, edge_box;
    DBuf<BpEntry> entries, tri_table, edge_table;
    DBuf<std::int64_t> tri_bstart, edge_bstart, off, qoff;
    DBuf<std::int32_t> cnt, bcnt, qcnt;
    DBuf<int> pt_partner, pt_pairs, pt_stencils, ee_partner, ee_pairs, ee_stencils;
    DBuf<double> scal;
    std::int64_t n_pt = 0, n_ee = 0;
};

struct PcgWork {
    DBuf<double> x, r, p, ap, z, b, tmp;
    DBuf<double> partials;       // per-CTA partial dots
    DBuf<unsigned> tickets;      // last-block-done counters
    DBuf<double> scal;           // device scalars (see pcg.cu)
    DBuf<int> flags;             // device flags (see pcg.cu)
};

struct Ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    std::string err;

    DeviceMatrix A;

    // assembly scratch
    DBuf<std::uint64_t> keys, sorted, merge_scratch;
    DBuf<double> vals;
    DBuf<std::int32_t> row_cnt, row_cursor, uniq_cnt, big_rows;
    DBuf<std::int64_t> row_start, uniq_start, scan_scratch;
    DBuf<std::int32_t> counters;
    DBuf<std::int32_t> huge_info, huge_work;  // rows > kHugeRow: (row, len) and the (row, chunk / tile) work lists
    DBuf<std::uint8_t> pinned;
    DBuf<std::int32_t> pin_keep;
    DBuf<std::int64_t> pin_pos, pin_spos;
    // two-level ABD reduction (abd.cu): level-1 node-pair matrix, tile counts /
    // offsets, and the reduced tiles of the device fast path (assemble_contact)
    DeviceMatrix abd_l1;
    DBuf<std::int32_t> abd_cnt;
    DBuf<std::int64_t> abd_off;
    DBuf<std::uint64_t> tile_keys;
    // rows longer than a warp sort in the last bucket sort, and the segments
    // the reduction cuts them into (assemble.cu)
    std::int32_t sort_long_rows = 0;
    DBuf<std::int32_t> seg_cnt, seg_row, seg_heads;
    DBuf<std::int64_t> seg_ptr, seg_bounds, seg_u;
    // element-Hessian producer (energy.cu): the emitted stream + the value
    DBuf<std::uint64_t> fem_keys;
    DBuf<double> fem_vals, fem_value;
    DBuf<unsigned char> hinge_work;  // per-thread dual scratch of the hinge producer
    // indefinite element stencils deferred to the projection pass (energy.cu)
    DBuf<double> fem_defer_m;
    DBuf<std::int64_t> fem_defer_t;
    DBuf<unsigned long long> fem_defer_n;
    // contact producers (contact.cu): activity flags / counts, their prefix
    // sums, the per-thread dual scratch, value / touch / ccd scalars
    DBuf<std::int32_t> ct_on;
    DBuf<std::int64_t> ct_rank;
    DBuf<unsigned char> ct_work;
    DBuf<double> ct_scal;
    BroadState bp;
    DBuf<double> tile_vals;
    // staging of the host-pointer entry points (contact node stream, DofMap)
    DBuf<std::uint64_t> io_keys, io_keys2;
    DBuf<double> io_vals, io_vals2, io_jac;
    DBuf<std::int32_t> io_body;

    // preconditioner
    PrecondKind pkind = kNone;
    host::Partition l0;             // level-0 partition (set once per scene)
    std::uint64_t l0_version = 0, l0_dev_version = ~0ull;  // device copies of l0 (level-1 pass)
    int l0_max_members = 0;
    DBuf<std::int32_t> l0_part, l0_mem_ptr, l0_members, l0_pos;
    DBuf<std::int32_t> l1_up, l1_ncomp, l1_cnt, l1_adj;
    DBuf<std::int64_t> l1_base, l1_ptr;
    DBuf<std::uint64_t> l1_keys;
    std::int64_t l1_E = 0;          // edges of the level-1 graph in l1_ptr / l1_adj
    HostStage stage, stage_up;      // pinned staging of the graphs / node maps that come down
    host::Graph host_graph[3];      // host copies of the coarse graphs (capacity kept across rebuilds)
    // aggregation passes above level 1 on the device (cold build): the
    // level's member lists, the next level's node map, and its graph
    // (ping-pong between two buffers)
    DBuf<std::int32_t> ag_part, ag_mem_ptr, ag_members, ag_pos, ag_up, ag_ncomp, ag_cnt, ag_adj[2];
    DBuf<std::int64_t> ag_base, ag_ptr[2];
    DBuf<std::int32_t> ag_kcnt;     // compacted super-node keys per fine node
    DBuf<std::int64_t> ag_koff;
    int max_levels = 4;
    bool have_l0 = false;
    host::MasHierarchy hier;        // last built hierarchy (host copy)
    std::uint64_t hier_version = ~0ull;
    std::vector<std::unique_ptr<DeviceLevel>> levels;
    DBuf<double> jinv;              // block-Jacobi 3x3 inverses, column-major
    std::int32_t jinv_n = -1;       // their block count
    DBuf<double> invert_scratch;    // global work arrays for subdomains too large for smem
    DBuf<int> build_status;
    long shifts_applied = 0;
    bool cache_hierarchy = false;   // reuse the hierarchy while the pattern is unchanged

    PcgWork w;
    DBuf<unsigned long long> step_max;  // step_inf_norm result (step.cu)
    // level-0 graph of the cold hierarchy build (block_edges + build_graph on the device)
    DBuf<std::int32_t> graph_deg, graph_adj;
    DBuf<std::int64_t> graph_ptr;

    // Solve order (MAS): the PCG and the preconditioner run on A renumbered so
    // that every level-0 subdomain is a contiguous slot range,
    // perm[i] = first slot of subdomain part_of[i] + rank of i inside it
    // (pos_of order, mas.hpp:42-45, is preserved, so the subdomain matrices
    // and inverses are the reference's). The vectors of the level-0 solve,
    // the update pass and the prolongation become unit-stride streams and the
    // SpMV gathers gain locality. Internal only: the C-ABI takes and returns
    // vectors and matrices in the reference's numbering.
    bool solve_order = true;       // ADIPC_OPT_SOLVE_ORDER
    bool perm_active = false;      // the current preconditioner / solve matrix use `perm`
    bool levels_permuted = false;  // the device levels were built in solve order
    std::uint64_t levels_version = 0;  // bumped whenever the device levels are rebuilt
    // level 0 in solve order depends on the level-0 partition alone (fixed per
    // scene): built once per l0_version and kept across cold rebuilds, with
    // the host copies the coarse levels are linked against
    std::uint64_t l0_levels_version = ~0ull;
    std::vector<std::int32_t> perm_host, l0_solve_part_of;
    // byte-balanced work splits of the preconditioner kernels (solve_order.cu)
    struct Split {
        int np = 0;
        std::uint64_t version = ~0ull;
        DBuf<std::int32_t> buf;
    };
    std::vector<Split> splits;
    DBuf<std::int32_t> perm;       // reference slot -> solve slot
    DeviceMatrix As;               // A in solve order (upper triangle re-canonicalised)
    DBuf<std::uint64_t> perm_keys; // scratch stream for building As
    DBuf<std::uint32_t> as_src;    // As entry -> A entry (bit 31: transposed); valid for as_src_version
    std::uint64_t as_src_version = ~0ull;
    std::uint64_t as_a_version = ~0ull;  // A.version As was built from
    DBuf<double> perm_vals;
    DBuf<double> pv_in, pv_out;    // rhs / solution in solve order
    const DeviceMatrix& S() const { return perm_active ? As : A; }
    DeviceMatrix& S() { return perm_active ? As : A; }

    // side stream + fork/join events: the coarse MAS chain runs concurrently
    // with the level-0 solve inside each PCG iteration
    cudaStream_t side = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    // asynchronous done-flag polling of the PCG chunks (pinned, double-buffered)
    cudaStream_t copy_stream = nullptr;  // value uploads overlapping the key sort (host-pointer assembly)
    cudaEvent_t ev_keys = nullptr, ev_vals = nullptr;
    int* h_flags = nullptr;
    cudaEvent_t ev_chunk[2] = {nullptr, nullptr};

    // packed inverses in flight per warp pair of the preconditioner (TMA ring
    // depth, ADIPC_OPT_L0_STAGES) and warp pairs per CTA (ADIPC_OPT_PC_PAIRS:
    // 5 -> 59.5 vs 61.0 us at cfg5)
    int l0_stages = 2;
    int pc_pairs = 5;
    // solve-order iteration kernels (ADIPC_OPT_SO_KERNELS) when the levels allow them
    bool so_kernels = true;

    // deterministic mode (ADIPC_OPT_DETERMINISTIC; the reference's
    // ExecPolicy::deterministic, core/parallel.hpp:40-43): no floating-point
    // atomics anywhere on the path — the row-owner SpMV of the serial
    // srbk_spmv order (spmv.cu k_spmv_det, through the column index below),
    // fixed-order coarse restrictions in the MAS build and the PCG update
    // pass — so repeated solves are bitwise identical
    bool deterministic = false;
    DBuf<std::int64_t> det_tptr;   // column index of the solve matrix: tptr[c].. lists entries (r, c), r < c
    DBuf<std::uint32_t> det_tidx;
    std::uint64_t det_version = ~0ull;
    const DeviceMatrix* det_matrix = nullptr;

    // per-kernel-class PCG timing (ADIPC_OPT_PROFILE): spmv, level 0, coarse, final
    bool profile = false;
    std::vector<cudaEvent_t> prof_events;
    float prof_ms[4] = {0, 0, 0, 0};
    int prof_iters = 0;

    // timings of the last calls, ms (CUDA events on `stream`)
    float ms_assemble = 0, ms_build = 0, ms_build_host = 0, ms_pcg = 0;
    int last_iters = 0;
};

Ctx* unwrap(adipc_gpu_ctx* c);

// assemble.cu
// row bucketing + per-row sort of 64-bit keys (c.sorted / row_start / uniq_cnt);
// d_vidx: emission index of key q (null: q itself)
void bucket_sort(Ctx& c, const std::uint64_t* d_keys, std::int64_t T, std::int32_t n, const std::uint32_t* d_vidx);
// vals_ready: event the reduction waits for (values uploaded on another stream
// while the keys are sorted), or null
void assemble(Ctx& c, const std::uint64_t* d_keys, const double* d_vals, std::int64_t T, std::int32_t n_block_rows,
              int deterministic, cudaEvent_t vals_ready = nullptr);
// filter_pinned + sort + reduce; optionally a second stream segment appended
// after the first (the two-level contact tiles)
// Element-Hessian producer input (energy.cu; incremental_potential.hpp:
// 170-180, 222-239): device arrays except tet_begin / mu / lambda (host,
// one entry per solid mesh; tet_begin has n_meshes + 1).
struct FemDesc {
    std::int32_t n_verts = 0;
    const double* x = nullptr;        // 3 n_verts
    const double* x_tilde = nullptr;  // 3 n_verts
    const double* mass = nullptr;     // n_verts
    std::int32_t n_meshes = 0;
    const std::int64_t* tet_begin = nullptr;
    const double* mu = nullptr;
    const double* lambda = nullptr;
    const std::int32_t* tets = nullptr;     // 4 global slots per tet
    const double* rest_inv9 = nullptr;      // Dm^-1, 9 column-major per tet
    const double* rest_volume = nullptr;    // per tet
    double dt2 = 0;
    int project = 1;
    const std::uint8_t* pinned = nullptr;   // n_verts + 4 n_bodies or null
    // affine bodies (block rows n_verts + 4 b .. + 3)
    std::int32_t n_bodies = 0;
    const double* q = nullptr;             // 12 per body
    const double* q_tilde = nullptr;       // 12 per body
    const double* reduced_mass = nullptr;  // 144 per body, column-major
    const double* body_kappa = nullptr;
    const double* body_volume = nullptr;
    // shells (membrane triangles + hinges) and the scene's mesh order
    std::int32_t n_shells = 0;
    const std::int64_t* tri_begin = nullptr;    // host, n_shells + 1
    const std::int32_t* tris = nullptr;         // 3 per triangle
    const double* tri_rest = nullptr;           // MembraneRest: Dm^-1 (2x2 column-major) + area, 5 per triangle
    const std::int64_t* hinge_begin = nullptr;  // host, n_shells + 1
    const std::int32_t* hinges = nullptr;       // 4 per hinge
    const double* hinge_rest = nullptr;         // HingeRest: rest angle, weight
    const double* shell_material = nullptr;     // host, 5 per shell: thickness, stretch, strain limit, shear fraction, bending
    std::int32_t n_kinds = 0;                   // scene mesh order (0 solid, 1 shell); 0: solids only
    const std::int32_t* mesh_kind = nullptr;    // host
};
void fem_emit(Ctx& c, const FemDesc& d, std::uint64_t* d_keys, double* d_vals, double* d_grad, double* d_value);

// Contact producer input (contact.cu; incremental_potential.hpp:322-384):
// device arrays over the contact-node universe (FEM vertices, then body
// vertices, abd_reduce.hpp:11-27). Stencils are node ids: PT (v, t0, t1, t2),
// EE (a0, a1, b0, b1) — the broad phase's candidates resolved to nodes.
struct ContactDesc {
    std::int32_t n_nodes = 0;
    const double* pos = nullptr;  // 3 per node
    std::int64_t n_pt = 0, n_ee = 0;
    const std::int32_t* pt = nullptr;
    const std::int32_t* ee = nullptr;
    double dhat = 0, kappa = 0;
    int ground = 0;
    double ground_normal[3] = {0, 1, 0};
    double ground_height = 0;
    std::int32_t n_surf_verts = 0;
    const std::int32_t* surf_verts = nullptr;
    std::int64_t n_friction = 0;
    const std::int32_t* fr_nodes = nullptr;  // 4 per constraint
    const std::int32_t* fr_n_nodes = nullptr;
    const double* fr_coeff = nullptr;        // 4 per constraint
    const double* fr_t1 = nullptr;           // 3 per constraint
    const double* fr_t2 = nullptr;
    const double* fr_lambda = nullptr;
    const double* fr_base = nullptr;         // 3 per node
    double mu = 0, fr_eps = 1;
};
// Broad phase input (broad.cu; broad_phase.hpp:143-211): device arrays
struct BroadDesc {
    std::int32_t n_nodes = 0;
    const double* pos = nullptr;   // 3 per node
    const double* disp = nullptr;  // 3 per node or null (ccd_candidates: swept boxes)
    std::int32_t n_verts = 0, n_edges = 0, n_tris = 0;
    const int* verts = nullptr;    // ContactSurface::verts
    const int* edges = nullptr;    // 2 per edge
    const int* tris = nullptr;     // 3 per triangle
    double inflate = 0;
};
void broad_phase(Ctx& c, const BroadDesc& d, std::int64_t* n_pt, std::int64_t* n_ee);

std::int64_t contact_emit(Ctx& c, const ContactDesc& d, double dt2, int project, std::uint64_t* d_keys, double* d_vals,
                          std::int64_t capacity, double* d_node_grad, double* d_value);
std::int64_t friction_constraints(Ctx& c, const ContactDesc& d, std::int64_t capacity, std::int32_t* d_nodes4,
                                  std::int32_t* d_n, double* d_coeff4, double* d_t1, double* d_t2, double* d_lambda);
double contact_value(Ctx& c, const ContactDesc& d, double dt2);
double ccd_step(Ctx& c, const ContactDesc& d, const double* d_disp);

void assemble_filtered(Ctx& c, const std::uint64_t* d_keys, const double* d_vals, std::int64_t T, std::int32_t n,
                       const std::uint8_t* d_pinned, cudaEvent_t vals_ready = nullptr,
                       const std::uint64_t* d_keys2 = nullptr, const double* d_vals2 = nullptr, std::int64_t T2 = 0);
void sort_reduce(Ctx& c, const std::uint64_t* d_keys, const double* d_vals, std::int64_t T, std::int32_t n,
                 DeviceMatrix& out, cudaEvent_t vals_ready = nullptr);
void sort_stream(Ctx& c, const std::uint64_t* d_keys, const double* d_vals, std::int64_t T, std::uint64_t* d_out_keys,
                 double* d_out_vals);
void blocks_aos_to_soa(Ctx& c, const double* aos, double* soa, std::int64_t U);
void blocks_soa_to_aos(Ctx& c, const double* soa, double* aos, std::int64_t U);
void upload_matrix(Ctx& c, std::int32_t n, std::int64_t U, const std::uint32_t* rows, const std::uint32_t* cols,
                   const double* blocks, bool host_ptrs);
void segment_reduce(Ctx& c, const std::int32_t* d_O, std::int64_t n, const double* d_V, int width,
                    std::int32_t n_segments, double* d_R);
std::int64_t filter_pinned(Ctx& c, const std::uint64_t* d_keys, const double* d_vals, std::int64_t T,
                           const std::uint8_t* d_pinned, std::int32_t n_slots, std::uint64_t* d_out_keys,
                           double* d_out_vals);

std::int64_t assemble_contact(Ctx& c, const std::uint64_t* d_keys, const double* d_vals, std::int64_t T,
                              const std::uint64_t* d_nkeys, const double* d_nvals, std::int64_t Tn,
                              std::int32_t n_fem, std::int32_t n_bodies, std::int32_t n_abd, const std::int32_t* d_body,
                              const double* d_jac36, std::int32_t n, const std::uint8_t* d_pinned,
                              cudaEvent_t vals_ready = nullptr);

// step.cu (newton.hpp:257-290): the step after the solve
void contact_positions(Ctx& c, const double* d_state, std::int32_t n_fem, std::int32_t n_abd,
                       const std::int32_t* d_abd_body, const double* d_jac36, double* d_out);
void lift_node_grad(Ctx& c, const double* d_node_grad, std::int32_t n_fem, std::int32_t n_abd,
                    const std::int32_t* d_abd_body, const double* d_jac36, const std::uint8_t* d_pinned,
                    double* d_grad);
double step_inf_norm(Ctx& c, const double* d_dir, std::int32_t n_fem, std::int32_t n_bodies, const double* d_max_xbar);
void apply_direction(Ctx& c, const double* d_state, const double* d_dir, double alpha, std::int64_t n, double* d_out);
void node_displacements(Ctx& c, const double* d_dir, std::int32_t n_fem, std::int32_t n_abd,
                        const std::int32_t* d_abd_body, const double* d_jac36, double* d_out);

// abd.cu
std::int64_t two_level_abd_reduce(Ctx& c, const std::uint64_t* d_keys, const double* d_vals, std::int64_t Tn,
                                  std::int32_t n_fem, std::int32_t n_bodies, std::int32_t n_abd,
                                  const std::int32_t* d_body, const double* d_jac36, std::uint64_t* d_out_keys,
                                  double* d_out_vals, std::int64_t out_cap);

// spmv.cu
void spmv(Ctx& c, const double* d_x, double* d_y);
int spmv_grid(const Ctx& c, const DeviceMatrix& M);
// deterministic mode: build the solve matrix's column index ahead of a graph capture
void prepare_spmv(Ctx& c, const DeviceMatrix& M);
void spmv_launch(Ctx& c, const DeviceMatrix& M, const double* d_x, double* d_y, bool zero_y, const int* flags,
                 double* partials, unsigned* ticket, double* dot_out);

// mas.cu
void build_preconditioner(Ctx& c, PrecondKind kind);
void build_mas_from_hierarchy(Ctx& c, const host::MasHierarchy& h);
void precond_apply(Ctx& c, const double* d_r, double* d_z);
// vectors between the reference numbering and the solve order (Ctx::perm)
void permute_vec(Ctx& c, const double* src, double* dst, bool to_solve);
// before a PCG solve: the preconditioner fits A; As follows A's current values
void check_solve_matrix(Ctx& c);

// pcg.cu
struct PcgOut {
    int iters = 0;
    double rel_residual = 0;
    int converged = 0;
};
PcgOut pcg(Ctx& c, const double* d_b, double rel_tol, int restart, int max_iters, double* d_x);

}  // namespace adipc_gpu
