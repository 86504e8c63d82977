/*
 * adipc_gpu.h — C-ABI of the B200 (sm_100a) per-Newton linear-solve hot path
 * of StiffGIPC (arXiv 2411.06224), drop-in for the reference `adipc` C++
 * interfaces under /root/reference/proj/include/adipc (cited as adipc/...).
 *
 * Conventions (mirroring the reference's data layout so a C++ shim can pass
 * std::vector storage straight through):
 *   - block keys: uint64 (row << 32) | col           (adipc/sparse/block_coo.hpp:13-21)
 *   - 3x3 blocks: 9 doubles, COLUMN-MAJOR            (Eigen Mat3 storage, core/types.hpp:21)
 *   - vectors:    3n doubles, slot-major (x0 y0 z0 x1 ...) (VecX / std::vector<Vec3>)
 *   - edges:      int32 pairs (a, b) interleaved      (std::vector<std::pair<Index,Index>>)
 *   - Index = int32, Real = double                    (core/types.hpp:9-10)
 * Plain pointers and sizes only. Functions without `_device` take HOST
 * pointers and copy; `_device` variants take device pointers on the context's
 * device and never copy. Every call is stream-ordered on the context stream
 * and returns after its results are ready.
 *
 * Status codes (the shim maps them back to the reference's exceptions):
 *   ADIPC_OK 0
 *   ADIPC_INVALID_ARGUMENT 1 -> std::invalid_argument (e.g. adipc/sparse/reduction.hpp:34)
 *   ADIPC_INDEFINITE 2       -> std::runtime_error "subdomain matrix stayed indefinite
 *                               after regularization" (adipc/precond/mas.hpp:74-77)
 *   ADIPC_CUDA_ERROR 3
 * adipc_gpu_last_error(ctx) returns the message of the last failure.
 * A context is not thread-safe; distinct contexts may be used from distinct
 * host threads and devices.
 */
#ifndef ADIPC_GPU_H
#define ADIPC_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ADIPC_OK 0
#define ADIPC_INVALID_ARGUMENT 1
#define ADIPC_INDEFINITE 2
#define ADIPC_CUDA_ERROR 3

#define ADIPC_PRECOND_MAS 1    /* MasPreconditioner   (adipc/precond/mas.hpp:32-115)        */
#define ADIPC_PRECOND_JACOBI 2 /* BlockJacobiPreconditioner (adipc/precond/block_jacobi.hpp:8-26) */

#define ADIPC_OPT_CACHE_HIERARCHY 1 /* reuse the MAS hierarchy while the sparsity is unchanged */
#define ADIPC_OPT_PROFILE 2         /* time each PCG kernel class with CUDA events */
#define ADIPC_OPT_SOLVE_ORDER 4     /* 1 (default): MAS/PCG renumber slots by level-0 subdomain internally */
#define ADIPC_OPT_SO_KERNELS 6      /* 1 (default): solve-order PCG iteration kernels; 0: the generic level kernels */
#define ADIPC_OPT_PC_PAIRS 11       /* warp pairs per CTA of the preconditioner kernel (1..5, default 5) */
#define ADIPC_OPT_L0_STAGES 7       /* 2 (default) or 3: packed inverses in flight per warp pair in the preconditioner */
#define ADIPC_OPT_DETERMINISTIC 12  /* 1: ExecPolicy::deterministic (core/parallel.hpp:40-43): no fp atomics on the path
                                       (serial-order SpMV of srbk_spmv.hpp:20-27, fixed-order restrictions), so
                                       repeated builds and solves are bitwise identical; default 0 */

typedef struct adipc_gpu_ctx adipc_gpu_ctx;
typedef struct adipc_hierarchy adipc_hierarchy;

/* ---- context ------------------------------------------------------------ */
int adipc_gpu_create(int device, adipc_gpu_ctx** out);
int adipc_gpu_destroy(adipc_gpu_ctx* ctx);
const char* adipc_gpu_last_error(const adipc_gpu_ctx* ctx);
/* Run on an external cudaStream_t (NULL: the context's own stream). */
int adipc_gpu_set_stream(adipc_gpu_ctx* ctx, void* cuda_stream);
int adipc_gpu_set_option(adipc_gpu_ctx* ctx, int option, int value);
/* number of CUDA kernels this library has launched in the process so far */
int64_t adipc_gpu_kernel_launches(void);
/* with ADIPC_OPT_PROFILE: summed ms of the last PCG solve's SpMV, level-0 MAS
 * (+ vector update), coarse MAS and prolongation/p-update launches, and the
 * number of iterations they cover */
int adipc_gpu_pcg_profile(adipc_gpu_ctx* ctx, float* ms4, int* iters);
/* ms of the last assemble / preconditioner build (device) / build host part / pcg loop */
int adipc_gpu_last_timings(adipc_gpu_ctx* ctx, float* ms4);

/* ---- assembly ------------------------------------------------------------------
 * sort_stream + fast_hash_reduction into the context's SortedSymBlockCoo, as at
 * adipc/solver/incremental_potential.hpp:256-257. Replaces
 *   void sort_stream(BlockTripletStream&, const ExecPolicy&)            block_coo.hpp:106
 *   SortedSymBlockCoo fast_hash_reduction(const BlockTripletStream&, Index, const ExecPolicy&)
 *                                                                        reduction.hpp:83
 * Values are bitwise equal to the reference's deterministic mode (ExecPolicy::
 * deterministic, reduction.hpp:39-53) whatever `deterministic` says. Keys must
 * have row < n_block_rows. */
int adipc_gpu_assemble(adipc_gpu_ctx* ctx, const uint64_t* keys, const double* vals9, int64_t T,
                       int32_t n_block_rows, int deterministic, int64_t* n_unique);
int adipc_gpu_assemble_device(adipc_gpu_ctx* ctx, const uint64_t* d_keys, const double* d_vals9, int64_t T,
                              int32_t n_block_rows, int deterministic, int64_t* n_unique);
/* filter_pinned + sort_stream + fast_hash_reduction in one call, exactly the
 * sequence of incremental_potential.hpp:255-257 (pinned: one byte per block
 * slot); the raw stream crosses PCIe once. */
int adipc_gpu_assemble_filtered(adipc_gpu_ctx* ctx, const uint64_t* keys, const double* vals9, int64_t T,
                                int32_t n_block_rows, const uint8_t* pinned, int deterministic, int64_t* n_unique);
int adipc_gpu_assemble_filtered_device(adipc_gpu_ctx* ctx, const uint64_t* d_keys, const double* d_vals9, int64_t T,
                                       int32_t n_block_rows, const uint8_t* d_pinned, int deterministic,
                                       int64_t* n_unique);
int adipc_gpu_matrix_info(adipc_gpu_ctx* ctx, int32_t* n_block_rows, int64_t* n_blocks);
/* copy SortedSymBlockCoo{rows, cols, blocks} out (block_coo.hpp:54-61) */
int adipc_gpu_copy_matrix(adipc_gpu_ctx* ctx, uint32_t* rows, uint32_t* cols, double* blocks9);
/* binary capture of the context's matrix (SPEC.md External Interfaces: binary triplet file for offline
 * oracle checks): "ADIPCMAT", u32 version 1, i32 n_block_rows, i64 U, rows u32[U], cols u32[U],
 * blocks f64[U][9] column-major; api.load_matrix_binary reads it back */
int adipc_gpu_dump_matrix_binary(adipc_gpu_ctx* ctx, const char* path);

/* ---- the step after the solve (TimeStepper, adipc/solver/newton.hpp:257-290), device pointers ----
 * Vectors in the reference block numbering: n_fem FEM vertices, then 4 blocks (p, rows of A) per body. */
/* step_inf_norm (newton.hpp:257-270): max(|d_i| over FEM vertices, |d_p| + |d_A|_F max_xbar[b] over bodies) */
int adipc_gpu_step_inf_norm_device(adipc_gpu_ctx* ctx, const double* d_dir, int32_t n_fem, int32_t n_bodies,
                                   const double* d_max_xbar, double* out);
/* apply_direction (newton.hpp:283-290): out = state + alpha dir over n_dofs (x of the vertices, q of the bodies) */
int adipc_gpu_apply_direction_device(adipc_gpu_ctx* ctx, const double* d_state, const double* d_dir, double alpha,
                                     int64_t n_dofs, double* d_out);
/* the contact gradient lift of assemble_contact (incremental_potential.hpp:395-403):
 * d_grad (block numbering) += node gradient, through J^T for affine-body nodes;
 * slots with d_pinned[slot] != 0 (nullable) receive nothing, as the reference
 * zeroes them right after (:253-254). */
int adipc_gpu_lift_node_grad_device(adipc_gpu_ctx* ctx, const double* d_node_grad, int32_t n_fem, int32_t n_abd,
                                    const int32_t* d_abd_node_body, const double* d_abd_node_jacobian36,
                                    const uint8_t* d_pinned, double* d_grad);
/* contact_node_positions (scene.hpp:112-120): the contact-node positions of a
 * block-numbered state [x; q] — FEM vertices copy x, affine-body node a is
 * affine_point (core/types.hpp:34-40) A x_bar + p in the reference's
 * operation order (x_bar from the node's Jacobian) */
int adipc_gpu_contact_positions_device(adipc_gpu_ctx* ctx, const double* d_state, int32_t n_fem, int32_t n_abd,
                                       const int32_t* d_abd_node_body, const double* d_abd_node_jacobian36,
                                       double* d_out);
/* node_displacements (newton.hpp:272-281): FEM nodes copy d; affine-body node a moves by J_a d_body
 * (abd_node_jacobian 3x12 column-major, 36 doubles per node, DofMap abd_reduce.hpp:11-27) */
int adipc_gpu_node_displacements_device(adipc_gpu_ctx* ctx, const double* d_dir, int32_t n_fem, int32_t n_abd,
                                        const int32_t* d_abd_node_body, const double* d_abd_jacobian36,
                                        double* d_out);

/* dump_block_coo (adipc/sparse/srbk_spmv.hpp:52-60; the CLI's --dump-hessian, adipc_cli.cpp:107-113) of
 * the context's matrix into a text file, byte-identical to the reference's output */
int adipc_gpu_dump_block_coo(adipc_gpu_ctx* ctx, const char* path);
/* upload an existing SortedSymBlockCoo (strictly increasing keys) */
int adipc_gpu_set_matrix(adipc_gpu_ctx* ctx, int32_t n_block_rows, int64_t n_blocks, const uint32_t* rows,
                         const uint32_t* cols, const double* blocks9);
int adipc_gpu_set_matrix_device(adipc_gpu_ctx* ctx, int32_t n_block_rows, int64_t n_blocks, const uint32_t* d_rows,
                                const uint32_t* d_cols, const double* d_blocks9);

/* sort_stream alone (block_coo.hpp:106-113): stable, in place on host arrays. */
int adipc_gpu_sort_stream(adipc_gpu_ctx* ctx, uint64_t* keys, double* vals9, int64_t T);

/* fast_segment_reduction<V> (reduction.hpp:30-79), V = Real (width 1), Vec3 (3)
 * or Mat3 (9). nO != nV -> ADIPC_INVALID_ARGUMENT ("segment map size mismatch"). */
int adipc_gpu_segment_reduce(adipc_gpu_ctx* ctx, const int32_t* O, int64_t nO, const double* V, int64_t nV,
                             int width, int32_t n_segments, int deterministic, double* R);

/* two_level_abd_reduce (adipc/sparse/abd_reduce.hpp:32-74) for the DofMap
 * {n_fem_nodes, n_bodies, abd_node_body[n_abd], abd_node_jacobian[n_abd]
 * (3x12 column-major, 36 doubles each)} (abd_reduce.hpp:11-27). Writes the
 * unsorted tile stream (<= 16 per unique node pair) in the reference's order. */
int adipc_gpu_two_level_abd_reduce(adipc_gpu_ctx* ctx, const uint64_t* keys, const double* vals9, int64_t Tn,
                                   int32_t n_fem, int32_t n_bodies, int32_t n_abd, const int32_t* abd_node_body,
                                   const double* abd_node_jacobian36, uint64_t* out_keys, double* out_vals9,
                                   int64_t out_capacity, int64_t* n_out);

/* The contact half of IncrementalPotential::assemble as one device call:
 *   stream_.append(two_level_abd_reduce(node_stream_, dofs, pol))   incremental_potential.hpp:392-394
 *   filter_pinned(); sort_stream(...); hess = fast_hash_reduction(...)          :253-257
 * The DOF stream (keys/vals9, T) is followed by the reduced tiles, which never
 * leave the device; pinned (n bytes, may be NULL = nothing pinned) filters as
 * filter_pinned does. The result is the context matrix (as adipc_gpu_assemble);
 * n_tiles receives the number of appended tiles. Bit-exact with the reference's
 * deterministic mode. */
int adipc_gpu_assemble_contact(adipc_gpu_ctx* ctx, const uint64_t* keys, const double* vals9, int64_t T,
                               const uint64_t* node_keys, const double* node_vals9, int64_t Tn, int32_t n_fem,
                               int32_t n_bodies, int32_t n_abd, const int32_t* abd_node_body,
                               const double* abd_node_jacobian36, int32_t n_block_rows, const uint8_t* pinned,
                               int64_t* n_unique, int64_t* n_tiles);
int adipc_gpu_assemble_contact_device(adipc_gpu_ctx* ctx, const uint64_t* d_keys, const double* d_vals9, int64_t T,
                                      const uint64_t* d_node_keys, const double* d_node_vals9, int64_t Tn,
                                      int32_t n_fem, int32_t n_bodies, int32_t n_abd, const int32_t* d_abd_node_body,
                                      const double* d_abd_node_jacobian36, int32_t n_block_rows,
                                      const uint8_t* d_pinned, int64_t* n_unique, int64_t* n_tiles);


/* ---- element-Hessian producer --------------------------------
 * The inertia + solid-mesh part of IncrementalPotential::assemble
 * (adipc/solver/incremental_potential.hpp:170-180, 222-239; scatter12 :310-318;
 * pinned gradient :253-254) on the device: stable Neo-Hookean stencils
 * (energy/neo_hookean.hpp:64-104) projected to PSD (energy/psd.hpp:8-14),
 * the triplet stream in the reference's emission order (n_verts inertia
 * diagonals, then 10 blocks per tet), the gradient and the value.
 * Arrays are DEVICE pointers except tet_begin / mu / lambda (host, per solid
 * mesh; tet_begin has n_meshes + 1 entries, tets are global slot ids).
 * Deformable-solid scenes: the FEM vertices are block slots [0, n_verts). */
typedef struct adipc_fem_desc {
    int32_t n_verts;
    const double* x;            /* 3 n_verts: SystemState::x */
    const double* x_tilde;      /* 3 n_verts: the inertial target */
    const double* mass;         /* n_verts: vertex_mass */
    int32_t n_meshes;
    const int64_t* tet_begin;   /* host */
    const double* mu;           /* host, per mesh: solid.mu() */
    const double* lambda;       /* host, per mesh: solid.lambda() */
    const int32_t* tets;        /* 4 per tet */
    const double* rest_inv9;    /* TetRest::inv_rest_edges, 9 column-major per tet */
    const double* rest_volume;  /* TetRest::volume per tet */
    double dt2;
    int project;                /* 1: project_psd every stencil (the reference's default) */
    const uint8_t* pinned;      /* n_verts + 4 n_bodies or NULL: zero gradient on pinned slots */
    /* affine bodies (scene.hpp Body; block rows n_verts + 4 b .. + 3): inertia
     * tiles of the reduced mass (:181-188) and the orthogonality penalty
     * (energy/abd_energy.hpp:19-42, :242-249) */
    int32_t n_bodies;
    const double* q;            /* 12 per body */
    const double* q_tilde;      /* 12 per body */
    const double* reduced_mass; /* 144 per body, column-major */
    const double* body_kappa;
    const double* body_volume;
    /* shells (scene/mesh.hpp is_shell; :190-221): membrane triangles
     * (IncrementalPotential::membrane_stencil, energy/membrane.hpp) and hinges
     * (energy/bending.hpp); per-shell ranges / material on the host */
    int32_t n_shells;
    const int64_t* tri_begin;      /* host, n_shells + 1 */
    const int32_t* tris;           /* 3 per triangle */
    const double* tri_rest;        /* MembraneRest: Dm^-1 (2x2 column-major), area: 5 per triangle */
    const int64_t* hinge_begin;    /* host, n_shells + 1 */
    const int32_t* hinges;         /* 4 per hinge (edge x0-x1, wings x2, x3) */
    const double* hinge_rest;      /* HingeRest: rest angle, weight */
    const double* shell_material;  /* host, 5 per shell: thickness, stretch, strain limit, shear fraction, bending */
    /* the scene's mesh order (0 solid, 1 shell), NULL / 0: solid meshes only */
    int32_t n_kinds;
    const int32_t* mesh_kind;      /* host */
} adipc_fem_desc;
/* the raw stream (n_verts + 10 n_tets + 20 n_bodies + 6 n_tris + 10 n_hinges entries) + gradient
 * (3 (n_verts + 4 n_bodies)) + value */
int adipc_gpu_fem_emit_device(adipc_gpu_ctx* ctx, const adipc_fem_desc* desc, uint64_t* d_keys, double* d_vals9,
                              double* d_grad, double* value);
/* IncrementalPotential::value's inertia + elastic + body terms (:61-131) for
 * the line search: no stream; d_grad may be NULL */
int adipc_gpu_fem_value_device(adipc_gpu_ctx* ctx, const adipc_fem_desc* desc, double* d_grad, double* value);
/* emit + filter_pinned + sort + reduce into the context matrix (the whole
 * assemble() for these scenes; the stream never leaves HBM) */
int adipc_gpu_fem_assemble_device(adipc_gpu_ctx* ctx, const adipc_fem_desc* desc, double* d_grad, double* value,
                                  int64_t* n_unique);


/* ---- contact producers --------------------------------------
 * The contact-node part of IncrementalPotential::assemble_contact
 * (adipc/solver/incremental_potential.hpp:322-384) for given candidates:
 * PT / EE barrier stencils (contact/distance.hpp:13-223, contact/barrier.hpp:
 * 14-66, PSD-projected), the ground barrier (barrier.hpp:70-91) and lagged
 * friction (contact/friction.hpp:12-91). The node stream comes out in the
 * reference's emission order (active PT pairs, active EE pairs, ground
 * contacts, friction constraints) and feeds adipc_gpu_assemble_contact_device.
 * Device arrays over the contact-node universe (FEM vertices, then the body
 * vertices: DofMap, sparse/abd_reduce.hpp:11-27); stencils are node ids —
 * PT (v, t0, t1, t2), EE (a0, a1, b0, b1) — i.e. the broad phase's surface
 * candidates (contact/broad_phase.hpp:146-211) resolved to nodes. */
typedef struct adipc_contact_desc {
    int32_t n_nodes;
    const double* pos;          /* 3 per node */
    int64_t n_pt;
    const int32_t* pt;          /* 4 per PT stencil */
    int64_t n_ee;
    const int32_t* ee;          /* 4 per EE stencil */
    double dhat, kappa;
    int ground;                 /* GroundPlane::enabled */
    double ground_normal[3];
    double ground_height;
    int32_t n_surf_verts;
    const int32_t* surf_verts;  /* ContactSurface::verts as nodes */
    int64_t n_friction;         /* FrictionConstraint arrays: */
    const int32_t* fr_nodes;    /*   4 per constraint */
    const int32_t* fr_n_nodes;
    const double* fr_coeff;     /*   4 per constraint */
    const double* fr_t1;        /*   3 per constraint */
    const double* fr_t2;
    const double* fr_lambda;
    const double* fr_base;      /* 3 per node: positions at the step start */
    double mu, fr_eps;
} adipc_contact_desc;
/* node stream (capacity >= 10 (n_pt + n_ee) + n_surf_verts + 10 n_friction
 * entries), node gradient (3 n_nodes), value; *n_out = entries written */
int adipc_gpu_contact_emit_device(adipc_gpu_ctx* ctx, const adipc_contact_desc* desc, double dt2, int project,
                                  uint64_t* d_node_keys, double* d_node_vals9, int64_t capacity, double* d_node_grad,
                                  double* value, int64_t* n_out);
/* the contact terms of IncrementalPotential::value (:133-157); +inf when a
 * stencil or a surface vertex touches */
int adipc_gpu_contact_value_device(adipc_gpu_ctx* ctx, const adipc_contact_desc* desc, double dt2, double* value);
/* build_friction_constraints (contact/friction.hpp:95-149) for the given
 * candidate stencils — the proximity broad phase of :99 is
 * adipc_gpu_broad_phase_device with inflate dhat: the active PT stencils
 * (0 < closest-feature distance < dhat, distance.hpp:226-256), the active EE
 * stencils, then the ground contacts of desc->surf_verts, in that order, as
 * the lagged friction arrays adipc_contact_desc takes (nodes 4, node count,
 * coefficients 4, tangents t1 / t2, lambda = -b'(d^2) 2 d; tangent_basis
 * :43-47). The friction block of *desc is ignored. capacity >= n_pt + n_ee +
 * n_surf_verts always suffices; the count goes to *n_out. */
int adipc_gpu_friction_constraints_device(adipc_gpu_ctx* ctx, const adipc_contact_desc* desc, int64_t capacity,
                                          int32_t* d_nodes4, int32_t* d_n_nodes, double* d_coeff4, double* d_t1,
                                          double* d_t2, double* d_lambda, int64_t* n_out);
/* scene_ccd_step over the given stencils (contact/ccd.hpp:17-110): the largest
 * fraction of d_disp (3 per node) no stencil or surface vertex can cross */
int adipc_gpu_ccd_step_device(adipc_gpu_ctx* ctx, const adipc_contact_desc* desc, const double* d_disp,
                              double* alpha);


/* ---- broad phase (contact/broad_phase.hpp:143-211) --------------
 * Vertex-triangle and edge-edge candidates of the contact surface whose boxes,
 * inflated by inflate/2 per side (and swept over d_disp when given:
 * ccd_candidates), overlap; stencils sharing a node dropped; sorted and
 * duplicate free (find_candidates' exact result). Device arrays: d_pos /
 * d_disp 3 per node, d_verts (ContactSurface::verts), d_edges 2 / d_tris 3
 * node ids each. The results stay in the context until the next call. */
int adipc_gpu_broad_phase_device(adipc_gpu_ctx* ctx, int32_t n_nodes, const double* d_pos, const double* d_disp,
                                 int32_t n_verts, const int32_t* d_verts, int32_t n_edges, const int32_t* d_edges,
                                 int32_t n_tris, const int32_t* d_tris, double inflate, int64_t* n_pt, int64_t* n_ee);
/* copy the last candidates (host or device destinations, any may be NULL):
 * pairs as surface slots (vert, tri) / (edge, edge), stencils as node ids
 * (v, t0, t1, t2) / (a0, a1, b0, b1) — the contact producer's input */
int adipc_gpu_broad_phase_copy(adipc_gpu_ctx* ctx, int32_t* pt_pairs, int32_t* pt_stencils, int32_t* ee_pairs,
                               int32_t* ee_stencils);

/* IncrementalPotential::filter_pinned (incremental_potential.hpp:410-425):
 * drop blocks touching a pinned slot, append I3 per pinned slot.
 * out capacity >= T + n_slots. */
int adipc_gpu_filter_pinned(adipc_gpu_ctx* ctx, const uint64_t* keys, const double* vals9, int64_t T,
                            const uint8_t* pinned, int32_t n_slots, uint64_t* out_keys, double* out_vals9,
                            int64_t* n_out);
int adipc_gpu_filter_pinned_device(adipc_gpu_ctx* ctx, const uint64_t* d_keys, const double* d_vals9, int64_t T,
                                   const uint8_t* d_pinned, int32_t n_slots, uint64_t* d_out_keys,
                                   double* d_out_vals9, int64_t* n_out);

/* ---- SpMV ------------------------------------------------------------------------
 * srbk_spmv (adipc/sparse/srbk_spmv.hpp:13-49) on the context matrix: y = A x,
 * x and y of 3 * n_block_rows doubles. */
int adipc_gpu_spmv(adipc_gpu_ctx* ctx, const double* x, double* y);
int adipc_gpu_spmv_device(adipc_gpu_ctx* ctx, const double* d_x, double* d_y);

/* ---- partition / hierarchy (host-side integer code, no GPU needed) ---------------- */
int32_t adipc_subdomain_count(int32_t v, int32_t n, int32_t n_o);              /* partition.hpp:12-15 */
int32_t adipc_chunk_partition(int32_t v, int32_t capacity, int32_t* part_of);  /* partition.hpp:25-32, returns n_parts */
int32_t adipc_partition_block_graph(int32_t v, const int32_t* edge_pairs, int64_t n_edges, int32_t capacity,
                                    int32_t* part_of);                         /* partition.hpp:88-159, returns n_parts */
/* build_hierarchy (adipc/precond/hierarchy.hpp:30-100) */
adipc_hierarchy* adipc_build_hierarchy(const int32_t* l0_part_of, int32_t n_slots, int32_t n_parts, int32_t capacity,
                                       const int32_t* edge_pairs, int64_t n_edges, int32_t max_levels);
int adipc_hierarchy_n_levels(const adipc_hierarchy* h);
/* part_of (n_nodes) and agg (n_slots) may be NULL to query sizes */
int adipc_hierarchy_level(const adipc_hierarchy* h, int level, int32_t* n_nodes, int32_t* n_parts, int32_t* part_of,
                          int32_t* agg);
void adipc_hierarchy_free(adipc_hierarchy* h);

/* ---- preconditioner ------------------------------------------------------------------
 * Level-0 partition, fixed per scene (TimeStepper ctor, adipc/solver/newton.hpp:66-68). */
int adipc_gpu_set_level0_partition(adipc_gpu_ctx* ctx, const int32_t* part_of, int32_t n_slots, int32_t n_parts,
                                   int32_t capacity, int32_t max_levels);
/* TimeStepper::build_preconditioner (newton.hpp:243-255): MAS = block_edges +
 * build_hierarchy + MasPreconditioner::build (mas.hpp:34-83), or Jacobi. */
int adipc_gpu_build_preconditioner(adipc_gpu_ctx* ctx, int kind);
/* MasPreconditioner::build(A, h) (mas.hpp:34-83) with a caller-built hierarchy
 * (adipc_build_hierarchy); the level-0 partition is taken from h. */
int adipc_gpu_build_mas(adipc_gpu_ctx* ctx, const adipc_hierarchy* h);
int adipc_gpu_precond_n_levels(adipc_gpu_ctx* ctx);
int adipc_gpu_precond_level(adipc_gpu_ctx* ctx, int level, int32_t* n_nodes, int32_t* n_parts, int32_t* part_of,
                            int32_t* agg);
/* explicit inverse of subdomain `sub` at `level` (dim x dim column-major, dim = 3 f); out may be NULL */
int adipc_gpu_precond_subdomain_inverse(adipc_gpu_ctx* ctx, int level, int32_t sub, int32_t* dim, double* out);
/* number of diagonal regularisation shifts applied by the last build (mas.hpp:68-80) */
int adipc_gpu_precond_shifts(adipc_gpu_ctx* ctx, int64_t* shifts);
/* Preconditioner::apply (mas.hpp:12-15, 85-99; block_jacobi.hpp:16-22) */
int adipc_gpu_precond_apply(adipc_gpu_ctx* ctx, const double* r, double* z);
int adipc_gpu_precond_apply_device(adipc_gpu_ctx* ctx, const double* d_r, double* d_z);

/* ---- PCG -------------------------------------------------------------------------------
 * pcg_solve (adipc/solver/pcg.hpp:34-88) with the context matrix and its built
 * preconditioner: x0 = 0, stop when r.z <= rel_tol^2 r0.z0, residual recomputed
 * every `restart` iterations. Returns PcgResult {iters, rel_residual, converged}. */
int adipc_gpu_pcg(adipc_gpu_ctx* ctx, const double* b, double rel_tol, int restart, int max_iters, double* x,
                  int* iters, double* rel_residual, int* converged);
int adipc_gpu_pcg_device(adipc_gpu_ctx* ctx, const double* d_b, double rel_tol, int restart, int max_iters,
                         double* d_x, int* iters, double* rel_residual, int* converged);

#ifdef __cplusplus
}
#endif

#endif /* ADIPC_GPU_H */
