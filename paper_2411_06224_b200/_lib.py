"""ctypes binding of libadipc_gpu.so (include/adipc_gpu.h). Loading fails
loudly when the native library is missing: there is no CPU fallback on the
product path."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

PKG = os.path.dirname(os.path.abspath(__file__))
GPU_LIB = os.environ.get("ADIPC_GPU_LIB") or os.path.join(PKG, "libadipc_gpu.so")  # env: an A/B build (tools/)

u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
vp, ci, cd, i32, i64 = C.c_void_p, C.c_int, C.c_double, C.c_int32, C.c_int64

OK, INVALID_ARGUMENT, INDEFINITE, CUDA_ERROR = 0, 1, 2, 3
PRECOND_MAS, PRECOND_JACOBI = 1, 2
OPT_CACHE_HIERARCHY = 1
OPT_PROFILE = 2
OPT_SOLVE_ORDER = 4
OPT_SO_KERNELS = 6
OPT_L0_STAGES = 7
OPT_PC_PAIRS = 11
OPT_DETERMINISTIC = 12

# Every symbol include/adipc_gpu.h declares, with its ctypes signature.
class FemDesc(C.Structure):
    """adipc_fem_desc (include/adipc_gpu.h): the element-Hessian producer's
    input — device pointers except tet_begin / mu / lambda (host)."""
    _fields_ = [("n_verts", C.c_int32), ("x", C.c_void_p), ("x_tilde", C.c_void_p), ("mass", C.c_void_p),
                ("n_meshes", C.c_int32), ("tet_begin", C.c_void_p), ("mu", C.c_void_p), ("lam", C.c_void_p),
                ("tets", C.c_void_p), ("rest_inv9", C.c_void_p), ("rest_volume", C.c_void_p), ("dt2", C.c_double),
                ("project", C.c_int), ("pinned", C.c_void_p), ("n_bodies", C.c_int32), ("q", C.c_void_p),
                ("q_tilde", C.c_void_p), ("reduced_mass", C.c_void_p), ("body_kappa", C.c_void_p),
                ("body_volume", C.c_void_p), ("n_shells", C.c_int32), ("tri_begin", C.c_void_p), ("tris", C.c_void_p),
                ("tri_rest", C.c_void_p), ("hinge_begin", C.c_void_p), ("hinges", C.c_void_p),
                ("hinge_rest", C.c_void_p), ("shell_material", C.c_void_p), ("n_kinds", C.c_int32),
                ("mesh_kind", C.c_void_p)]


class ContactDesc(C.Structure):
    """adipc_contact_desc (include/adipc_gpu.h): device arrays over the
    contact-node universe; stencils as node ids."""
    _fields_ = [("n_nodes", C.c_int32), ("pos", C.c_void_p), ("n_pt", C.c_int64), ("pt", C.c_void_p),
                ("n_ee", C.c_int64), ("ee", C.c_void_p), ("dhat", C.c_double), ("kappa", C.c_double),
                ("ground", C.c_int), ("ground_normal", C.c_double * 3), ("ground_height", C.c_double),
                ("n_surf_verts", C.c_int32), ("surf_verts", C.c_void_p), ("n_friction", C.c_int64),
                ("fr_nodes", C.c_void_p), ("fr_n_nodes", C.c_void_p), ("fr_coeff", C.c_void_p),
                ("fr_t1", C.c_void_p), ("fr_t2", C.c_void_p), ("fr_lambda", C.c_void_p), ("fr_base", C.c_void_p),
                ("mu", C.c_double), ("fr_eps", C.c_double)]


GPU_SIGNATURES = {
    "adipc_gpu_create": (ci, [ci, C.POINTER(vp)]),
    "adipc_gpu_destroy": (ci, [vp]),
    "adipc_gpu_last_error": (C.c_char_p, [vp]),
    "adipc_gpu_set_stream": (ci, [vp, vp]),
    "adipc_gpu_set_option": (ci, [vp, ci, ci]),
    "adipc_gpu_last_timings": (ci, [vp, f32p]),
    "adipc_gpu_kernel_launches": (i64, []),
    "adipc_gpu_pcg_profile": (ci, [vp, f32p, C.POINTER(ci)]),
    "adipc_gpu_assemble": (ci, [vp, vp, vp, i64, i32, ci, C.POINTER(i64)]),
    "adipc_gpu_assemble_device": (ci, [vp, vp, vp, i64, i32, ci, C.POINTER(i64)]),
    "adipc_gpu_assemble_filtered": (ci, [vp, vp, vp, i64, i32, vp, ci, C.POINTER(i64)]),
    "adipc_gpu_assemble_filtered_device": (ci, [vp, vp, vp, i64, i32, vp, ci, C.POINTER(i64)]),
    "adipc_gpu_matrix_info": (ci, [vp, C.POINTER(i32), C.POINTER(i64)]),
    "adipc_gpu_copy_matrix": (ci, [vp, vp, vp, vp]),
    "adipc_gpu_dump_block_coo": (ci, [vp, C.c_char_p]),
    "adipc_gpu_dump_matrix_binary": (ci, [vp, C.c_char_p]),
    "adipc_gpu_step_inf_norm_device": (ci, [vp, vp, i32, i32, vp, C.POINTER(cd)]),
    "adipc_gpu_apply_direction_device": (ci, [vp, vp, vp, cd, i64, vp]),
    "adipc_gpu_node_displacements_device": (ci, [vp, vp, i32, i32, vp, vp, vp]),
    "adipc_gpu_contact_positions_device": (ci, [vp, vp, i32, i32, vp, vp, vp]),
    "adipc_gpu_set_matrix": (ci, [vp, i32, i64, vp, vp, vp]),
    "adipc_gpu_set_matrix_device": (ci, [vp, i32, i64, vp, vp, vp]),
    "adipc_gpu_sort_stream": (ci, [vp, vp, vp, i64]),
    "adipc_gpu_segment_reduce": (ci, [vp, vp, i64, vp, i64, ci, i32, ci, vp]),
    "adipc_gpu_two_level_abd_reduce": (ci, [vp, vp, vp, i64, i32, i32, i32, vp, vp, vp, vp, i64, C.POINTER(i64)]),
    "adipc_gpu_assemble_contact": (ci, [vp, vp, vp, i64, vp, vp, i64, i32, i32, i32, vp, vp, i32, vp,
                                        C.POINTER(i64), C.POINTER(i64)]),
    "adipc_gpu_assemble_contact_device": (ci, [vp, vp, vp, i64, vp, vp, i64, i32, i32, i32, vp, vp, i32, vp,
                                               C.POINTER(i64), C.POINTER(i64)]),
    "adipc_gpu_filter_pinned": (ci, [vp, vp, vp, i64, vp, i32, vp, vp, C.POINTER(i64)]),
    "adipc_gpu_lift_node_grad_device": (ci, [vp, vp, i32, i32, vp, vp, vp, vp]),
    "adipc_gpu_broad_phase_device": (ci, [vp, i32, vp, vp, i32, vp, i32, vp, i32, vp, cd, C.POINTER(i64),
                                          C.POINTER(i64)]),
    "adipc_gpu_broad_phase_copy": (ci, [vp, vp, vp, vp, vp]),
    "adipc_gpu_contact_emit_device": (ci, [vp, C.POINTER(ContactDesc), cd, ci, vp, vp, i64, vp, C.POINTER(cd),
                                           C.POINTER(i64)]),
    "adipc_gpu_contact_value_device": (ci, [vp, C.POINTER(ContactDesc), cd, C.POINTER(cd)]),
    "adipc_gpu_ccd_step_device": (ci, [vp, C.POINTER(ContactDesc), vp, C.POINTER(cd)]),
    "adipc_gpu_friction_constraints_device": (ci, [vp, C.POINTER(ContactDesc), i64, vp, vp, vp, vp, vp, vp,
                                                   C.POINTER(i64)]),
    "adipc_gpu_fem_emit_device": (ci, [vp, C.POINTER(FemDesc), vp, vp, vp, C.POINTER(cd)]),
    "adipc_gpu_fem_value_device": (ci, [vp, C.POINTER(FemDesc), vp, C.POINTER(cd)]),
    "adipc_gpu_fem_assemble_device": (ci, [vp, C.POINTER(FemDesc), vp, C.POINTER(cd), C.POINTER(i64)]),
    "adipc_gpu_filter_pinned_device": (ci, [vp, vp, vp, i64, vp, i32, vp, vp, C.POINTER(i64)]),
    "adipc_gpu_spmv": (ci, [vp, vp, vp]),
    "adipc_gpu_spmv_device": (ci, [vp, vp, vp]),
    "adipc_subdomain_count": (i32, [i32, i32, i32]),
    "adipc_chunk_partition": (i32, [i32, i32, vp]),
    "adipc_partition_block_graph": (i32, [i32, vp, i64, i32, vp]),
    "adipc_build_hierarchy": (vp, [vp, i32, i32, i32, vp, i64, i32]),
    "adipc_hierarchy_n_levels": (ci, [vp]),
    "adipc_hierarchy_level": (ci, [vp, ci, C.POINTER(i32), C.POINTER(i32), vp, vp]),
    "adipc_hierarchy_free": (None, [vp]),
    "adipc_gpu_set_level0_partition": (ci, [vp, vp, i32, i32, i32, i32]),
    "adipc_gpu_build_preconditioner": (ci, [vp, ci]),
    "adipc_gpu_build_mas": (ci, [vp, vp]),
    "adipc_gpu_precond_n_levels": (ci, [vp]),
    "adipc_gpu_precond_level": (ci, [vp, ci, C.POINTER(i32), C.POINTER(i32), vp, vp]),
    "adipc_gpu_precond_subdomain_inverse": (ci, [vp, ci, i32, C.POINTER(i32), vp]),
    "adipc_gpu_precond_shifts": (ci, [vp, C.POINTER(i64)]),
    "adipc_gpu_precond_apply": (ci, [vp, vp, vp]),
    "adipc_gpu_precond_apply_device": (ci, [vp, vp, vp]),
    "adipc_gpu_pcg": (ci, [vp, vp, cd, ci, ci, vp, C.POINTER(ci), C.POINTER(cd), C.POINTER(ci)]),
    "adipc_gpu_pcg_device": (ci, [vp, vp, cd, ci, ci, vp, C.POINTER(ci), C.POINTER(cd), C.POINTER(ci)]),
}


_gpu = None


def _load(path, sigs):
    if not os.path.exists(path):
        raise ImportError(
            f"{os.path.basename(path)} is not built (run __graft_entry__.build() or "
            f"python paper_2411_06224_b200/_build.py); there is no CPU fallback")
    L = C.CDLL(path)
    for name, (res, args) in sigs.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    return L


def gpu():
    global _gpu
    if _gpu is None:
        _gpu = _load(GPU_LIB, GPU_SIGNATURES)
    return _gpu


def ptr(a) -> int | None:
    """Raw address of a numpy array or torch tensor (None for None)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data if a.size else None
    return a.data_ptr()  # torch tensor
