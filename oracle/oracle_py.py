"""ORACLE — TEST INFRASTRUCTURE ONLY.

ctypes wrappers over ``oracle/build/liboracle.so`` (the C++ restatement of
the reference hot path, see ``oracle/oracle.hpp``). Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline / reference legs
may import this module; the product package never does.

Array conventions (shared with the product C-ABI, include/adipc_gpu.h):
keys uint64[T]; blocks float64[T, 9] column-major (Eigen ``Mat3::data()``
order); vectors float64[3n]; edges int32[E, 2].
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "build", "liboracle.so")

u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
vp = C.c_void_p
sz = C.c_size_t
i32 = C.c_int32
i64 = C.c_int64
ci = C.c_int
cd = C.c_double


def build() -> None:
    """Compile the oracle with its Makefile (g++ -O2 -fopenmp)."""
    subprocess.check_call(["make", "-s", "-C", _HERE])


_lib = None
_CONTACT_ARGS = [i32, f64p, i64, vp, i64, vp, cd, cd, ci, vp, cd, i32, vp, i64, vp, vp, vp, vp, vp, vp, vp, cd, cd]


def lib():
    global _lib
    if _lib is not None:
        return _ref_dispatch() if _backend == "reference" else _lib
    if not os.path.exists(_LIB_PATH):
        build()
    L = C.CDLL(_LIB_PATH)
    sig = {
        "oracle_last_error": (C.c_char_p, []),
        "oracle_max_threads": (ci, []),
        "oracle_set_default_threads": (None, [ci]),
        "oracle_make_block_key": (C.c_uint64, [C.c_uint32, C.c_uint32]),
        "oracle_emit": (C.c_uint64, [i32, i32, f64p, f64p]),
        "oracle_radix_sort_keys": (None, [u64p, u32p, sz]),
        "oracle_sort_stream": (None, [u64p, f64p, sz, ci, ci, ci]),
        "oracle_fast_hash_reduction": (i64, [u64p, f64p, sz, i32, ci, ci, ci, u32p, u32p, f64p]),
        "oracle_segment_reduce": (ci, [i32p, sz, f64p, sz, ci, i32, ci, ci, ci, f64p]),
        "oracle_srbk_spmv": (None, [i32, sz, u32p, u32p, f64p, f64p, sz, ci, ci, ci, f64p]),
        "oracle_split": (ci, [ci, i32, i32, f64p, u64p, f64p]),
        "oracle_two_level_abd_reduce": (i64, [u64p, f64p, sz, i32, i32, sz, i32p, f64p, ci, ci, ci, u64p, f64p]),
        "oracle_filter_pinned": (i64, [u64p, f64p, sz, u8p, i32, u64p, f64p]),
        "oracle_subdomain_count": (i32, [i32, i32, i32]),
        "oracle_chunk_partition": (i32, [i32, i32, i32p]),
        "oracle_partition_block_graph": (i32, [i32, i32p, sz, i32, i32p]),
        "oracle_block_edges": (i64, [sz, u32p, u32p, i32p]),
        "oracle_build_hierarchy": (vp, [i32p, i32, i32, i32, i32p, sz, ci]),
        "oracle_hierarchy_free": (None, [vp]),
        "oracle_hierarchy_n_levels": (ci, [vp]),
        "oracle_hierarchy_level": (None, [vp, ci, C.POINTER(i32), C.POINTER(i32), vp, vp]),
        "oracle_matrix_new": (vp, [i32, sz, u32p, u32p, f64p]),
        "oracle_matrix_free": (None, [vp]),
        "oracle_mas_build": (vp, [vp, vp]),
        "oracle_precond_free": (None, [vp]),
        "oracle_mas_shifts": (C.c_long, [vp]),
        "oracle_mas_n_levels": (ci, [vp]),
        "oracle_mas_level_matrix": (ci, [vp, ci, i32, vp]),
        "oracle_jacobi_build": (vp, [vp]),
        "oracle_precond_apply": (None, [vp, f64p, sz, f64p]),
        "oracle_pcg_solve": (ci, [vp, f64p, sz, vp, cd, ci, ci, ci, ci, ci, f64p,
                                  C.POINTER(ci), C.POINTER(cd), C.POINTER(ci)]),
        "oracle_rng_new": (vp, [C.c_uint32]),
        "oracle_rng_free": (None, [vp]),
        "oracle_dist_uniform_int": (vp, [C.c_long, C.c_long]),
        "oracle_dist_normal": (vp, [cd, cd]),
        "oracle_dist_uniform_real": (vp, [cd, cd]),
        "oracle_dist_free": (None, [vp]),
        "oracle_dist_draw": (cd, [vp, vp]),
        "oracle_dist_fill": (None, [vp, vp, f64p, sz]),
        "oracle_random_stream": (None, [vp, ci, ci, u64p, f64p]),
        "oracle_random_spd3": (None, [vp, cd, f64p]),
        "oracle_tet_rest": (ci, [f64p, f64p, f64p]),
        "oracle_pt_dist2_derivs": (None, [f64p, f64p, f64p, f64p]),
        "oracle_ee_dist2_derivs": (None, [f64p, f64p, f64p, f64p]),
        "oracle_pt_dist2": (cd, [f64p]),
        "oracle_ee_dist2": (cd, [f64p]),
        "oracle_barrier_pair_derivs": (None, [cd, f64p, f64p, cd, cd, ci, f64p, f64p, f64p]),
        "oracle_ground_barrier_derivs": (None, [f64p, f64p, cd, cd, cd, ci, f64p, f64p, f64p, f64p]),
        "oracle_contact_assemble": (i64, _CONTACT_ARGS + [cd, ci, u64p, f64p, f64p, f64p]),
        "oracle_contact_value": (cd, _CONTACT_ARGS + [cd]),
        "oracle_ccd_step": (cd, _CONTACT_ARGS + [f64p]),
        "oracle_find_candidates": (i64, [i32, f64p, vp, i32, vp, i32, vp, i32, vp, cd, vp, i64, vp, i64,
                                         C.POINTER(i64)]),
        "oracle_stable_neo_hookean": (None, [f64p, f64p, cd, cd, cd, ci, f64p, f64p, f64p]),
        "oracle_project_psd": (None, [ci, f64p, f64p]),
        "oracle_ip_fem_assemble": (i64, [i32, f64p, f64p, f64p, i32, i64p, f64p, f64p, i32p, f64p, f64p, cd, vp, ci,
                                         u64p, f64p, f64p, f64p, i32, vp, vp, vp, vp, vp,
                                         i32, vp, vp, vp, vp, vp, vp, vp, i32, vp]),
        "oracle_membrane_rest": (ci, [f64p, f64p]),
        "oracle_membrane_stencil": (None, [f64p, f64p, f64p, ci, f64p, f64p, f64p]),
        "oracle_hinge_rest": (ci, [f64p, f64p]),
        "oracle_hinge_bending": (None, [f64p, f64p, cd, ci, f64p, f64p, f64p]),
        "oracle_abd_orthogonality": (None, [f64p, cd, cd, ci, f64p, f64p, f64p]),
        "oracle_pt_contact_frame": (None, [f64p, f64p, f64p, f64p]),
        "oracle_ee_contact_frame": (None, [f64p, f64p, f64p, f64p]),
        "oracle_tangent_basis": (None, [f64p, f64p, f64p]),
        "oracle_friction_constraints": (i64, _CONTACT_ARGS + [i64, vp, vp, vp, vp, vp, vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    global _SIG
    _SIG = sig
    return _ref_dispatch() if _backend == "reference" else L


# ------------------------------------------------------- reference backend --
# oracle/_ref/libadipc_ref.so is the reference's OWN hot-path code compiled in
# place (oracle/ref_capi.cpp, oracle/Makefile target `ref`). Its ref_* entries
# have the oracle_* signatures, so every wrapper below runs on either library:
# `with use_backend("reference"): ...` routes compute entries to it (entries
# it lacks — the test RNG — stay on the restatement).
_REF_PATH = os.path.join(_HERE, "_ref", "libadipc_ref.so")
_REF_SRC = "/root/reference/proj/include"
_backend = "restated"
_SIG = None
_ref = None


def reference_available() -> bool:
    if os.path.exists(_REF_PATH):
        return True
    if os.path.isdir(_REF_SRC):
        try:
            subprocess.check_call(["make", "-s", "-C", _HERE, "ref"])
        except (OSError, subprocess.CalledProcessError):
            return False
        return os.path.exists(_REF_PATH)
    return False


class _Dispatch:
    def __init__(self, base, ref):
        self._base, self._ref = base, ref

    def __getattr__(self, name):
        f = getattr(self._ref, "ref_" + name[len("oracle_"):], None) if name.startswith("oracle_") else None
        if f is None:
            return getattr(self._base, name)
        res, args = _SIG[name]
        f.restype, f.argtypes = res, args
        return f


def _ref_dispatch():
    global _ref
    if _ref is None:
        if not reference_available():
            raise RuntimeError("oracle/_ref/libadipc_ref.so missing and /root/reference not present")
        _ref = _Dispatch(_lib, C.CDLL(_REF_PATH))
    return _ref


def backend() -> str:
    return _backend


class use_backend:
    """Context manager: ``"restated"`` (oracle.hpp) or ``"reference"``."""

    def __init__(self, name):
        assert name in ("restated", "reference")
        self.name = name

    def __enter__(self):
        global _backend
        self.prev, _backend = _backend, self.name
        return lib()

    def __exit__(self, *exc):
        global _backend
        _backend = self.prev


def _pol(policy):
    if policy is None:
        return 0, 0, 32
    return int(bool(policy.deterministic)), int(policy.threads), int(policy.lane_width)


class ExecPolicy:
    """core/parallel.hpp:18-22."""

    def __init__(self, deterministic=False, threads=0, lane_width=32):
        self.deterministic = deterministic
        self.threads = threads
        self.lane_width = lane_width


# ---------------------------------------------------------------- RNG ------
class Rng:
    """std::mt19937 of the reference tests (libstdc++ draws)."""

    def __init__(self, seed: int):
        self.h = lib().oracle_rng_new(seed)

    def __del__(self):
        if getattr(self, "h", None):
            lib().oracle_rng_free(self.h)
            self.h = None


class _Dist:
    def __init__(self, h):
        self.h = h

    def __call__(self, rng: Rng):
        return lib().oracle_dist_draw(self.h, rng.h)

    def fill(self, rng: Rng, n: int) -> np.ndarray:
        out = np.empty(n, np.float64)
        lib().oracle_dist_fill(self.h, rng.h, out, n)
        return out

    def __del__(self):
        if getattr(self, "h", None):
            lib().oracle_dist_free(self.h)
            self.h = None


class UniformInt(_Dist):
    def __init__(self, a, b):
        super().__init__(lib().oracle_dist_uniform_int(a, b))

    def __call__(self, rng):
        return int(super().__call__(rng))


class Normal(_Dist):
    def __init__(self, m=0.0, s=1.0):
        super().__init__(lib().oracle_dist_normal(m, s))


class UniformReal(_Dist):
    def __init__(self, a, b):
        super().__init__(lib().oracle_dist_uniform_real(a, b))


def random_stream(rng: Rng, n_blocks: int, n_entries: int):
    keys = np.empty(n_entries, np.uint64)
    vals = np.empty((n_entries, 9), np.float64)
    lib().oracle_random_stream(rng.h, n_blocks, n_entries, keys, vals)
    return keys, vals


def random_spd3(rng: Rng, shift: float = 1.0) -> np.ndarray:
    out = np.empty(9, np.float64)
    lib().oracle_random_spd3(rng.h, shift, out)
    return out


# --------------------------------------------------------------- sparse ----
def make_block_key(r, c):
    return lib().oracle_make_block_key(r, c)


def emit(r, c, m9):
    out = np.empty(9, np.float64)
    k = lib().oracle_emit(r, c, np.ascontiguousarray(m9, np.float64), out)
    return k, out


def radix_sort_keys(keys):
    k = np.array(keys, np.uint64)
    perm = np.empty(len(k), np.uint32)
    lib().oracle_radix_sort_keys(k, perm, len(k))
    return k, perm


def sort_stream(keys, vals, policy=None):
    k = np.array(keys, np.uint64)
    v = np.array(vals, np.float64).reshape(-1, 9).copy()
    lib().oracle_sort_stream(k, v, len(k), *_pol(policy))
    return k, v


def fast_hash_reduction(keys, vals, n_block_rows, policy=None):
    k = np.ascontiguousarray(keys, np.uint64)
    v = np.ascontiguousarray(vals, np.float64).reshape(-1, 9)
    T = len(k)
    rows = np.empty(max(T, 1), np.uint32)
    cols = np.empty(max(T, 1), np.uint32)
    blocks = np.empty((max(T, 1), 9), np.float64)
    U = lib().oracle_fast_hash_reduction(k, v, T, n_block_rows, *_pol(policy), rows, cols, blocks)
    return rows[:U].copy(), cols[:U].copy(), blocks[:U].copy()


def fast_segment_reduction(O, V, n_segments, policy=None):
    O = np.ascontiguousarray(O, np.int32)
    V = np.ascontiguousarray(V, np.float64)
    width = 1 if V.ndim == 1 else V.shape[1]
    nV = V.shape[0]
    R = np.empty((max(n_segments, 1), width), np.float64)
    rc = lib().oracle_segment_reduce(O, len(O), V.reshape(-1) if nV else np.zeros(1), nV, width,
                                     n_segments, *_pol(policy), R)
    if rc != 0:
        raise ValueError(lib().oracle_last_error().decode())
    R = R[:n_segments]
    return R[:, 0].copy() if width == 1 else R.copy()


def reference_dump_block_coo(n_block_rows, rows, cols, blocks) -> str:
    """The reference's own dump_block_coo (srbk_spmv.hpp:52-60), compiled in
    oracle/_ref: the text the CLI's --dump-hessian writes."""
    if not reference_available():
        raise RuntimeError("oracle/_ref unavailable")
    f = C.CDLL(_REF_PATH).ref_dump_block_coo
    f.restype = C.c_int64
    U = len(rows)
    r = np.ascontiguousarray(rows, np.uint32) if U else np.zeros(1, np.uint32)
    c = np.ascontiguousarray(cols, np.uint32) if U else np.zeros(1, np.uint32)
    b = np.ascontiguousarray(blocks, np.float64).reshape(-1) if U else np.zeros(9)
    args = [C.c_int32(n_block_rows), C.c_size_t(U), r.ctypes.data_as(C.c_void_p), c.ctypes.data_as(C.c_void_p),
            b.ctypes.data_as(C.c_void_p)]
    size = f(*args, None, C.c_size_t(0))
    buf = C.create_string_buffer(size + 1)
    f(*args, buf, C.c_size_t(size + 1))
    return buf.raw[:size].decode()


def srbk_spmv(n_block_rows, rows, cols, blocks, x, policy=None):
    x = np.ascontiguousarray(x, np.float64).reshape(-1)
    nx = len(x) // 3
    y = np.empty(max(3 * nx, 1), np.float64)
    U = len(rows)
    lib().oracle_srbk_spmv(n_block_rows, U, np.ascontiguousarray(rows, np.uint32) if U else np.zeros(1, np.uint32),
                           np.ascontiguousarray(cols, np.uint32) if U else np.zeros(1, np.uint32),
                           np.ascontiguousarray(blocks, np.float64).reshape(-1) if U else np.zeros(9),
                           x if nx else np.zeros(3), nx, *_pol(policy), y)
    return y[: 3 * nx].copy()


SPLIT_12x12, SPLIT_SYM_12x12, SPLIT_12x3, SPLIT_3x12 = 0, 1, 2, 3


def split(kind, rb, cb, H):
    """H given as a 2-D numpy array in natural shape (row, col)."""
    Hc = np.ascontiguousarray(np.asarray(H, np.float64).T).reshape(-1)  # column-major
    keys = np.empty(16, np.uint64)
    vals = np.empty((16, 9), np.float64)
    n = lib().oracle_split(kind, rb, cb, Hc, keys, vals)
    return keys[:n].copy(), vals[:n].copy()


def two_level_abd_reduce(keys, vals, n_fem, n_bodies, abd_node_body, jac36, policy=None):
    k = np.ascontiguousarray(keys, np.uint64)
    v = np.ascontiguousarray(vals, np.float64).reshape(-1, 9)
    body = np.ascontiguousarray(abd_node_body, np.int32)
    jac = np.ascontiguousarray(jac36, np.float64).reshape(-1)
    cap = max(16 * len(k), 1)
    ok = np.empty(cap, np.uint64)
    ov = np.empty((cap, 9), np.float64)
    n = lib().oracle_two_level_abd_reduce(k, v, len(k), n_fem, n_bodies, len(body),
                                          body if len(body) else np.zeros(1, np.int32),
                                          jac if len(jac) else np.zeros(1), *_pol(policy), ok, ov)
    return ok[:n].copy(), ov[:n].copy()


# ------------------------------------------- element-Hessian producer ----
def tet_rest(p12):
    """energy/neo_hookean.hpp:13-27 -> (inv_rest_edges 9 column-major, volume)."""
    p = np.ascontiguousarray(p12, np.float64).reshape(12)
    inv, vol = np.empty(9), np.empty(1)
    if lib().oracle_tet_rest(p, inv, vol) != 0:
        raise ValueError(lib().oracle_last_error().decode())
    return inv, float(vol[0])


def stable_neo_hookean(x12, inv9, vol, mu, lam, project=True):
    """energy/neo_hookean.hpp:64-104 -> (value, grad 12, hess 12x12 column-major)."""
    val, g, h = np.empty(1), np.empty(12), np.empty(144)
    lib().oracle_stable_neo_hookean(np.ascontiguousarray(x12, np.float64).reshape(12),
                                    np.ascontiguousarray(inv9, np.float64).reshape(9), vol, mu, lam, int(project),
                                    val, g, h)
    return float(val[0]), g, h.reshape(12, 12).T.copy()


def project_psd(M):
    """energy/psd.hpp:8-14 on a symmetric n x n matrix."""
    M = np.asarray(M, np.float64)
    n = M.shape[0]
    out = np.empty(n * n)
    lib().oracle_project_psd(n, np.ascontiguousarray(M.T).reshape(-1), out)
    return out.reshape(n, n).T.copy()


def membrane_rest(p9):
    """energy/membrane.hpp:17-32 -> 5 doubles: Dm^-1 (2x2 column-major), area."""
    out = np.empty(5)
    if lib().oracle_membrane_rest(np.ascontiguousarray(p9, np.float64).reshape(9), out) != 0:
        raise ValueError(lib().oracle_last_error().decode())
    return out


def membrane_stencil(x9, rest5, material5, project=True):
    """IncrementalPotential::membrane_stencil (incremental_potential.hpp:273-298)
    -> (value, grad 9, hess 9x9). material5 = thickness, stretch, strain
    limit, shear fraction, bending."""
    v, g, h = np.empty(1), np.empty(9), np.empty(81)
    lib().oracle_membrane_stencil(np.ascontiguousarray(x9, np.float64).reshape(9),
                                  np.ascontiguousarray(rest5, np.float64), np.ascontiguousarray(material5, np.float64),
                                  int(project), v, g, h)
    return float(v[0]), g, h.reshape(9, 9).T.copy()


def hinge_rest(p12):
    """energy/bending.hpp:36-48 -> (rest angle, weight)."""
    out = np.empty(2)
    if lib().oracle_hinge_rest(np.ascontiguousarray(p12, np.float64).reshape(12), out) != 0:
        raise ValueError(lib().oracle_last_error().decode())
    return out


def hinge_bending(x12, rest2, k, project=True):
    """energy/bending.hpp:60-75 -> (value, grad 12, hess 12x12)."""
    v, g, h = np.empty(1), np.empty(12), np.empty(144)
    lib().oracle_hinge_bending(np.ascontiguousarray(x12, np.float64).reshape(12),
                               np.ascontiguousarray(rest2, np.float64), k, int(project), v, g, h)
    return float(v[0]), g, h.reshape(12, 12).T.copy()


def abd_orthogonality(q12, kappa, volume, project=True):
    """energy/abd_energy.hpp:19-42 -> (value, grad 12, hess 12x12)."""
    v, g, h = np.empty(1), np.empty(12), np.empty(144)
    lib().oracle_abd_orthogonality(np.ascontiguousarray(q12, np.float64).reshape(12), kappa, volume, int(project),
                                   v, g, h)
    return float(v[0]), g, h.reshape(12, 12).T.copy()


_KEEP = []


def _keep(a):
    _KEEP.append(a)
    return a.ctypes.data


def _shell_ptrs(sh, ns):
    if not ns:
        return [None] * 7
    conv = [("tri_begin", np.int64), ("tris", np.int32), ("tri_rest", np.float64), ("hinge_begin", np.int64),
            ("hinges", np.int32), ("hinge_rest", np.float64), ("material", np.float64)]
    return [_keep(np.ascontiguousarray(sh[k], t).reshape(-1)) for k, t in conv]


def ip_fem_assemble(x, x_tilde, mass, tet_begin, mu, lam, tets, inv9, vol, dt2, pinned=None, project=True,
                    bodies=None, shells=None, mesh_kind=None):
    """IncrementalPotential::assemble restricted to inertia + solid meshes +
    affine bodies (incremental_potential.hpp:170-249, 310-318, 253-254) ->
    (value, grad 3 (n + 4 nb), keys, vals) in emission order. bodies: dict of
    q (nb x 12), q_tilde, reduced_mass (nb x 12 x 12), kappa, volume."""
    x = np.ascontiguousarray(x, np.float64).reshape(-1)
    n = len(x) // 3
    tb = np.ascontiguousarray(tet_begin, np.int64)
    nm = len(tb) - 1
    nt = int(tb[-1])
    nb = 0 if bodies is None else len(bodies["kappa"])
    sh = shells or {}
    ns = len(sh.get("material", []))
    n_tri = int(sh["tri_begin"][-1]) if ns else 0
    n_hg = int(sh["hinge_begin"][-1]) if ns else 0
    cap = max(n + 10 * nt + 20 * nb + 6 * n_tri + 10 * n_hg, 1)
    keys, vals = np.empty(cap, np.uint64), np.empty((cap, 9))
    grad, val = np.empty(3 * (n + 4 * nb)), np.empty(1)
    bq = {}
    if nb:
        bq = {k: np.ascontiguousarray(bodies[k], np.float64) for k in ("q", "q_tilde", "kappa", "volume")}
        bq["reduced_mass"] = np.ascontiguousarray(np.asarray(bodies["reduced_mass"], np.float64).transpose(0, 2, 1))
    bp = lambda k: bq[k].ctypes.data if nb else None  # noqa: E731
    pin = None if pinned is None else np.ascontiguousarray(pinned, np.uint8)
    T = lib().oracle_ip_fem_assemble(n, x, np.ascontiguousarray(x_tilde, np.float64).reshape(-1),
                                     np.ascontiguousarray(mass, np.float64), nm, tb,
                                     np.ascontiguousarray(mu, np.float64), np.ascontiguousarray(lam, np.float64),
                                     np.ascontiguousarray(tets, np.int32).reshape(-1),
                                     np.ascontiguousarray(inv9, np.float64).reshape(-1),
                                     np.ascontiguousarray(vol, np.float64), dt2,
                                     None if pin is None else pin.ctypes.data, int(project), keys, vals, grad, val,
                                     nb, bp("q"), bp("q_tilde"), bp("reduced_mass"), bp("kappa"), bp("volume"),
                                     ns, *_shell_ptrs(sh, ns),
                                     0 if mesh_kind is None else len(mesh_kind),
                                     None if mesh_kind is None else _keep(np.ascontiguousarray(mesh_kind, np.int32)))
    return float(val[0]), grad, keys[:T].copy(), vals[:T].copy()


# --------------------------------------------------- contact producers ----
def _x12(x):
    return np.ascontiguousarray(x, np.float64).reshape(12)


def pt_dist2_derivs(x12):
    """contact/distance.hpp:159-189 -> (dist2, grad 12, hess 12x12)."""
    d, g, h = np.empty(1), np.empty(12), np.empty(144)
    lib().oracle_pt_dist2_derivs(_x12(x12), d, g, h)
    return float(d[0]), g, h.reshape(12, 12).T.copy()


def ee_dist2_derivs(x12):
    """contact/distance.hpp:191-223."""
    d, g, h = np.empty(1), np.empty(12), np.empty(144)
    lib().oracle_ee_dist2_derivs(_x12(x12), d, g, h)
    return float(d[0]), g, h.reshape(12, 12).T.copy()


def pt_dist2(x12):
    return float(lib().oracle_pt_dist2(_x12(x12)))


def ee_dist2(x12):
    return float(lib().oracle_ee_dist2(_x12(x12)))


def barrier_pair_derivs(d2, g, H, shat, kappa, project=True):
    """contact/barrier.hpp:50-66 -> (value, grad 12, hess 12x12)."""
    v, og, oh = np.empty(1), np.empty(12), np.empty(144)
    lib().oracle_barrier_pair_derivs(d2, np.ascontiguousarray(g, np.float64),
                                     np.ascontiguousarray(np.asarray(H, np.float64).T).reshape(-1), shat, kappa,
                                     int(project), v, og, oh)
    return float(v[0]), og, oh.reshape(12, 12).T.copy()


def ground_barrier_derivs(x, normal, height, dhat, kappa, project=True):
    """contact/barrier.hpp:70-91 -> (value, grad 3, hess 3x3, dist)."""
    v, g, h, d = np.empty(1), np.empty(3), np.empty(9), np.empty(1)
    lib().oracle_ground_barrier_derivs(np.ascontiguousarray(x, np.float64), np.ascontiguousarray(normal, np.float64),
                                       height, dhat, kappa, int(project), v, g, h, d)
    return float(v[0]), g, h.reshape(3, 3).T.copy(), float(d[0])


class ContactInput:
    """Inputs of the contact-node part of assemble_contact / value / ccd:
    positions, PT / EE stencils (node ids), ground plane + surface vertices,
    lagged friction constraints."""

    def __init__(self, pos, pt=(), ee=(), dhat=1e-3, kappa=1.0, ground=None, surf_verts=(), friction=None,
                 fr_base=None, mu=0.0, fr_eps=1.0):
        self.pos = np.ascontiguousarray(pos, np.float64).reshape(-1, 3)
        self.pt = np.ascontiguousarray(np.asarray(pt, np.int32).reshape(-1, 4))
        self.ee = np.ascontiguousarray(np.asarray(ee, np.int32).reshape(-1, 4))
        self.dhat, self.kappa = float(dhat), float(kappa)
        self.ground = ground  # (normal 3, height) or None
        self.surf_verts = np.ascontiguousarray(np.asarray(surf_verts, np.int32).reshape(-1))
        f = friction or {}
        nf = len(f.get("n", []))
        self.fr_n = np.ascontiguousarray(np.asarray(f.get("n", []), np.int32).reshape(nf))
        self.fr_nodes = np.ascontiguousarray(np.asarray(f.get("nodes", np.zeros((nf, 4))), np.int32).reshape(nf, 4))
        self.fr_coeff = np.ascontiguousarray(np.asarray(f.get("coeff", np.zeros((nf, 4))), np.float64).reshape(nf, 4))
        self.fr_t1 = np.ascontiguousarray(np.asarray(f.get("t1", np.zeros((nf, 3))), np.float64).reshape(nf, 3))
        self.fr_t2 = np.ascontiguousarray(np.asarray(f.get("t2", np.zeros((nf, 3))), np.float64).reshape(nf, 3))
        self.fr_lambda = np.ascontiguousarray(np.asarray(f.get("lam", np.zeros(nf)), np.float64).reshape(nf))
        self.fr_base = np.ascontiguousarray(self.pos if fr_base is None else fr_base, np.float64).reshape(-1, 3)
        self.mu, self.fr_eps = float(mu), float(fr_eps)

    def args(self):
        p = lambda a: a.ctypes.data if a.size else None  # noqa: E731
        normal = np.ascontiguousarray(self.ground[0], np.float64) if self.ground is not None else None
        self._keep = normal
        return [len(self.pos), self.pos.reshape(-1), len(self.pt), p(self.pt), len(self.ee), p(self.ee), self.dhat,
                self.kappa, int(self.ground is not None), None if normal is None else normal.ctypes.data,
                float(self.ground[1]) if self.ground is not None else 0.0, len(self.surf_verts), p(self.surf_verts),
                len(self.fr_n), p(self.fr_nodes), p(self.fr_n), p(self.fr_coeff), p(self.fr_t1), p(self.fr_t2),
                p(self.fr_lambda), p(self.fr_base), self.mu, self.fr_eps]

    def max_entries(self):
        return 10 * (len(self.pt) + len(self.ee)) + len(self.surf_verts) + 10 * len(self.fr_n)


def contact_assemble(ci: ContactInput, dt2, project=True):
    """incremental_potential.hpp:322-384 node part -> (value, node_grad 3n, keys, vals)."""
    cap = max(ci.max_entries(), 1)
    keys, vals = np.empty(cap, np.uint64), np.empty((cap, 9))
    g, v = np.empty(3 * len(ci.pos)), np.empty(1)
    T = lib().oracle_contact_assemble(*ci.args(), dt2, int(project), keys, vals, g, v)
    return float(v[0]), g, keys[:T].copy(), vals[:T].copy()


def contact_value(ci: ContactInput, dt2):
    """incremental_potential.hpp:133-157 (contact terms of the line-search value)."""
    return float(lib().oracle_contact_value(*ci.args(), dt2))


def ccd_step(ci: ContactInput, disp):
    """contact/ccd.hpp:88-110 over the given stencils."""
    return float(lib().oracle_ccd_step(*ci.args(), np.ascontiguousarray(disp, np.float64).reshape(-1)))


def find_candidates(pos, verts, edges, tris, inflate, disp=None):
    """contact/broad_phase.hpp:143-211 -> (pt pairs (vert slot, tri slot),
    ee pairs (edge slot, edge slot), both sorted, duplicate free)."""
    pos = np.ascontiguousarray(pos, np.float64).reshape(-1)
    v = np.ascontiguousarray(verts, np.int32).reshape(-1)
    e = np.ascontiguousarray(edges, np.int32).reshape(-1)
    t = np.ascontiguousarray(tris, np.int32).reshape(-1)
    d = None if disp is None else np.ascontiguousarray(disp, np.float64).reshape(-1)
    p = lambda a: a.ctypes.data if a is not None and a.size else None  # noqa: E731
    cap_pt, cap_ee = max(len(v), 1) * 64, max(len(e) // 2, 1) * 64
    while True:
        pt, ee, nee = np.empty(2 * cap_pt, np.int32), np.empty(2 * cap_ee, np.int32), C.c_int64()
        npt = lib().oracle_find_candidates(len(pos) // 3, pos, p(d), len(v), p(v), len(e) // 2, p(e), len(t) // 3,
                                           p(t), float(inflate), pt.ctypes.data, cap_pt, ee.ctypes.data, cap_ee,
                                           C.byref(nee))
        if npt >= 0:
            return pt[:2 * npt].reshape(-1, 2).copy(), ee[:2 * nee.value].reshape(-1, 2).copy()
        cap_pt, cap_ee = cap_pt * 4, cap_ee * 4


def filter_pinned(keys, vals, pinned):
    k = np.ascontiguousarray(keys, np.uint64)
    v = np.ascontiguousarray(vals, np.float64).reshape(-1, 9)
    p = np.ascontiguousarray(pinned, np.uint8)
    cap = len(k) + len(p) + 1
    ok = np.empty(cap, np.uint64)
    ov = np.empty((cap, 9), np.float64)
    n = lib().oracle_filter_pinned(k, v, len(k), p, len(p), ok, ov)
    if n < 0:  # not exposed by the compiled reference (ref_capi.cpp): restated version
        n = _lib.oracle_filter_pinned(k, v, len(k), p, len(p), ok, ov)
    return ok[:n].copy(), ov[:n].copy()


# -------------------------------------------------------------- precond ----
def subdomain_count(v, n, n_o):
    return lib().oracle_subdomain_count(v, n, n_o)


def _edges(edges):
    e = np.ascontiguousarray(np.asarray(edges, np.int32).reshape(-1, 2))
    return (e if len(e) else np.zeros((1, 2), np.int32)), len(e)


def chunk_partition(v, cap):
    part = np.empty(max(v, 1), np.int32)
    n = lib().oracle_chunk_partition(v, cap, part)
    return part[:v].copy(), n


def partition_block_graph(v, edges, cap):
    e, ne = _edges(edges)
    part = np.empty(max(v, 1), np.int32)
    n = lib().oracle_partition_block_graph(v, e, ne, cap, part)
    return part[:v].copy(), n


def block_edges(rows, cols):
    U = len(rows)
    out = np.empty((max(U, 1), 2), np.int32)
    n = lib().oracle_block_edges(U, np.ascontiguousarray(rows, np.uint32), np.ascontiguousarray(cols, np.uint32), out)
    return out[:n].copy()


class Hierarchy:
    """MasHierarchy (hierarchy.hpp:15-28) restated."""

    def __init__(self, part_of, n_parts, capacity, edges, max_levels):
        part_of = np.ascontiguousarray(part_of, np.int32)
        e, ne = _edges(edges)
        self.n_slots = len(part_of)
        self.capacity = capacity
        self._L = L = lib()
        self.h = L.oracle_build_hierarchy(part_of if len(part_of) else np.zeros(1, np.int32),
                                              self.n_slots, n_parts, capacity, e, ne, max_levels)
        self.levels = []
        for l in range(self._L.oracle_hierarchy_n_levels(self.h)):
            nn, npart = i32(), i32()
            self._L.oracle_hierarchy_level(self.h, l, C.byref(nn), C.byref(npart), None, None)
            part = np.empty(max(nn.value, 1), np.int32)
            agg = np.empty(max(self.n_slots, 1), np.int32)
            self._L.oracle_hierarchy_level(self.h, l, C.byref(nn), C.byref(npart),
                                         part.ctypes.data_as(vp), agg.ctypes.data_as(vp))
            self.levels.append(dict(n_nodes=nn.value, n_parts=npart.value,
                                    part_of=part[: nn.value].copy(), agg=agg[: self.n_slots].copy()))

    def n_levels(self):
        return len(self.levels)

    def __del__(self):
        if getattr(self, "h", None):
            self._L.oracle_hierarchy_free(self.h)
            self.h = None


class Matrix:
    def __init__(self, n_block_rows, rows, cols, blocks):
        self.n_block_rows = n_block_rows
        U = len(rows)
        self._L = lib()
        self.h = self._L.oracle_matrix_new(n_block_rows, U,
                                         np.ascontiguousarray(rows, np.uint32) if U else np.zeros(1, np.uint32),
                                         np.ascontiguousarray(cols, np.uint32) if U else np.zeros(1, np.uint32),
                                         np.ascontiguousarray(blocks, np.float64).reshape(-1) if U else np.zeros(9))

    def __del__(self):
        if getattr(self, "h", None):
            self._L.oracle_matrix_free(self.h)
            self.h = None


class _Precond:
    def apply(self, r):
        r = np.ascontiguousarray(r, np.float64)
        z = np.empty_like(r)
        self._L.oracle_precond_apply(self.h, r, len(r), z)
        return z

    def __del__(self):
        if getattr(self, "h", None):
            self._L.oracle_precond_free(self.h)
            self.h = None


class MasPreconditioner(_Precond):
    def __init__(self, mat: Matrix, hier: Hierarchy):
        self._L = mat._L
        self.h = self._L.oracle_mas_build(mat.h, hier.h)
        if not self.h:
            raise RuntimeError(self._L.oracle_last_error().decode())

    def n_levels(self):
        return self._L.oracle_mas_n_levels(self.h)

    def shifts(self):
        return self._L.oracle_mas_shifts(self.h)

    def level_matrix(self, l, s):
        d = self._L.oracle_mas_level_matrix(self.h, l, s, None)
        out = np.empty(d * d, np.float64)
        self._L.oracle_mas_level_matrix(self.h, l, s, out.ctypes.data_as(vp))
        return out.reshape(d, d).T.copy()  # column-major -> natural


class BlockJacobiPreconditioner(_Precond):
    def __init__(self, mat: Matrix):
        self._L = mat._L
        self.h = self._L.oracle_jacobi_build(mat.h)


def pcg_solve(mat: Matrix, b, M: _Precond, rel_tol, restart, max_iters, policy=None):
    b = np.ascontiguousarray(b, np.float64)
    x = np.empty_like(b)
    it, rr, cv = ci(), cd(), ci()
    mat._L.oracle_pcg_solve(mat.h, b, len(b), M.h, rel_tol, restart, max_iters, *_pol(policy), x,
                           C.byref(it), C.byref(rr), C.byref(cv))
    return x, dict(iters=it.value, rel_residual=rr.value, converged=bool(cv.value))


# ---- the step after the solve (adipc/solver/newton.hpp:257-290), restated ----
# Vectors in block numbering: n_fem vertices, then 4 blocks (12 dofs: p, the
# rows of A) per affine body at block n_fem + 4 b (DofMap, abd_reduce.hpp:24).
def step_inf_norm(d, n_fem, n_bodies, max_xbar):
    """newton.hpp:257-270."""
    d = np.asarray(d, np.float64)
    worst = 0.0
    for i in range(n_fem):
        worst = max(worst, float(np.sqrt(d[3 * i] ** 2 + d[3 * i + 1] ** 2 + d[3 * i + 2] ** 2)))
    for b in range(n_bodies):
        s = d[3 * (n_fem + 4 * b): 3 * (n_fem + 4 * b) + 12]
        worst = max(worst, float(np.sqrt(np.sum(s[:3] ** 2)) + np.sqrt(np.sum(s[3:] ** 2)) * max_xbar[b]))
    return worst


def apply_direction(state, d, alpha):
    """newton.hpp:283-290 (x + alpha d for the vertices, q + alpha d for the bodies)."""
    return np.asarray(state, np.float64) + alpha * np.asarray(d, np.float64)


def node_displacements(d, n_fem, abd_node_body, jac36):
    """newton.hpp:272-281: FEM nodes copy d, affine-body node a gets J_a d_body."""
    d = np.asarray(d, np.float64)
    out = [d[: 3 * n_fem]]
    for a, b in enumerate(abd_node_body):
        J = np.asarray(jac36[a], np.float64).reshape(12, 3).T  # column-major 3x12
        out.append(J @ d[3 * (n_fem + 4 * b): 3 * (n_fem + 4 * b) + 12])
    return np.concatenate(out) if out else np.zeros(0)


def contact_node_positions(state, n_fem, abd_node_body, jac36):
    """scene.hpp:112-120 contact_node_positions: FEM vertices copy x; an
    affine-body node is affine_point(q, x_bar) = A x_bar + p (core/types.hpp:
    34-40), rows of A from q, in that operation order (x_bar read from the
    node's Jacobian)."""
    state = np.asarray(state, np.float64)
    out = [state[: 3 * n_fem].reshape(-1, 3)]
    J = np.asarray(jac36, np.float64).reshape(-1, 12, 3)  # [node][col][row]
    xb = J[:, 3:6, 0]  # x_bar_k = J(0, 3 + k)
    q = state[3 * n_fem:].reshape(-1, 12)[np.asarray(abd_node_body)]
    A = q[:, 3:].reshape(-1, 3, 3)
    pos = ((A[:, :, 0] * xb[:, 0:1] + A[:, :, 1] * xb[:, 1:2]) + A[:, :, 2] * xb[:, 2:3]) + q[:, :3]
    out.append(pos)
    return np.concatenate(out)


def abd_jacobian(rest):
    """mesh.hpp:196-201: J = [I3 | rows r: rest^T at columns 3 + 3 r], column-major 36 doubles."""
    J = np.zeros((3, 12))
    J[:, :3] = np.eye(3)
    for r in range(3):
        J[r, 3 + 3 * r: 6 + 3 * r] = rest
    return J.T.reshape(-1).copy()


# ---- IncrementalPotential::assemble composed (incremental_potential.hpp:162-258) ----
def lift_node_grad(node_grad, n_fem, abd_node_body, jac36, grad):
    """:395-403 — grad (block numbering) += node gradient: FEM nodes copy-add,
    affine-body node a adds J_a^T g_a to its body's 12 dofs, in node order."""
    g = np.asarray(node_grad, np.float64).reshape(-1, 3)
    grad[: 3 * n_fem] += g[:n_fem].reshape(-1)  # zero node gradients add nothing
    for a, b in enumerate(abd_node_body):
        gn = g[n_fem + a]
        if np.dot(gn, gn) == 0:
            continue
        J = np.asarray(jac36[a], np.float64).reshape(12, 3)  # J^T rows
        s = 3 * (n_fem + 4 * int(b))
        grad[s: s + 12] += J @ gn
    return grad


def ip_assemble(sc, state, policy=None, project=True, ground=None, friction=None, fr_base=None, mu=0.0, fr_eps=1.0):
    """IncrementalPotential::assemble on a scene of one solid mesh + affine
    bodies + a contact surface (scenegen.geom.GeomHybrid's attributes): the
    element stream (ip_fem_assemble), contact-node positions, the proximity
    broad phase (find_candidates, inflate dhat, :330), the contact node part
    (contact_assemble), the gradient lift, two_level_abd_reduce appended to
    the stream, pinned gradient zeroing (:253-254), filter_pinned, sort and
    reduce. ground = (normal, height) adds the ground barrier of the surface
    vertices; friction (friction_constraints' dict) with fr_base / mu /
    fr_eps the lagged friction. Returns (value, grad, rows, cols, blocks,
    counts)."""
    state = np.asarray(state, np.float64)
    n_fem, nb = sc.n_fem, sc.n_bodies
    x, q = state[: 3 * n_fem], state[3 * n_fem:].reshape(nb, 12)
    bodies = None
    if nb:
        bodies = {"q": q, "q_tilde": sc.q_tilde, "reduced_mass": sc.reduced_mass, "kappa": sc.kappa_abd,
                  "volume": sc.body_volume}
    dt2 = sc.dt * sc.dt
    val, grad, keys, vals = ip_fem_assemble(x, sc.x_tilde, sc.mass, sc.tet_begin, [sc.mu], [sc.lam], sc.tets,
                                            sc.rest_inv9, sc.rest_volume, dt2, None, project, bodies)
    pos = contact_node_positions(state, n_fem, sc.abd_body, sc.jac36)
    pt, ee = find_candidates(pos, sc.surf_verts, sc.edges, sc.tris, sc.dhat)
    ci = ContactInput(pos, np.c_[sc.surf_verts[pt[:, 0]], sc.tris[pt[:, 1]]],
                      np.c_[sc.edges[ee[:, 0]], sc.edges[ee[:, 1]]], dhat=sc.dhat, kappa=sc.kappa, ground=ground,
                      surf_verts=sc.surf_verts, friction=friction, fr_base=fr_base, mu=mu, fr_eps=fr_eps)
    cv, ng, nk, nv = contact_assemble(ci, dt2, project)
    val += cv
    tk, tv = two_level_abd_reduce(nk, nv, n_fem, nb, sc.abd_body, sc.jac36, policy)
    lift_node_grad(ng, n_fem, sc.abd_body, sc.jac36, grad)
    grad.reshape(-1, 3)[np.asarray(sc.pinned, bool)] = 0
    fk, fv = filter_pinned(np.concatenate([keys, tk]), np.concatenate([vals, tv]), sc.pinned)
    sk, sv = sort_stream(fk, fv, policy)
    rows, cols, blocks = fast_hash_reduction(sk, sv, sc.n_blocks, policy)
    return val, grad, rows, cols, blocks, {"n_pt": len(pt), "n_ee": len(ee), "node_blocks": len(nk),
                                           "contact_tiles": len(tk)}


# ---- friction constraints (friction.hpp:43-149, distance.hpp:226-256) -----------
def pt_contact_frame(x12):
    """distance.hpp:232-242 -> (dist, normal 3, coeff 4)."""
    d, nrm, cf = np.zeros(1), np.zeros(3), np.zeros(4)
    lib().oracle_pt_contact_frame(_x12(x12), d, nrm, cf)
    return float(d[0]), nrm, cf


def ee_contact_frame(x12):
    """distance.hpp:244-256 -> (dist, normal 3, coeff 4)."""
    d, nrm, cf = np.zeros(1), np.zeros(3), np.zeros(4)
    lib().oracle_ee_contact_frame(_x12(x12), d, nrm, cf)
    return float(d[0]), nrm, cf


def tangent_basis(n):
    """friction.hpp:43-47 -> (t1, t2)."""
    t1, t2 = np.zeros(3), np.zeros(3)
    lib().oracle_tangent_basis(np.ascontiguousarray(n, np.float64), t1, t2)
    return t1, t2


def _friction_arrays(cap):
    return {"nodes": np.empty((cap, 4), np.int32), "n": np.empty(cap, np.int32), "coeff": np.empty((cap, 4)),
            "t1": np.empty((cap, 3)), "t2": np.empty((cap, 3)), "lam": np.empty(cap)}


def _friction_trim(f, k):
    return {key: v[:k].copy() for key, v in f.items()}


def friction_constraints(ci: ContactInput):
    """build_friction_constraints (friction.hpp:95-149) over the ContactInput's
    GIVEN candidate stencils (active PT, active EE, ground contacts) -> dict
    nodes / n / coeff / t1 / t2 / lam (ContactInput's friction format)."""
    cap = max(len(ci.pt) + len(ci.ee) + len(ci.surf_verts), 1)
    f = _friction_arrays(cap)
    k = lib().oracle_friction_constraints(*ci.args(), cap, *[a.ctypes.data for a in f.values()])
    return _friction_trim(f, int(k))


def build_friction_constraints(pos, verts, edges, tris, dhat, kappa, ground=None):
    """friction.hpp:95-149 with its own proximity broad phase: the reference's
    compiled function under the reference backend; the restatement composes
    find_candidates (inflate dhat) with friction_constraints."""
    pos = np.ascontiguousarray(pos, np.float64).reshape(-1, 3)
    verts = np.ascontiguousarray(verts, np.int32).reshape(-1)
    edges = np.ascontiguousarray(edges, np.int32).reshape(-1, 2)
    tris = np.ascontiguousarray(tris, np.int32).reshape(-1, 3)
    if _backend == "reference":
        L = C.CDLL(_REF_PATH)
        fn = L.ref_build_friction_constraints
        fn.restype = i64
        fn.argtypes = [i32, f64p, i32, vp, i32, vp, i32, vp, ci, vp, cd, cd, cd, i64, vp, vp, vp, vp, vp, vp]
        cap = max(len(verts) * 64, 1)
        while True:
            f = _friction_arrays(cap)
            nrm = None if ground is None else np.ascontiguousarray(ground[0], np.float64)
            k = fn(len(pos), pos.reshape(-1), len(verts), verts.ctypes.data, len(edges), edges.ctypes.data, len(tris),
                   tris.ctypes.data, int(ground is not None), None if nrm is None else nrm.ctypes.data,
                   0.0 if ground is None else float(ground[1]), float(dhat), float(kappa), cap,
                   *[a.ctypes.data for a in f.values()])
            if k >= 0:
                return _friction_trim(f, int(k))
            cap = int(-k - 1)
    pt, ee = find_candidates(pos, verts, edges, tris, dhat)
    cin = ContactInput(pos, np.c_[verts[pt[:, 0]], tris[pt[:, 1]]], np.c_[edges[ee[:, 0]], edges[ee[:, 1]]],
                       dhat=dhat, kappa=kappa, ground=ground, surf_verts=verts)
    return friction_constraints(cin)


# ---- the reference's own Scene + IncrementalPotential (oracle/_ref) ------------
class RefScene:
    """The reference's Scene (scene/scene.hpp: finalize — boundary extraction,
    masses, rest data, body reduced masses), its DofMap and ContactSurface, and
    IncrementalPotential::assemble (solver/incremental_potential.hpp:19-258),
    compiled in place. meshes: dicts rest (n x 3), tets (local, m x 4),
    youngs, poisson, density; bodies: dicts rest, tets, kappa, density."""

    def __init__(self, meshes, bodies, dt, ground=None, shells=()):
        """shells (after the solid meshes in the scene's mesh order): dicts
        rest, tris, density, thickness, stretch, strain_limit, shear_fraction,
        bending."""
        if not reference_available():
            raise RuntimeError("oracle/_ref not built")
        L = self._L = C.CDLL(_REF_PATH)
        L.ref_scene_new.restype = vp
        L.ref_scene_new.argtypes = [i32, vp, vp, vp, vp, vp, vp, vp, i32, vp, vp, vp, vp, vp, vp, cd, ci, vp, cd,
                                    i32, vp, vp, vp, vp, vp]
        L.ref_scene_shell_sizes.argtypes = [vp, vp, vp]
        L.ref_scene_shell_export.argtypes = [vp] + [vp] * 7
        L.ref_scene_free.argtypes = [vp]
        L.ref_scene_sizes.argtypes = [vp, vp]
        L.ref_scene_export.argtypes = [vp] + [vp] * 14
        L.ref_scene_begin_friction.restype = i64
        L.ref_scene_begin_friction.argtypes = [vp, f64p, f64p, cd, cd, cd, cd]
        L.ref_scene_assemble.restype = i64
        L.ref_scene_assemble.argtypes = [vp, f64p, f64p, f64p, f64p, cd, cd, ci, f64p, f64p, i64, vp, vp, vp]
        cat = lambda xs, dt_: np.ascontiguousarray(np.concatenate(xs) if xs else np.zeros(0), dt_)  # noqa: E731
        begin = lambda xs: np.ascontiguousarray(np.r_[0, np.cumsum([len(x) for x in xs])], np.int64)  # noqa: E731
        self._keep = [cat([m["rest"] for m in meshes], np.float64), begin([m["rest"] for m in meshes]),
                      cat([m["tets"] for m in meshes], np.int32), begin([m["tets"] for m in meshes]),
                      np.array([m["youngs"] for m in meshes], np.float64),
                      np.array([m["poisson"] for m in meshes], np.float64),
                      np.array([m["density"] for m in meshes], np.float64),
                      cat([b["rest"] for b in bodies], np.float64), begin([b["rest"] for b in bodies]),
                      cat([b["tets"] for b in bodies], np.int32), begin([b["tets"] for b in bodies]),
                      np.array([b["kappa"] for b in bodies], np.float64),
                      np.array([b["density"] for b in bodies], np.float64),
                      None if ground is None else np.ascontiguousarray(ground[0], np.float64),
                      cat([m["rest"] for m in shells], np.float64), begin([m["rest"] for m in shells]),
                      cat([m["tris"] for m in shells], np.int32), begin([m["tris"] for m in shells]),
                      np.array([[m["density"], m["thickness"], m["stretch"], m["strain_limit"], m["shear_fraction"],
                                 m["bending"]] for m in shells], np.float64).reshape(-1)]
        k = self._keep
        p = lambda a: None if a is None or a.size == 0 else a.ctypes.data  # noqa: E731
        self.h = L.ref_scene_new(len(meshes), p(k[1]), p(k[0]), p(k[3]), p(k[2]), p(k[4]), p(k[5]), p(k[6]),
                                 len(bodies), p(k[8]), p(k[7]), p(k[10]), p(k[9]), p(k[11]), p(k[12]), float(dt),
                                 int(ground is not None), p(k[13]), 0.0 if ground is None else float(ground[1]),
                                 len(shells), p(k[15]), p(k[14]), p(k[17]), p(k[16]), p(k[18]))
        sz = np.zeros(9, np.int64)
        L.ref_scene_sizes(self.h, sz.ctypes.data)
        (self.n_fem, self.n_bodies, self.n_blocks, self.n_nodes, n_tets, n_sv, n_e, n_t, n_m) = (int(v) for v in sz)
        d = {"mass": np.zeros(self.n_fem), "rest_inv9": np.zeros((n_tets, 9)), "rest_volume": np.zeros(n_tets),
             "tets": np.zeros((n_tets, 4), np.int32), "mu": np.zeros(n_m), "lam": np.zeros(n_m),
             "reduced_mass": np.zeros((self.n_bodies, 144)), "body_volume": np.zeros(self.n_bodies),
             "abd_body": np.zeros(self.n_nodes - self.n_fem, np.int32),
             "jac36": np.zeros((self.n_nodes - self.n_fem, 36)), "surf_verts": np.zeros(n_sv, np.int32),
             "edges": np.zeros((n_e, 2), np.int32), "tris": np.zeros((n_t, 3), np.int32),
             "length_scale": np.zeros(1)}
        L.ref_scene_export(self.h, *[p(d[k_]) if d[k_].size else None for k_ in
                                     ("mass", "rest_inv9", "rest_volume", "tets", "mu", "lam", "reduced_mass",
                                      "body_volume", "abd_body", "jac36", "surf_verts", "edges", "tris")],
                           d["length_scale"].ctypes.data)
        d["tet_begin"] = np.r_[0, np.cumsum([len(m["tets"]) for m in meshes])].astype(np.int64)
        d["mu"], d["lam"] = d["mu"][:len(meshes)], d["lam"][:len(meshes)]
        if shells:
            ntr, nh = np.zeros(1, np.int64), np.zeros(1, np.int64)
            L.ref_scene_shell_sizes(self.h, ntr.ctypes.data, nh.ctypes.data)
            sh = {"tris": np.zeros((int(ntr[0]), 3), np.int32), "tri_rest": np.zeros((int(ntr[0]), 5)),
                  "hinges": np.zeros((int(nh[0]), 4), np.int32), "hinge_rest": np.zeros((int(nh[0]), 2)),
                  "material": np.zeros((len(shells), 5)), "tri_count": np.zeros(len(shells), np.int64),
                  "hinge_count": np.zeros(len(shells), np.int64)}
            L.ref_scene_shell_export(self.h, *[p(sh[k_]) if sh[k_].size else None for k_ in
                                               ("tris", "tri_rest", "hinges", "hinge_rest", "material", "tri_count",
                                                "hinge_count")])
            sh["tri_begin"] = np.r_[0, np.cumsum(sh["tri_count"])].astype(np.int64)
            sh["hinge_begin"] = np.r_[0, np.cumsum(sh["hinge_count"])].astype(np.int64)
            d["shells"] = sh
            d["mesh_kind"] = np.array([0] * len(meshes) + [1] * len(shells), np.int32)
        self.data = d

    def __del__(self):
        if getattr(self, "h", None):
            self._L.ref_scene_free(self.h)
            self.h = None

    def begin_friction(self, x, q, dhat, kappa, mu, eps):
        """newton.hpp:104-113: build_friction_constraints at (x, q), base = those positions."""
        return int(self._L.ref_scene_begin_friction(self.h, np.ascontiguousarray(x, np.float64).reshape(-1),
                                                    np.ascontiguousarray(q, np.float64).reshape(-1), dhat, kappa,
                                                    mu, eps))

    def assemble(self, x, q, x_tilde, q_tilde, dhat, kappa, deterministic=True):
        """IncrementalPotential::assemble -> (value, grad, rows, cols, blocks)."""
        grad = np.zeros(3 * self.n_blocks)
        val = np.zeros(1)
        cap = 64 * self.n_blocks + 1024
        while True:
            rows, cols = np.zeros(cap, np.uint32), np.zeros(cap, np.uint32)
            blocks = np.zeros((cap, 9))
            U = self._L.ref_scene_assemble(self.h, np.ascontiguousarray(x, np.float64).reshape(-1),
                                           np.ascontiguousarray(q, np.float64).reshape(-1),
                                           np.ascontiguousarray(x_tilde, np.float64).reshape(-1),
                                           np.ascontiguousarray(q_tilde, np.float64).reshape(-1), dhat, kappa,
                                           int(deterministic), val, grad, cap, rows.ctypes.data, cols.ctypes.data,
                                           blocks.ctypes.data)
            if U >= 0:
                return float(val[0]), grad, rows[:U].copy(), cols[:U].copy(), blocks[:U].copy()
            cap = int(-U - 1)
