"""Synthetic benchmark / test scenes (BASELINE.json configs 1-5): input
generation for bench.py and the tests, NOT part of the product package.

The generators (scenegen/scenes.cpp, host C++) stand in for the reference's
element and contact producers (out of scope) and restate its
mesh generators and emission order — see the header of scenes.cpp. The same
source is built twice: scenegen/libadipc_scenes.so for the GPU arm and the
tests, and oracle/build/libadipc_scenes.so for the reference arm of bench.py,
which loads only libraries under oracle/ (`use_library("oracle")`).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIBS = {"scenegen": os.path.join(HERE, "libadipc_scenes.so"),
        "oracle": os.path.join(ROOT, "oracle", "build", "libadipc_scenes.so")}
CXX = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"

vp, ci, cd = C.c_void_p, C.c_int, C.c_double
SIGNATURES = {
    "adipc_scene_fem_box": (vp, [ci, ci, ci, cd, cd, cd, cd, cd, cd, cd, ci, cd, C.c_uint]),
    "adipc_scene_cloth": (vp, [ci, ci, cd, cd, C.c_uint]),
    "adipc_scene_abd_stack": (vp, [ci, ci, ci, C.c_uint]),
    "adipc_scene_hybrid": (vp, [ci, ci, ci, ci, ci, cd, C.c_uint]),
    "adipc_scene_free": (None, [vp]),
    "adipc_scene_mesh_sizes": (None, [vp, vp, vp]),
    "adipc_scene_copy_mesh": (None, [vp, vp, vp, vp]),
    "adipc_scene_sizes": (None, [vp, vp]),
    "adipc_scene_copy": (None, [vp, vp, vp, vp, vp, vp, vp, vp, vp]),
}
_which = "scenegen"
_lib = None


def build(verbose: bool = False) -> None:
    """Compile scenes.cpp into scenegen/libadipc_scenes.so (in-tree, travels
    with the snapshot). The oracle copy is built by oracle/Makefile."""
    src = os.path.join(HERE, "scenes.cpp")
    out = LIBS["scenegen"]
    if os.path.exists(out) and os.path.getmtime(out) >= os.path.getmtime(src):
        return
    cmd = [CXX, "-O2", "-std=c++17", "-fPIC", "-Wall", "-Wextra", "-shared", "-o", out, src]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.check_call(cmd)


def use_library(which: str) -> None:
    """Select the generator build: "scenegen" (default) or "oracle"."""
    global _which, _lib
    if which not in LIBS:
        raise ValueError(which)
    _which, _lib = which, None


def lib():
    global _lib
    if _lib is None:
        path = LIBS[_which]
        if not os.path.exists(path):
            raise ImportError(f"{path} is not built (run __graft_entry__.build())")
        L = C.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def ptr(a):
    return a.ctypes.data if a.size else None


class Scene:
    """Triplet streams + pins + rest connectivity of one synthetic scene.

    keys/vals:            DOF stream before contact tiles (emission order)
    node_keys/node_vals:  contact node-pair stream (two-level ABD input)
    abd_body/jac36:       DofMap of the contact-node universe
    pinned:               uint8 per block slot
    rest_edges:           int32 [E, 2] (newton.hpp:204-241), the L0 partition input
    """

    def __init__(self, handle):
        L = lib()
        try:
            sz = np.zeros(7, np.int64)
            L.adipc_scene_sizes(handle, ptr(sz))
            self.n_blocks, self.n_fem, self.n_bodies, n_abd, T, Tn, ne = (int(v) for v in sz)
            self.keys = np.empty(T, np.uint64)
            self.vals = np.empty((T, 9), np.float64)
            self.node_keys = np.empty(Tn, np.uint64)
            self.node_vals = np.empty((Tn, 9), np.float64)
            self.abd_body = np.empty(n_abd, np.int32)
            self.jac36 = np.empty((n_abd, 36), np.float64)
            self.pinned = np.empty(self.n_blocks, np.uint8)
            self.rest_edges = np.empty((ne, 2), np.int32)
            L.adipc_scene_copy(handle, ptr(self.keys), ptr(self.vals), ptr(self.node_keys), ptr(self.node_vals),
                               ptr(self.abd_body), ptr(self.jac36), ptr(self.pinned), ptr(self.rest_edges))
            ms, mat = np.zeros(2, np.int64), np.zeros(2)
            L.adipc_scene_mesh_sizes(handle, ptr(ms), ptr(mat))
            self.verts = np.empty((int(ms[0]), 3))
            self.tets = np.empty((int(ms[1]), 4), np.int32)
            self.mass = np.empty(int(ms[0]))
            self.mu, self.lam = float(mat[0]), float(mat[1])
            L.adipc_scene_copy_mesh(handle, ptr(self.verts), ptr(self.tets), ptr(self.mass))
        finally:
            L.adipc_scene_free(handle)


def fem_box(nx, ny, nz, sx=1.0, sy=1.0, sz=1.0, E=1e8, nu=0.3, rho=1000.0, dt=0.01, pin_x0=True, jitter=0.0,
            seed=5) -> Scene:
    """make_box_tets + first-Newton stable Neo-Hookean matrix (cfg1, cfg5, stiff beam);
    jitter > 0 moves every vertex by jitter * h * U(-1, 1) (mt19937(seed))."""
    return Scene(lib().adipc_scene_fem_box(nx, ny, nz, sx, sy, sz, E, nu, rho, dt, int(pin_x0), float(jitter), seed))


def cloth(nx=224, ny=224, sx=1.0, sy=1.0, seed=2) -> Scene:
    """cfg2: make_grid cloth with triangle + hinge stencils, two pinned corners."""
    return Scene(lib().adipc_scene_cloth(nx, ny, sx, sy, seed))


def abd_stack(bx=10, by=5, bz=10, seed=3) -> Scene:
    """cfg3: 500 affine bodies with seeded PSD contact stencils."""
    return Scene(lib().adipc_scene_abd_stack(bx, by, bz, seed))


def hybrid(n_soft=4, soft_res=20, n_gears=40, gear_res=8, stencils_per_pair=1250, E=1e5, seed=4) -> Scene:
    """cfg4: FEM blocks (Young's modulus E) + ABD gears (kappa 1e8), seeded
    PSD contact stencils between neighbouring objects (FEM-FEM, FEM-ABD,
    ABD-ABD pairs) feeding two_level_abd_reduce."""
    return Scene(lib().adipc_scene_hybrid(n_soft, soft_res, n_gears, gear_res, stencils_per_pair, float(E), seed))


def ballistic_direction(sc: Scene, dt: float = 0.01, g=(0.0, -9.81, 0.0)) -> np.ndarray:
    """x* for b = A x*: every FEM slot and every body translation moved by
    dt^2 g, affine parts unchanged (the free-fall displacement of one step)."""
    x = np.zeros((sc.n_blocks, 3))
    x[: sc.n_fem] = np.asarray(g, np.float64) * dt * dt
    for b in range(sc.n_bodies):
        x[sc.n_fem + 4 * b] = np.asarray(g, np.float64) * dt * dt
    x[sc.pinned.astype(bool)] = 0.0
    return np.ascontiguousarray(x.reshape(-1))


def tet_rest_data(verts: np.ndarray, tets: np.ndarray):
    """TetRest per tet (energy/neo_hookean.hpp:13-27) for the producer's input:
    Dm^-1 (9 doubles column-major, cofactors / det like Eigen's fixed 3x3
    inverse) and volume det(Dm) / 6; vectorised."""
    p = verts[tets]  # nt x 4 x 3
    Dm = np.stack([p[:, 1] - p[:, 0], p[:, 2] - p[:, 0], p[:, 3] - p[:, 0]], axis=2)  # nt x 3(row) x 3(col)
    det = np.linalg.det(Dm)
    if not np.all(det > 0):
        raise ValueError("inverted or degenerate rest tet")
    inv = np.linalg.inv(Dm)  # nt x 3 x 3
    inv9 = np.ascontiguousarray(inv.transpose(0, 2, 1).reshape(-1, 9))  # column-major
    return inv9, det / 6.0


def inertial_target(sc: Scene, dt: float = 0.01, g=(0.0, -9.81, 0.0)) -> np.ndarray:
    """x_tilde of the first step from rest: x + dt v + dt^2 g with v = 0
    (TimeStepper's targets, newton.hpp:85-99); pinned vertices stay."""
    xt = sc.verts + (dt * dt) * np.asarray(g, np.float64)[None, :]
    xt[sc.pinned.astype(bool)] = sc.verts[sc.pinned.astype(bool)]
    return np.ascontiguousarray(xt.reshape(-1))


def gravity_rhs(sc: Scene, dt: float = 0.01, g=(0.0, -9.81, 0.0)) -> np.ndarray:
    """Newton right-hand side of the first iteration of a step from rest:
    -grad E = -M (x - x_tilde) = M dt^2 g (incremental_potential.hpp:170-180,
    newton.hpp:85-99), zero on pinned slots (incremental_potential.hpp:253-254).
    FEM-only scenes: the first n_blocks stream entries are the mass diagonals."""
    assert sc.n_bodies == 0, "gravity_rhs is defined for deformable-only scenes"
    mass = sc.vals[: sc.n_blocks, 0]
    b = mass[:, None] * (dt * dt) * np.asarray(g, np.float64)[None, :]
    b[sc.pinned.astype(bool)] = 0.0
    return np.ascontiguousarray(b.reshape(-1))


def cfg5_batch_scene(seed: int) -> Scene:
    """One scene of the cfg5 batch: seeds 5..12, vertices
    jittered by +-1e-3 h; seed 5 is the unjittered headline scene."""
    if seed == 5:
        return CONFIGS["cfg5_stiff_box"]()
    return fem_box(68, 68, 68, 1.0, 1.0, 1.0, E=1e8, jitter=1e-3, seed=seed)


CONFIGS = {
    "cfg1_soft_cube": lambda: fem_box(11, 11, 11, 0.1, 0.1, 0.1, E=1e5, pin_x0=False),
    "cfg2_cloth": lambda: cloth(224, 224),
    "cfg3_abd_stack": lambda: abd_stack(10, 5, 10),
    "cfg4_hybrid": lambda: hybrid(),
    # the north star's ~1M-DOF stiff hybrid scene: 8 FEM blocks of 34^3 cells
    # (E = 1e8) + 40 ABD gears, 96 object pairs x 1,100 contact stencils
    "cfg4_hybrid_1m": lambda: hybrid(8, 34, 40, 8, 1100, E=1e8, seed=4),
    "cfg5_stiff_box": lambda: fem_box(68, 68, 68, 1.0, 1.0, 1.0, E=1e8),
    "stiff_beam": lambda: fem_box(34, 11, 11, 0.7, 0.22, 0.22, E=1e8),
}
