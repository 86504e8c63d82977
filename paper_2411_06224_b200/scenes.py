"""Synthetic benchmark scenes (BASELINE.json configs 1-5) from
libadipc_scenes.so — see csrc/scenes.cpp for what each generator restates."""
from __future__ import annotations

import numpy as np

from . import _lib
from ._lib import ptr


class Scene:
    """Triplet streams + pins + rest connectivity of one synthetic scene.

    keys/vals:            DOF stream before contact tiles (emission order)
    node_keys/node_vals:  contact node-pair stream (two-level ABD input)
    abd_body/jac36:       DofMap of the contact-node universe
    pinned:               uint8 per block slot
    rest_edges:           int32 [E, 2] (newton.hpp:204-241), the L0 partition input
    """

    def __init__(self, handle):
        L = _lib.scenes()
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
        finally:
            L.adipc_scene_free(handle)


def fem_box(nx, ny, nz, sx=1.0, sy=1.0, sz=1.0, E=1e8, nu=0.3, rho=1000.0, dt=0.01, pin_x0=True) -> Scene:
    """make_box_tets + first-Newton stable Neo-Hookean matrix (cfg1, cfg5, stiff beam)."""
    return Scene(_lib.scenes().adipc_scene_fem_box(nx, ny, nz, sx, sy, sz, E, nu, rho, dt, int(pin_x0)))


def cloth(nx=224, ny=224, sx=1.0, sy=1.0, seed=2) -> Scene:
    """cfg2: make_grid cloth with triangle + hinge stencils, two pinned corners."""
    return Scene(_lib.scenes().adipc_scene_cloth(nx, ny, sx, sy, seed))


def abd_stack(bx=10, by=5, bz=10, seed=3) -> Scene:
    """cfg3: 500 affine bodies with seeded PSD contact stencils."""
    return Scene(_lib.scenes().adipc_scene_abd_stack(bx, by, bz, seed))


def hybrid(n_soft=4, soft_res=20, n_gears=40, gear_res=8, stencils_per_pair=1250, seed=4) -> Scene:
    """cfg4: soft FEM blocks + ABD gears, ~100K contact stencils."""
    return Scene(_lib.scenes().adipc_scene_hybrid(n_soft, soft_res, n_gears, gear_res, stencils_per_pair, seed))


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


CONFIGS = {
    "cfg1_soft_cube": lambda: fem_box(11, 11, 11, 0.1, 0.1, 0.1, E=1e5, pin_x0=False),
    "cfg2_cloth": lambda: cloth(224, 224),
    "cfg3_abd_stack": lambda: abd_stack(10, 5, 10),
    "cfg4_hybrid": lambda: hybrid(),
    "cfg5_stiff_box": lambda: fem_box(68, 68, 68, 1.0, 1.0, 1.0, E=1e8),
    "stiff_beam": lambda: fem_box(34, 11, 11, 0.7, 0.22, 0.22, E=1e8),
}
