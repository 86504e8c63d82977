"""Geometric hybrid scene (bench / test input, not product): soft-but-stiff
FEM blocks in a grid and affine bodies resting on them, every interface a
gap of dhat / 2 — the north star's ~1M-DOF stiff hybrid scene with REAL
contact (the broad phase over the boundary surfaces finds ~100 K active
point-triangle / edge-edge stencils) instead of the seeded stencils of
`cfg4_hybrid_1m`. Restates the reference's mesh generators and scene setup:
make_box_tets (geometry/shapes.hpp:56-76), boundary surfaces and edges
(scene/mesh.hpp:84-95, contact/broad_phase.hpp:22-53), lumped masses
(mesh.hpp:146-160), body Jacobians and reduced masses (mesh.hpp:196-201,
scene.hpp), rest connectivity (newton.hpp:204-241) and the barrier stiffness
heuristic (contact/barrier.hpp:43-48)."""
from __future__ import annotations

import math

import numpy as np

_CUBE = np.array([[0, 1, 3, 7], [0, 3, 2, 7], [0, 2, 6, 7], [0, 6, 4, 7], [0, 4, 5, 7], [0, 5, 1, 7]])


def box_tets(nx, ny, nz, sx, sy, sz):
    """make_box_tets: vertex id (k vy + j) vx + i, six tets per cell."""
    vx, vy, vz = nx + 1, ny + 1, nz + 1
    k, j, i = np.meshgrid(np.arange(vz), np.arange(vy), np.arange(vx), indexing="ij")
    verts = np.stack([sx * i / nx, sy * j / ny, sz * k / nz], axis=-1).reshape(-1, 3)
    ck, cj, ci = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    ci, cj, ck = ci.reshape(-1), cj.reshape(-1), ck.reshape(-1)
    corner = np.stack([((ck + ((b >> 2) & 1)) * vy + cj + ((b >> 1) & 1)) * vx + ci + (b & 1) for b in range(8)], 1)
    tets = corner[:, _CUBE].reshape(-1, 4)
    return verts, tets.astype(np.int32)


def boundary_tris(tets):
    """Faces of the tets that belong to exactly one tet (the boundary)."""
    f = np.concatenate([tets[:, [0, 1, 2]], tets[:, [0, 1, 3]], tets[:, [0, 2, 3]], tets[:, [1, 2, 3]]])
    k = np.sort(f, axis=1).astype(np.int64)
    key = (k[:, 0] << 42) | (k[:, 1] << 21) | k[:, 2]
    _, inv, cnt = np.unique(key, return_inverse=True, return_counts=True)
    return f[cnt[inv] == 1].astype(np.int32)


def unique_pairs(e):
    e = np.sort(e, axis=1).astype(np.int64)
    k = np.unique((e[:, 0] << 32) | e[:, 1])
    return np.stack([k >> 32, k & 0xFFFFFFFF], 1).astype(np.int32)


def edges_of(tris):
    return unique_pairs(np.concatenate([tris[:, [0, 1]], tris[:, [1, 2]], tris[:, [2, 0]]]))


def lumped_mass(verts, tets, rho):
    p = verts[tets]
    vol = np.abs(np.linalg.det(np.stack([p[:, 1] - p[:, 0], p[:, 2] - p[:, 0], p[:, 3] - p[:, 0]], 2))) / 6
    m = np.zeros(len(verts))
    np.add.at(m, tets.reshape(-1), np.repeat(rho * vol / 4, 4))
    return m


def jacobian36(rest):
    """abd_jacobian (mesh.hpp:196-201): J = [I | diag rows x_bar^T], 3 x 12 column-major."""
    n = len(rest)
    J = np.zeros((n, 12, 3))
    for r in range(3):
        J[:, r, r] = 1.0
        for k in range(3):
            J[:, 3 + 3 * r + k, r] = rest[:, k]
    return J.reshape(n, 36)


def reduced_mass(rest, mass):
    J = jacobian36(rest).reshape(-1, 12, 3)  # [node][col][row]
    return np.einsum("n,nci,ndi->cd", mass, J, J)


def barrier_stiffness(avg_mass, dt, dhat, scale=1.0):
    """initial_barrier_stiffness (barrier.hpp:43-48) with its curvature helper (:35-39)."""
    def b1(s, sh):
        r = s - sh
        return -(2 * r * math.log(s / sh) + r * r / s)

    def b2(s, sh):
        r = s - sh
        return -(2 * math.log(s / sh) + 4 * r / s - r * r / (s * s))

    d = dhat / 2
    s, sh = d * d, dhat * dhat
    unit = abs(4 * s * b2(s, sh) + 2 * b1(s, sh))
    return scale * (avg_mass / (dt * dt)) / unit


class GeomHybrid:
    """Arrays of the geometric hybrid scene (see the module docstring):
    FEM mesh (verts, tets, mass, mu, lam) over slots [0, n_fem); bodies
    (q, q_tilde, reduced_mass, kappa, volume) on slots n_fem + 4 b ..;
    contact-node universe (FEM vertices, then body vertices: abd_body,
    jac36); contact surface (surf_verts, edges, tris as nodes); rest_edges;
    x, x_tilde (the first Newton iteration of a step from rest). One solid
    mesh (all blocks share the material), rest data from tet_rest_data."""

    def __init__(self, grid=(2, 2, 2), res=34, size=0.2, bodies=(5, 5), body_res=2, body_size=0.05, dhat=1e-3,
                 E=1e8, nu=0.3, rho=1000.0, kappa_abd=1e8, dt=0.01, g=(0.0, -9.81, 0.0)):
        gap = 0.5 * dhat
        V, T, S, M = [], [], [], []
        off = 0
        h = size / res
        v0, t0 = box_tets(res, res, res, size, size, size)
        bt0, m0 = boundary_tris(t0), lumped_mass(v0, t0, rho)
        for bz in range(grid[2]):
            for by in range(grid[1]):
                for bx in range(grid[0]):
                    # tangential offsets of (0.4, 0.1) cells across every interface:
                    # opposing faces are not vertex-aligned (no coincident parallel
                    # edges; their diagonals stay > dhat apart)
                    shift = h * np.array([0.1 * by + 0.4 * bz, 0.4 * bx + 0.1 * bz, 0.1 * bx + 0.4 * by])
                    V.append(v0 + np.array([bx, by, bz]) * (size + gap) + shift)
                    T.append(t0 + off)
                    S.append(bt0 + off)
                    M.append(m0)
                    off += len(v0)
        self.verts = np.concatenate(V)
        self.tets = np.concatenate(T).astype(np.int32)
        self.n_fem = len(self.verts)
        self.mass = np.concatenate(M)
        from . import tet_rest_data

        self.rest_inv9, self.rest_volume = tet_rest_data(self.verts, self.tets)
        self.tet_begin = np.array([0, len(self.tets)], np.int64)
        self.mu, self.lam = E / (2 * (1 + nu)), E * nu / ((1 + nu) * (1 - 2 * nu))
        self.dt = dt
        top = self.verts[:, 1].max()
        span_x = grid[0] * size + (grid[0] - 1) * gap
        span_z = grid[2] * size + (grid[2] - 1) * gap
        bt_all, body_of, rest_all, ms, vols, bmass = [], [], [], [], [], []
        self.body_tets = []  # local tets of each body (the reference builds bodies from rest + tets)
        node = self.n_fem
        vb0, tb0 = box_tets(body_res, body_res, body_res, body_size, body_size, body_size)
        btb0 = boundary_tris(tb0)
        nb = 0
        # bodies side by side (gap apart: body-body contacts too), centred on the top face
        pitch = body_size + gap
        x0 = 0.5 * (span_x - bodies[0] * pitch + gap)
        z0 = 0.5 * (span_z - bodies[1] * pitch + gap)
        for iz in range(bodies[1]):
            for ix in range(bodies[0]):
                v, t = vb0 + np.array([x0 + ix * pitch, top + gap, z0 + iz * pitch]), tb0
                m = lumped_mass(v, t, rho)
                bmass.append(m)
                bt_all.append(btb0 + node)
                rest_all.append(v)
                self.body_tets.append(tb0)
                body_of.append(np.full(len(v), nb, np.int32))
                ms.append(reduced_mass(v, m))
                p = v[t]
                vols.append(float(np.sum(np.abs(np.linalg.det(np.stack([p[:, 1] - p[:, 0], p[:, 2] - p[:, 0],
                                                                         p[:, 3] - p[:, 0]], 2))) / 6)))
                node += len(v)
                nb += 1
        self.n_bodies = nb
        self.n_blocks = self.n_fem + 4 * nb
        self.abd_rest = np.concatenate(rest_all)
        self.body_rest = rest_all
        self.E, self.nu, self.rho = E, nu, rho
        self.abd_body = np.concatenate(body_of)
        self.jac36 = jacobian36(self.abd_rest)
        self.reduced_mass = np.stack(ms)
        self.kappa_abd = np.full(nb, kappa_abd)
        self.body_volume = np.array(vols)
        self.q = np.tile(np.array([0, 0, 0, 1, 0, 0, 0, 1, 0, 0, 0, 1.0]), (nb, 1))
        gv = np.asarray(g, np.float64)
        self.q_tilde = self.q.copy()
        self.q_tilde[:, :3] += dt * dt * gv
        self.x = self.verts.copy()
        self.x_tilde = self.verts + dt * dt * gv
        self.dt2 = dt * dt
        tris = np.concatenate(S + bt_all).astype(np.int32)
        self.tris = tris
        self.edges = edges_of(tris)
        self.surf_verts = np.unique(tris).astype(np.int32)
        self.n_nodes = node
        self.dhat = dhat
        all_mass = np.concatenate([self.mass] + bmass)
        self.kappa = barrier_stiffness(float(np.mean(all_mass)), dt, dhat)
        # rest connectivity (newton.hpp:204-241): element cliques + 4-slot body cliques
        pairs = [self.tets[:, [a, b]] for a in range(4) for b in range(a + 1, 4)]
        for b in range(nb):
            base = self.n_fem + 4 * b
            pairs.append(np.array([[base + a, base + c] for a in range(4) for c in range(a + 1, 4)], np.int32))
        self.rest_edges = unique_pairs(np.concatenate(pairs))
        self.pinned = np.zeros(self.n_blocks, np.uint8)

    def state(self):
        """The block-numbered state: FEM x, then q per body (12 dofs)."""
        return np.concatenate([self.x.reshape(-1), self.q.reshape(-1)])

    def node_positions(self):
        """contact_node_positions (scene.hpp): FEM x, body nodes A x_bar + p."""
        A = self.q[self.abd_body, 3:].reshape(-1, 3, 3)
        p = self.q[self.abd_body, :3]
        return np.concatenate([self.x, np.einsum("nij,nj->ni", A, self.abd_rest) + p])
