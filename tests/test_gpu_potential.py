"""GPU parity of the device IncrementalPotential (paper_2411_06224_b200/
potential.py: incremental_potential.hpp:162-258 composed from the C-ABI
producers) against the oracle's composition of the restated pieces
(oracle_py.ip_assemble) on the geometric hybrid scene (scenegen/geom.py:
FEM blocks + affine bodies, every interface dhat / 2 apart, so the broad
phase finds FEM-FEM, FEM-body and body-body stencils): the reduced matrix
pattern bitwise, its blocks to 1e-9 of sqrt(|D_r| |D_c|), the gradient
and the value to 1e-10 / 1e-12, the line-search value, the CCD bound, and
one whole Newton linear solve (cold MAS + PCG on -grad) against the
oracle's MAS + PCG."""
import numpy as np
import pytest
import torch

import oracle_py as O
from paper_2411_06224_b200 import api as P
from paper_2411_06224_b200.context import Context
from paper_2411_06224_b200.potential import IncrementalPotential
from scenegen.geom import GeomHybrid

pytestmark = pytest.mark.gpu
DET = O.ExecPolicy(deterministic=True)
CAP, LEVELS = 16, 4


@pytest.fixture(scope="module")
def ctx():
    c = Context(0)
    yield c
    c.close()


def device_potential(ctx, g):
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    mesh = {"mass": t(g.mass), "tets": t(g.tets), "rest_inv9": t(g.rest_inv9), "rest_volume": t(g.rest_volume),
            "tet_begin": g.tet_begin, "mu": [g.mu], "lam": [g.lam],
            "bodies": {"reduced_mass": t(g.reduced_mass.transpose(0, 2, 1)), "kappa": t(g.kappa_abd),
                       "volume": t(g.body_volume)}}
    surf = {"verts": t(g.surf_verts), "edges": t(g.edges), "tris": t(g.tris)}
    dofs = {"n_fem": g.n_fem, "abd_body": t(g.abd_body), "jac36": t(g.jac36)}
    ip = IncrementalPotential(ctx, mesh, surf, dofs, g.dt, pinned=t(g.pinned))
    ip.set_targets(t(g.x_tilde.reshape(-1)), t(g.q_tilde))
    ip.set_contact(g.dhat, g.kappa)
    return ip, t


def assert_matrix_close(rows, cols, blocks, orow, ocol, oblk, tol):
    assert np.array_equal(rows, orow) and np.array_equal(cols, ocol)
    d = np.zeros(int(orow.max()) + 1)
    diag = orow == ocol
    d[orow[diag]] = np.linalg.norm(oblk[diag], axis=1)
    scale = np.sqrt(d[orow] * d[ocol])
    err = np.linalg.norm(blocks - oblk, axis=1)
    assert np.all(err <= tol * scale), float(np.max(err / scale))


@pytest.fixture(scope="module")
def scene():
    return GeomHybrid(grid=(2, 2, 1), res=5, bodies=(3, 2), body_res=1)


def test_assemble_matches_oracle(ctx, scene):
    g = scene
    ip, t = device_potential(ctx, g)
    rng = np.random.default_rng(4)
    state = g.state() + rng.normal(0, 5e-5, 3 * g.n_blocks) * np.r_[np.ones(3 * g.n_fem), np.tile(
        [1, 1, 1, 0.1, 0.1, 0.1, 0.1, 0.1, 0.1, 0.1, 0.1, 0.1], g.n_bodies)]
    ov, og, orow, ocol, oblk, cnt = O.ip_assemble(g, state, DET)
    assert cnt["n_pt"] > 0 and cnt["n_ee"] > 0 and cnt["contact_tiles"] > 0
    val, grad = ip.assemble(t(state))
    assert ip.last["n_pt"] == cnt["n_pt"] and ip.last["n_ee"] == cnt["n_ee"]
    assert ip.last["node_blocks"] == cnt["node_blocks"]
    n, rows, cols, blocks = ctx.copy_matrix()
    assert n == g.n_blocks
    assert_matrix_close(rows, cols, blocks, orow, ocol, oblk, 1e-9)
    gd = grad.cpu().numpy()
    assert np.linalg.norm(gd - og) <= 1e-10 * np.linalg.norm(og)
    assert abs(val - ov) <= 1e-12 * abs(ov)
    # the line-search value at the same state (:61-159)
    assert ip.value(t(state)) == pytest.approx(val, rel=1e-12)
    # contact terms are present: the same state without contact differs
    assert abs(val - O.ip_fem_assemble(state[:3 * g.n_fem], g.x_tilde, g.mass, g.tet_begin, [g.mu], [g.lam], g.tets,
                                       g.rest_inv9, g.rest_volume, g.dt ** 2, None, True,
                                       {"q": state[3 * g.n_fem:].reshape(-1, 12), "q_tilde": g.q_tilde,
                                        "reduced_mass": g.reduced_mass, "kappa": g.kappa_abd,
                                        "volume": g.body_volume})[0]) > 0


def test_ccd_step_matches_oracle(ctx, scene):
    g = scene
    ip, t = device_potential(ctx, g)
    state = g.state()
    rng = np.random.default_rng(11)
    for s in (1e-4, 1e-3):
        d = rng.normal(0, s, 3 * g.n_blocks)
        a = ip.ccd_step(t(state), t(d))
        pos = O.contact_node_positions(state, g.n_fem, g.abd_body, g.jac36)
        disp = O.node_displacements(d, g.n_fem, g.abd_body, g.jac36).reshape(-1, 3)
        pt, ee = O.find_candidates(pos, g.surf_verts, g.edges, g.tris, g.dhat, disp=disp)
        ci = O.ContactInput(pos, np.c_[g.surf_verts[pt[:, 0]], g.tris[pt[:, 1]]],
                            np.c_[g.edges[ee[:, 0]], g.edges[ee[:, 1]]], dhat=g.dhat, kappa=g.kappa)
        assert a == pytest.approx(O.ccd_step(ci, disp), rel=1e-12, abs=1e-15)
        assert 0 < a <= 1


def test_newton_linear_solve_matches_oracle(ctx, scene):
    """One Newton iteration's linear solve: device assemble -> cold MAS ->
    PCG on -grad, against the oracle's assemble -> Hierarchy + MAS -> PCG:
    iterations within 2 % at the bench tolerance (1e-4), and the direction
    within 1e-6 when both solve to 1e-10 (at 1e-4 the two stopping points
    differ by the contact-stiff system's conditioning times the tolerance)."""
    g = scene
    ip, t = device_potential(ctx, g)
    state = g.state()
    l0 = P.partition_block_graph(g.n_blocks, g.rest_edges, CAP)
    ctx.set_level0_partition(l0.part_of, l0.n_parts, CAP, LEVELS)
    _, grad = ip.assemble(t(state))
    ctx.build_preconditioner()
    b = -grad
    x = torch.empty_like(b)
    _, res = ctx.pcg(b, 1e-4, 250, 100000, x=x)
    ov, og, orow, ocol, oblk, _ = O.ip_assemble(g, state, DET)
    A = O.Matrix(g.n_blocks, orow, ocol, oblk)
    H = O.Hierarchy(l0.part_of, l0.n_parts, CAP, O.block_edges(orow, ocol), LEVELS)
    xo, ro = O.pcg_solve(A, -og, O.MasPreconditioner(A, H), 1e-4, 250, 100000, DET)
    assert res.converged and ro["converged"]
    assert abs(res.iters - ro["iters"]) <= max(1, 0.02 * ro["iters"])
    _, res = ctx.pcg(b, 1e-10, 250, 100000, x=x)
    xo, ro = O.pcg_solve(A, -og, O.MasPreconditioner(A, H), 1e-10, 250, 100000, DET)
    assert res.converged and ro["converged"]
    assert np.linalg.norm(x.cpu().numpy() - xo) <= 1e-6 * np.linalg.norm(xo)


def test_potential_without_contact_or_bodies(ctx):
    """Edge cases of the composition: contact disabled (dhat = 0: no broad
    phase, an empty node stream into the two-level assembly) and a scene with
    no affine bodies: the result is the element / inertia assembly alone,
    against the oracle's ip_fem_assemble + filter + sort + reduce."""
    g = GeomHybrid(grid=(1, 1, 1), res=4, bodies=(1, 1), body_res=1)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    mesh = {"mass": t(g.mass), "tets": t(g.tets), "rest_inv9": t(g.rest_inv9), "rest_volume": t(g.rest_volume),
            "tet_begin": g.tet_begin, "mu": [g.mu], "lam": [g.lam]}
    ip = IncrementalPotential(ctx, mesh, {"verts": t(g.surf_verts[:0]), "edges": t(g.edges[:0]),
                                          "tris": t(g.tris[:0])}, {"n_fem": g.n_fem}, g.dt)
    ip.set_targets(t(g.x_tilde.reshape(-1)))
    x = g.x.reshape(-1) + np.random.default_rng(3).normal(0, 1e-4, 3 * g.n_fem)
    val, grad = ip.assemble(t(x))
    assert ip.last["n_pt"] == 0 and ip.last["node_blocks"] == 0 and ip.last["contact_tiles"] == 0
    ov, og, keys, vals = O.ip_fem_assemble(x, g.x_tilde, g.mass, g.tet_begin, [g.mu], [g.lam], g.tets, g.rest_inv9,
                                           g.rest_volume, g.dt ** 2)
    sk, sv = O.sort_stream(keys, vals, DET)
    orow, ocol, oblk = O.fast_hash_reduction(sk, sv, g.n_fem, DET)
    n, rows, cols, blocks = ctx.copy_matrix()
    assert_matrix_close(rows, cols, blocks, orow, ocol, oblk, 1e-9)
    assert np.linalg.norm(grad.cpu().numpy() - og) <= 1e-10 * np.linalg.norm(og)
    assert abs(val - ov) <= 1e-12 * abs(ov)
