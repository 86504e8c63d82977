"""The device IncrementalPotential against the reference's OWN
IncrementalPotential::assemble (oracle/_ref: the reference's scene, broad
phase, contact / ground / friction terms, element and body stencils,
two-level reduction, filter, sort and reduction, compiled in place) on the
scene data the reference derives itself (Scene::finalize masses and rest data,
body reduced masses, make_dof_map, build_contact_surface): the matrix pattern
bitwise, blocks to 1e-9 of sqrt(|D_r||D_c|), gradient 1e-10, value 1e-11 —
plain, with the ground, with friction frozen at the step start, and with a
cloth (shell membrane + hinges) in the scene's mesh order."""
import numpy as np
import pytest
import torch

import oracle_py as O
from paper_2411_06224_b200.context import Context
from paper_2411_06224_b200.potential import IncrementalPotential
from scenegen.geom import GeomHybrid
from test_gpu_potential import assert_matrix_close

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not O.reference_available(), reason="oracle/_ref not built")]
GROUND = ((0.0, 1.0, 0.0), -0.0004)


@pytest.fixture(scope="module")
def ctx():
    c = Context(0)
    yield c
    c.close()


def build(ctx, g, ground):
    rs = O.RefScene([{"rest": g.verts, "tets": g.tets, "youngs": g.E, "poisson": g.nu, "density": g.rho}],
                    [{"rest": r, "tets": t, "kappa": float(k), "density": g.rho}
                     for r, t, k in zip(g.body_rest, g.body_tets, g.kappa_abd)], g.dt, ground=ground)
    d = rs.data
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    mesh = {"mass": t(d["mass"]), "tets": t(d["tets"]), "rest_inv9": t(d["rest_inv9"]),
            "rest_volume": t(d["rest_volume"]), "tet_begin": d["tet_begin"], "mu": list(d["mu"]),
            "lam": list(d["lam"]),
            "bodies": {"reduced_mass": t(d["reduced_mass"]), "kappa": t(g.kappa_abd), "volume": t(d["body_volume"])}}
    ip = IncrementalPotential(ctx, mesh, {"verts": t(d["surf_verts"]), "edges": t(d["edges"]), "tris": t(d["tris"])},
                              {"n_fem": rs.n_fem, "abd_body": t(d["abd_body"]), "jac36": t(d["jac36"])}, g.dt,
                              pinned=t(np.zeros(rs.n_blocks, np.uint8)))
    ip.set_targets(t(g.x_tilde.reshape(-1)), t(g.q_tilde))
    ip.set_contact(g.dhat, g.kappa)
    if ground is not None:
        ip.set_ground(*ground)
    return rs, ip, t


@pytest.mark.parametrize("with_ground,with_friction", [(False, False), (True, False), (True, True)])
def test_device_potential_equals_reference(ctx, with_ground, with_friction):
    g = GeomHybrid(grid=(2, 2, 1), res=4, bodies=(3, 2), body_res=1)
    rs, ip, t = build(ctx, g, GROUND if with_ground else None)
    rng = np.random.default_rng(11)
    x0 = g.x + rng.normal(0, 3e-5, g.x.shape)
    q0 = g.q + rng.normal(0, 3e-6, g.q.shape)
    if with_friction:
        mu, eps = 0.4, 1e-5
        n_ref = rs.begin_friction(x0, q0, g.dhat, g.kappa, mu, eps)
        n_dev = ip.begin_friction(t(np.concatenate([x0.reshape(-1), q0.reshape(-1)])), mu, eps)
        assert n_dev == n_ref > 0
    x1 = x0 + rng.normal(0, 2e-5, g.x.shape)
    q1 = q0 + rng.normal(0, 2e-6, g.q.shape)
    val, grad, rows, cols, blocks = rs.assemble(x1, q1, g.x_tilde, g.q_tilde, g.dhat, g.kappa)
    dval, dgrad = ip.assemble(t(np.concatenate([x1.reshape(-1), q1.reshape(-1)])))
    n, drows, dcols, dblocks = ctx.copy_matrix()
    assert n == rs.n_blocks and ip.last["n_pt"] > 0 and ip.last["n_ee"] > 0
    assert_matrix_close(drows, dcols, dblocks, rows, cols, blocks, 1e-9)
    assert np.linalg.norm(dgrad.cpu().numpy() - grad) <= 1e-10 * np.linalg.norm(grad)
    assert abs(dval - val) <= 1e-11 * abs(val)


def test_device_potential_with_a_shell_equals_reference(ctx):
    """A cloth resting dhat / 2 above a stiff block plus an affine body: the
    shell's membrane and hinge stencils join the element stream in the
    reference's mesh order (solid, then shell), the cloth's vertices join the
    contact surface; device IncrementalPotential vs the reference's own."""
    from contact_cases import make_grid
    from scenegen.geom import box_tets

    bv, bt = box_tets(3, 3, 3, 0.2, 0.2, 0.2)
    cv, ct = make_grid(9, 9, 0.18, 0.18)
    dhat = 1e-3
    cloth = np.stack([cv[:, 0] + 0.01, np.full(len(cv), 0.2 + 0.5 * dhat), cv[:, 1] + 0.01], axis=1)
    rv, rt = box_tets(1, 1, 1, 0.05, 0.05, 0.05)
    rv = rv + np.array([0.5, 0.0, 0.0])
    shell = {"rest": cloth, "tris": ct, "density": 200.0, "thickness": 1e-3, "stretch": 5e4, "strain_limit": 5e6,
             "shear_fraction": 0.3, "bending": 1e-6}
    dt = 0.01
    rs = O.RefScene([{"rest": bv, "tets": bt, "youngs": 1e8, "poisson": 0.3, "density": 1000.0}],
                    [{"rest": rv, "tets": rt, "kappa": 1e8, "density": 1000.0}], dt, shells=[shell])
    d = rs.data
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    sh = d["shells"]
    mesh = {"mass": t(d["mass"]), "tets": t(d["tets"]), "rest_inv9": t(d["rest_inv9"]),
            "rest_volume": t(d["rest_volume"]), "tet_begin": d["tet_begin"], "mu": list(d["mu"]),
            "lam": list(d["lam"]), "mesh_kind": d["mesh_kind"],
            "shells": {"tris": t(sh["tris"]), "tri_rest": t(sh["tri_rest"]), "hinges": t(sh["hinges"]),
                       "hinge_rest": t(sh["hinge_rest"]), "tri_begin": sh["tri_begin"],
                       "hinge_begin": sh["hinge_begin"], "material": sh["material"]},
            "bodies": {"reduced_mass": t(d["reduced_mass"]), "kappa": t(np.array([1e8])),
                       "volume": t(d["body_volume"])}}
    ip = IncrementalPotential(ctx, mesh, {"verts": t(d["surf_verts"]), "edges": t(d["edges"]), "tris": t(d["tris"])},
                              {"n_fem": rs.n_fem, "abd_body": t(d["abd_body"]), "jac36": t(d["jac36"])}, dt)
    rest_x = np.concatenate([bv, cloth])
    gv = np.array([0.0, -9.81, 0.0])
    x_tilde = rest_x + dt * dt * gv
    q0 = np.array([[0, 0, 0, 1, 0, 0, 0, 1, 0, 0, 0, 1.0]])
    q_tilde = q0.copy()
    q_tilde[:, :3] += dt * dt * gv
    kappa = 1e5
    ip.set_targets(t(x_tilde.reshape(-1)), t(q_tilde))
    ip.set_contact(dhat, kappa)
    rng = np.random.default_rng(4)
    x1 = rest_x + rng.normal(0, 2e-5, rest_x.shape)
    q1 = q0 + rng.normal(0, 2e-6, q0.shape)
    val, grad, rows, cols, blocks = rs.assemble(x1, q1, x_tilde, q_tilde, dhat, kappa)
    dval, dgrad = ip.assemble(t(np.concatenate([x1.reshape(-1), q1.reshape(-1)])))
    n, drows, dcols, dblocks = ctx.copy_matrix()
    assert ip.last["n_pt"] > 0 and ip.last["n_ee"] > 0
    assert_matrix_close(drows, dcols, dblocks, rows, cols, blocks, 1e-9)
    assert np.linalg.norm(dgrad.cpu().numpy() - grad) <= 1e-10 * np.linalg.norm(grad)
    # the value sums ~10^3 stencil energies of very different sizes in
    # another order (CTA sums + fp64 atomics): 1e-10
    assert abs(dval - val) <= 1e-10 * abs(val)
