"""The oracle's IncrementalPotential::assemble composition (oracle_py.ip_assemble,
incremental_potential.hpp:162-258) on the geometric hybrid scene: its
gradient — element, body and lifted contact parts together
(:395-403, J^T for affine-body nodes) — is the derivative of its value
(central differences along random directions), the contact part is
present (FEM-FEM, FEM-body and body-body stencils all occur), and the
restated pieces agree with the reference's own compiled code where it
exports them (oracle/_ref)."""
import numpy as np
import pytest

import oracle_py as O
from scenegen.geom import GeomHybrid

DET = O.ExecPolicy(deterministic=True)


@pytest.fixture(scope="module")
def scene():
    return GeomHybrid(grid=(2, 1, 1), res=3, bodies=(2, 2), body_res=1)


def test_gradient_is_derivative_of_value(scene):
    g = scene
    rng = np.random.default_rng(1)
    # off the aligned rest configuration (parallel edges there make the
    # distance a non-smooth min over features)
    s = g.state() + rng.normal(0, 5e-5, 3 * g.n_blocks)
    val, grad, *_ = O.ip_assemble(g, s, DET)
    for _ in range(3):
        d = rng.normal(0, 1, 3 * g.n_blocks)
        d *= 1e-6 / np.abs(d).max()
        vp = O.ip_assemble(g, s + d, DET)[0]
        vm = O.ip_assemble(g, s - d, DET)[0]
        fd = (vp - vm) / 2
        assert fd == pytest.approx(float(grad @ d), rel=1e-3)


def test_contact_kinds_present(scene):
    g = scene
    pos = O.node_displacements(g.state(), g.n_fem, g.abd_body, g.jac36).reshape(-1, 3)
    pt, ee = O.find_candidates(pos, g.surf_verts, g.edges, g.tris, g.dhat)
    st = np.r_[np.c_[g.surf_verts[pt[:, 0]], g.tris[pt[:, 1]]], np.c_[g.edges[ee[:, 0]], g.edges[ee[:, 1]]]]
    owner = np.where(st < g.n_fem, -1, g.abd_body[np.maximum(st - g.n_fem, 0)])
    box = np.where(st < g.n_fem, st // ((3 + 1) ** 3), -1)
    fem_fem = np.any((owner == -1).all(1) & (box.min(1) != box.max(1)))
    fem_body = np.any((owner == -1).any(1) & (owner >= 0).any(1))
    body_body = np.any((owner >= 0).all(1) & (owner.min(1) != owner.max(1)))
    assert fem_fem and fem_body and body_body


def test_lift_node_grad_restated():
    """FEM nodes copy-add; a body node adds J^T g (J = [I | x_bar (x) I])."""
    rng = np.random.default_rng(2)
    n_fem, rest = 3, rng.normal(0, 1, (4, 3))
    body = np.array([0, 1, 1, 0], np.int32)
    jac = np.stack([O.abd_jacobian(r) for r in rest])
    ng = rng.normal(0, 1, 3 * (n_fem + 4))
    grad = O.lift_node_grad(ng, n_fem, body, jac, np.zeros(3 * (n_fem + 8)))
    want = np.zeros(3 * (n_fem + 8))
    want[:9] = ng[:9]
    for a in range(4):
        J = np.zeros((3, 12))
        J[:, :3] = np.eye(3)
        for r in range(3):
            J[r, 3 + 3 * r: 6 + 3 * r] = rest[a]
        s = 3 * (n_fem + 4 * body[a])
        want[s:s + 12] += J.T @ ng[3 * (n_fem + a): 3 * (n_fem + a) + 3]
    assert np.allclose(grad, want, rtol=1e-14, atol=1e-14)


def test_pieces_equal_reference(scene):
    """ip_assemble through the reference's compiled element, contact, broad
    phase, two-level, sort and reduction code equals the restatement."""
    if not O.reference_available():
        pytest.skip("oracle/_ref not built")
    g = scene
    s = g.state() + np.random.default_rng(3).normal(0, 2e-5, 3 * g.n_blocks)
    a = O.ip_assemble(g, s, DET)
    with O.use_backend("reference"):
        b = O.ip_assemble(g, s, DET)
    assert np.array_equal(a[2], b[2]) and np.array_equal(a[3], b[3]) and a[5] == b[5]
    scale = np.abs(b[4]).max()
    assert np.abs(a[4] - b[4]).max() <= 1e-12 * scale
    assert np.linalg.norm(a[1] - b[1]) <= 1e-13 * np.linalg.norm(b[1])
    assert a[0] == pytest.approx(b[0], rel=1e-13)


def ref_scene(g, ground=None):
    return O.RefScene([{"rest": g.verts, "tets": g.tets, "youngs": g.E, "poisson": g.nu, "density": g.rho}],
                      [{"rest": r, "tets": t, "kappa": float(k), "density": g.rho}
                       for r, t, k in zip(g.body_rest, g.body_tets, g.kappa_abd)], g.dt, ground=ground)


def scene_view(g, rs):
    """The oracle composition's scene from the reference's own derived data."""
    import types

    d = rs.data
    return types.SimpleNamespace(
        n_fem=rs.n_fem, n_bodies=rs.n_bodies, n_blocks=rs.n_blocks, q_tilde=g.q_tilde,
        reduced_mass=d["reduced_mass"].reshape(-1, 12, 12).transpose(0, 2, 1), kappa_abd=g.kappa_abd,
        body_volume=d["body_volume"], dt=g.dt, x_tilde=g.x_tilde, mass=d["mass"], tet_begin=d["tet_begin"],
        mu=d["mu"][0], lam=d["lam"][0], tets=d["tets"], rest_inv9=d["rest_inv9"], rest_volume=d["rest_volume"],
        abd_body=d["abd_body"], jac36=d["jac36"], surf_verts=d["surf_verts"], edges=d["edges"], tris=d["tris"],
        dhat=g.dhat, kappa=g.kappa, pinned=np.zeros(rs.n_blocks, np.uint8))


@pytest.mark.parametrize("with_ground,with_friction", [(False, False), (True, False), (True, True)])
def test_composition_equals_reference_incremental_potential(with_ground, with_friction):
    """The oracle's ip_assemble against the reference's OWN IncrementalPotential::
    assemble (oracle/_ref: Scene::finalize, make_dof_map,
    build_contact_surface, the proximity broad phase, the contact, ground and
    friction terms, two_level_abd_reduce, filter, sort, reduce) on the scene
    data the reference derives: pattern bitwise, blocks / gradient / value to
    1e-14."""
    if not O.reference_available():
        pytest.skip("oracle/_ref not built")
    g = GeomHybrid(grid=(2, 1, 1), res=3, bodies=(2, 2), body_res=1)
    ground = ((0.0, 1.0, 0.0), -0.0004) if with_ground else None
    rs = ref_scene(g, ground)
    sc = scene_view(g, rs)
    rng = np.random.default_rng(7)
    x0 = g.x + rng.normal(0, 3e-5, g.x.shape)
    q0 = g.q + rng.normal(0, 3e-6, g.q.shape)
    kw = {"ground": ground}
    if with_friction:
        mu, eps = 0.4, 1e-5
        n = rs.begin_friction(x0, q0, g.dhat, g.kappa, mu, eps)
        s0 = np.concatenate([x0.reshape(-1), q0.reshape(-1)])
        pos0 = O.contact_node_positions(s0, rs.n_fem, sc.abd_body, sc.jac36)
        fr = O.build_friction_constraints(pos0, sc.surf_verts, sc.edges, sc.tris, g.dhat, g.kappa, ground)
        assert len(fr["n"]) == n > 0
        kw.update(friction=fr, fr_base=pos0, mu=mu, fr_eps=eps)
    x1 = x0 + rng.normal(0, 2e-5, g.x.shape)
    q1 = q0 + rng.normal(0, 2e-6, g.q.shape)
    val, grad, rows, cols, blocks = rs.assemble(x1, q1, g.x_tilde, g.q_tilde, g.dhat, g.kappa)
    s1 = np.concatenate([x1.reshape(-1), q1.reshape(-1)])
    ov, og, orow, ocol, oblk, cnt = O.ip_assemble(sc, s1, DET, **kw)
    assert cnt["n_pt"] > 0 and cnt["n_ee"] > 0
    assert np.array_equal(rows, orow) and np.array_equal(cols, ocol)
    assert np.abs(blocks - oblk).max() <= 1e-14 * np.abs(oblk).max()
    assert np.linalg.norm(grad - og) <= 1e-14 * np.linalg.norm(og)
    assert abs(val - ov) <= 1e-13 * abs(ov)
