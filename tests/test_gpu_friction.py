"""GPU parity of the device friction-constraint builder
(adipc_gpu_friction_constraints_device; friction.hpp:95-149) against the
oracle (pinned bitwise to the reference's compiled builder in
test_oracle_friction.py) on the same candidate stencils — nodes, counts,
coefficients and tangent frames bitwise, the lagged normal forces to 1e-14 —
and of a frictional step through the device IncrementalPotential: ground
barrier + friction frozen at the step start (begin_friction, newton.hpp:104-113),
then assemble at a moved state, against the oracle's composition."""
import numpy as np
import pytest
import torch

import oracle_py as O
from paper_2411_06224_b200.context import Context
from scenegen.geom import GeomHybrid
from test_gpu_potential import assert_matrix_close, device_potential

pytestmark = pytest.mark.gpu
DET = O.ExecPolicy(deterministic=True)
GROUND = ((0.0, 1.0, 0.0), -0.0004)


@pytest.fixture(scope="module")
def ctx():
    c = Context(0)
    yield c
    c.close()


@pytest.fixture(scope="module")
def scene():
    return GeomHybrid(grid=(2, 1, 1), res=4, bodies=(2, 2), body_res=1)


def test_builder_matches_oracle(ctx, scene):
    g = scene
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    rng = np.random.default_rng(5)
    for trial in range(3):
        pos = g.node_positions() + rng.normal(0, 5e-5, (g.n_nodes, 3))
        ground = GROUND if trial != 1 else None
        pt, ee = O.find_candidates(pos, g.surf_verts, g.edges, g.tris, g.dhat)
        pts = np.c_[g.surf_verts[pt[:, 0]], g.tris[pt[:, 1]]].astype(np.int32)
        ees = np.c_[g.edges[ee[:, 0]], g.edges[ee[:, 1]]].astype(np.int32)
        ci = O.ContactInput(pos, pts, ees, dhat=g.dhat, kappa=g.kappa, ground=ground, surf_verts=g.surf_verts)
        want = O.friction_constraints(ci)
        got = ctx.friction_constraints({"pos": t(pos), "pt": t(pts), "ee": t(ees), "dhat": g.dhat, "kappa": g.kappa,
                                        "ground": ground, "surf_verts": t(g.surf_verts)})
        assert len(want["n"]) > 0 and got["fr_n"].numel() == len(want["n"])
        assert np.array_equal(got["fr_n"].cpu().numpy(), want["n"])
        assert np.array_equal(got["fr_nodes"].cpu().numpy(), want["nodes"])
        for k_dev, k_or in (("fr_coeff", "coeff"), ("fr_t1", "t1"), ("fr_t2", "t2")):
            assert np.array_equal(got[k_dev].cpu().numpy(), want[k_or]), k_dev
        lam = got["fr_lambda"].cpu().numpy()
        assert np.all(np.abs(lam - want["lam"]) <= 1e-14 * np.abs(want["lam"]))


def test_frictional_step_matches_oracle(ctx, scene):
    g = scene
    ip, t = device_potential(ctx, g)
    ip.set_ground(*GROUND)
    rng = np.random.default_rng(6)
    s0 = g.state() + rng.normal(0, 3e-5, 3 * g.n_blocks)
    mu, eps = 0.4, 1e-5
    n_fr = ip.begin_friction(t(s0), mu, eps)
    pos0 = O.contact_node_positions(s0, g.n_fem, g.abd_body, g.jac36)
    fr = O.build_friction_constraints(pos0, g.surf_verts, g.edges, g.tris, g.dhat, g.kappa, GROUND)
    assert n_fr == len(fr["n"]) and n_fr > 0
    s1 = s0 + rng.normal(0, 2e-5, 3 * g.n_blocks)
    val, grad = ip.assemble(t(s1))
    ov, og, orow, ocol, oblk, _ = O.ip_assemble(g, s1, DET, ground=GROUND, friction=fr, fr_base=pos0, mu=mu,
                                                fr_eps=eps)
    n, rows, cols, blocks = ctx.copy_matrix()
    assert_matrix_close(rows, cols, blocks, orow, ocol, oblk, 1e-9)
    assert np.linalg.norm(grad.cpu().numpy() - og) <= 1e-10 * np.linalg.norm(og)
    # value: sums of many terms in different orders (fp64 REDs, the friction
    # and ground parts added per thread): 1e-11
    assert abs(val - ov) <= 1e-11 * abs(ov)
    assert ip.value(t(s1)) == pytest.approx(val, rel=1e-11)
    # friction contributes: without it the value differs
    ip.clear_friction()
    assert ip.value(t(s1)) != pytest.approx(val, rel=1e-9)
