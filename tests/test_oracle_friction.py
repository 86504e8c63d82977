"""Oracle of the friction-constraint builder (friction.hpp:43-149; contact
frames distance.hpp:226-256) and of the broad phase, pinned to the
reference's OWN compiled code (oracle/_ref: contact/friction.hpp with the
scene and broad-phase headers it includes, compiled against the Eigen
subset): the restated find_candidates equals the reference's
(proximity and swept, pairs and order), the frames and the tangent basis are
bitwise the reference's, and the restated build_friction_constraints
(find_candidates + the restated frame loop) equals the reference's own
build_friction_constraints, ground included, bitwise."""
import numpy as np
import pytest

import oracle_py as O
from contact_cases import layered_surface
from scenegen.geom import GeomHybrid

pytestmark = pytest.mark.skipif(not O.reference_available(), reason="oracle/_ref not built")


@pytest.mark.parametrize("n,swept", [(6, False), (6, True), (30, False), (30, True)])
def test_broad_phase_equals_reference(n, swept):
    pos, verts, edges, tris = layered_surface(n=n, layers=3)
    inflate = 0.11 if n == 6 else 0.03
    disp = np.random.default_rng(n).normal(0, 0.01, pos.shape) if swept else None
    a = O.find_candidates(pos, verts, edges, tris, inflate, disp=disp)
    with O.use_backend("reference"):
        b = O.find_candidates(pos, verts, edges, tris, inflate, disp=disp)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) and len(a[0]) > 0


def test_frames_and_basis_equal_reference():
    rng = np.random.default_rng(21)
    for t in range(300):
        x = rng.normal(0, 1, 12)
        if t % 5 == 0:
            x[:3] = x[3:6]  # touching: zero distance, UnitY normal
        for fn in (O.pt_contact_frame, O.ee_contact_frame):
            a = fn(x)
            with O.use_backend("reference"):
                b = fn(x)
            assert a[0] == b[0] and np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2])
        nrm = rng.normal(0, 1, 3)
        nrm /= np.linalg.norm(nrm)
        if t % 7 == 0:
            nrm = np.array([0.95, np.sqrt(1 - 0.95 ** 2), 0.0])  # |n.x| > 0.9: the UnitY reference
        a = O.tangent_basis(nrm)
        with O.use_backend("reference"):
            b = O.tangent_basis(nrm)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
        assert abs(a[0] @ nrm) < 1e-14 and abs(a[1] @ nrm) < 1e-14


def test_builder_equals_reference():
    g = GeomHybrid(grid=(2, 1, 1), res=4, bodies=(2, 2), body_res=1)
    rng = np.random.default_rng(3)
    for trial in range(3):
        pos = g.node_positions() + rng.normal(0, 5e-5, (g.n_nodes, 3))
        ground = ((0.0, 1.0, 0.0), -0.0004) if trial != 1 else None
        a = O.build_friction_constraints(pos, g.surf_verts, g.edges, g.tris, g.dhat, g.kappa, ground)
        with O.use_backend("reference"):
            b = O.build_friction_constraints(pos, g.surf_verts, g.edges, g.tris, g.dhat, g.kappa, ground)
        assert len(a["n"]) > 0
        for k in a:
            assert np.array_equal(a[k], b[k]), k
        if ground is not None:
            assert np.any(a["n"] == 1)  # ground contacts of the bottom faces
        assert np.all(a["lam"] > 0)
