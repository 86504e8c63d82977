"""The step after the solve (TimeStepper, adipc/solver/newton.hpp:257-290),
restated in oracle_py: known answers from the affine-body kinematics (a body
direction that is a pure translation moves every body vertex by it; a linear
part moves vertex xbar by A xbar and |A xbar| <= |A|_F |xbar|, the bound
step_inf_norm uses) and the FEM vertex norm."""
import numpy as np

import oracle_py as O


def _body_dir(t, A):
    return np.concatenate([t, np.asarray(A).reshape(-1)])  # p, then the rows of A


def test_translation_moves_every_body_vertex():
    rng = np.random.default_rng(1)
    t = np.array([0.3, -1.2, 0.5])
    rest = rng.standard_normal((6, 3))
    d = np.concatenate([np.zeros(3 * 2), _body_dir(t, np.zeros((3, 3)))])  # 2 FEM vertices, 1 body
    jac = [O.abd_jacobian(x) for x in rest]
    disp = O.node_displacements(d, 2, [0] * 6, jac).reshape(-1, 3)
    assert np.allclose(disp[2:], t, rtol=0, atol=0)
    assert O.step_inf_norm(d, 2, 1, [np.abs(rest).max()]) == np.linalg.norm(t)


def test_linear_part_and_norm_bound():
    rng = np.random.default_rng(2)
    A = rng.standard_normal((3, 3))
    rest = rng.standard_normal((10, 3))
    d = _body_dir(np.zeros(3), A)
    jac = [O.abd_jacobian(x) for x in rest]
    disp = O.node_displacements(d, 0, [0] * 10, jac).reshape(-1, 3)
    assert np.allclose(disp, rest @ A.T, rtol=1e-15, atol=1e-15)
    max_xbar = np.linalg.norm(rest, axis=1).max()
    bound = O.step_inf_norm(d, 0, 1, [max_xbar])
    assert np.isclose(bound, np.linalg.norm(A) * max_xbar, rtol=1e-15)
    assert np.linalg.norm(disp, axis=1).max() <= bound * (1 + 1e-15)


def test_fem_norm_and_apply_direction():
    d = np.array([3.0, 4.0, 0.0, 1.0, 2.0, 2.0])
    assert O.step_inf_norm(d, 2, 0, []) == 5.0
    s = np.arange(6.0)
    assert np.array_equal(O.apply_direction(s, d, 0.5), s + 0.5 * d)
