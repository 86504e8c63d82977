"""Oracle of the element-Hessian producer, pinned two ways:
the reference's own energy/neo_hookean.hpp + energy/psd.hpp compiled in place
(oracle/_ref; the eigen-solver under psd.hpp is oracle/sym_eig.hpp, standing
in for Eigen's) against the restatement in oracle/oracle.hpp, and ports of the
reference's tests/test_energies.cpp cases (:41-59 PSD projection, :224-238
rest-stable / inversion-safe Neo-Hookean, :240-260 finite differences) on
both backends. Also the emission order of the inertia + tet part of
IncrementalPotential::assemble (incremental_potential.hpp:170-180, 222-239,
scatter12 :310-318)."""
import numpy as np
import pytest

import oracle_py as O
import scenegen as scenes

P0 = np.array([0, 0, 0, 1, 0, 0, 0, 1, 0, 0, 0, 1], np.float64)


def rel_err(a, b):  # tests/test_util.hpp rel_err: |a - b| / max(|b|, tiny)
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


def test_psd_projection_clamps_and_is_idempotent(oracle_backend):
    """test_energies.cpp:41-59."""
    M = np.diag([1.0, -1.0])
    P = O.project_psd(M)
    assert P[0, 0] == pytest.approx(1.0)
    assert abs(P[1, 1]) <= 1e-14
    assert rel_err(O.project_psd(P), P) <= 1e-12
    rng = np.random.default_rng(3)
    R = rng.standard_normal((7, 7))
    S = R + R.T
    PS = O.project_psd(S)
    assert np.linalg.eigvalsh(PS).min() >= -1e-12 * np.linalg.norm(S)
    assert rel_err(O.project_psd(PS), PS) <= 1e-12
    # against numpy's eigh: the same spectral projector
    w, V = np.linalg.eigh(S)
    assert rel_err(PS, (V * np.maximum(w, 0)) @ V.T) <= 1e-13


def test_neo_hookean_rest_stable_and_inversion_safe(oracle_backend):
    """test_energies.cpp:224-238."""
    inv, vol = O.tet_rest(P0)
    assert vol == pytest.approx(1.0 / 6.0)
    _, g, _ = O.stable_neo_hookean(P0, inv, vol, 1e5, 4e5, project=False)
    assert np.linalg.norm(g) <= 1e-8 * 1e5 * vol
    x = P0.copy()
    x[9:] = [0, 0, -1]
    val, g, h = O.stable_neo_hookean(x, inv, vol, 1e5, 4e5, project=True)
    assert np.isfinite(val) and np.all(np.isfinite(g))
    assert np.linalg.eigvalsh(h).min() >= -1e-8 * np.linalg.norm(h)


def test_neo_hookean_matches_finite_differences(oracle_backend):
    """test_energies.cpp:240-260: gradient 1e-4, Hessian 1e-3 vs central FD."""
    rng = np.random.default_rng(17)
    inv, vol = O.tet_rest(P0)
    mu, lam = 2.0, 7.0
    for _ in range(12):
        x = P0 + rng.normal(0.0, 0.25, 12)
        val, g, h = O.stable_neo_hookean(x, inv, vol, mu, lam, project=False)
        eps = 1e-6
        fg = np.empty(12)
        fh = np.empty((12, 12))
        for k in range(12):
            d = np.zeros(12)
            d[k] = eps
            vp, gp, _ = O.stable_neo_hookean(x + d, inv, vol, mu, lam, project=False)
            vm, gm, _ = O.stable_neo_hookean(x - d, inv, vol, mu, lam, project=False)
            fg[k] = (vp - vm) / (2 * eps)
            fh[:, k] = (gp - gm) / (2 * eps)
        assert rel_err(g, fg) <= 1e-4
        assert rel_err(h, fh) <= 1e-3


def test_restatement_equals_reference_neo_hookean():
    """oracle.hpp's stencil vs the reference's own neo_hookean.hpp (oracle/_ref)
    on random deformations, projected and raw: the same arithmetic, bitwise."""
    if not O.reference_available():
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(5)
    for t in range(60):
        p = P0 + rng.normal(0.0, 0.05, 12)
        inv, vol = O.tet_rest(p)
        with O.use_backend("reference"):
            inv_r, vol_r = O.tet_rest(p)
        assert np.array_equal(inv, inv_r) and vol == vol_r
        x = p + rng.normal(0.0, 0.2, 12)
        for project in (False, True):
            a = O.stable_neo_hookean(x, inv, vol, 3.0, 11.0, project)
            with O.use_backend("reference"):
                b = O.stable_neo_hookean(x, inv, vol, 3.0, 11.0, project)
            assert a[0] == b[0] and np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2])


def test_ip_fem_assemble_emission_order():
    """Inertia diagonals first (every vertex, :170-180), then per tet the ten
    a <= b blocks of scatter12 (:310-318) through emit() (transposed keys when
    the slot order flips); value = inertia + dt^2 sum of element energies;
    grad zero on pinned slots (:253-254)."""
    sc = scenes.CONFIGS["cfg1_soft_cube"]()
    rng = np.random.default_rng(2)
    n, nt = len(sc.mass), len(sc.tets)
    inv9, vol = scenes.tet_rest_data(sc.verts, sc.tets)
    x = sc.verts.reshape(-1) + rng.normal(0, 1e-4, 3 * n)
    xt = scenes.inertial_target(sc)
    pinned = np.zeros(n, np.uint8)
    pinned[:121] = 1
    dt2 = 1e-4
    val, grad, keys, vals = O.ip_fem_assemble(x, xt, sc.mass, [0, nt], [sc.mu], [sc.lam], sc.tets, inv9, vol, dt2,
                                              pinned)
    assert len(keys) == n + 10 * nt
    assert np.array_equal(keys[:n], (np.arange(n, dtype=np.uint64) << np.uint64(32)) | np.arange(n, dtype=np.uint64))
    assert np.array_equal(vals[:n, 0], sc.mass) and np.all(vals[:n, [1, 2, 3, 5, 6, 7]] == 0)
    pairs = [(a, b) for a in range(4) for b in range(a, 4)]
    t = 17
    te = sc.tets[t]
    _, _, h = O.stable_neo_hookean(x.reshape(-1, 3)[te].reshape(-1), inv9[t], vol[t], sc.mu, sc.lam, True)
    for q, (a, b) in enumerate(pairs):
        k = int(keys[n + 10 * t + q])
        r, c = k >> 32, k & 0xFFFFFFFF
        blk = dt2 * h[3 * a:3 * a + 3, 3 * b:3 * b + 3]
        if te[a] <= te[b]:
            assert (r, c) == (te[a], te[b]) and np.array_equal(vals[n + 10 * t + q], blk.T.reshape(-1))
        else:
            assert (r, c) == (te[b], te[a]) and np.array_equal(vals[n + 10 * t + q], blk.reshape(-1))
    assert np.all(grad.reshape(-1, 3)[:121] == 0)
    dx = (x - xt).reshape(-1, 3)
    inertia = 0.5 * float(np.sum(sc.mass * np.sum(dx * dx, axis=1)))
    elastic = sum(O.stable_neo_hookean(x.reshape(-1, 3)[sc.tets[i]].reshape(-1), inv9[i], vol[i], sc.mu, sc.lam)[0]
                  for i in range(0, nt, 97))
    assert val > inertia - 1e-12 and np.isfinite(elastic)


def test_rest_state_stream_matches_scene_generator():
    """At rest (F = I) the producer's stream is the scene generator's cfg1
    stream (its restated rest Hessian, scenegen/scenes.cpp rest_tet_hessian)
    to rounding: same keys in the same order, values within 1e-12."""
    sc = scenes.CONFIGS["cfg1_soft_cube"]()
    n, nt = len(sc.mass), len(sc.tets)
    inv9, vol = scenes.tet_rest_data(sc.verts, sc.tets)
    x = sc.verts.reshape(-1)
    _, _, keys, vals = O.ip_fem_assemble(x, scenes.inertial_target(sc), sc.mass, [0, nt], [sc.mu], [sc.lam], sc.tets,
                                         inv9, vol, 1e-4)
    assert np.array_equal(keys, sc.keys)
    scale = np.abs(sc.vals).max()
    assert np.abs(vals - sc.vals).max() <= 1e-12 * scale


def test_shell_stencils_equal_reference_and_fd():
    """Membrane (incremental_potential.hpp:273-298 over energy/membrane.hpp)
    and hinge bending (energy/bending.hpp) restated vs the reference's own
    code (membrane to 1e-14, the chain-rule order differs; hinge bitwise),
    and their raw gradients / Hessians against central differences."""
    rng = np.random.default_rng(8)
    mat = [1e-3, 5e4, 5e6, 0.3, 1e-3]
    have_ref = O.reference_available()
    for t in range(40):
        p = np.array([0, 0, 0, 1, 0, 0, 0, 1, 0.0]) + rng.normal(0, 0.05, 9)
        r = O.membrane_rest(p)
        x = p * np.tile([1.1, 0.95, 1.0], 3) + rng.normal(0, 0.03, 9)
        q = np.concatenate([p, p[3:6] + p[6:9] - p[:3] + rng.normal(0, 0.05, 3)])
        hr = O.hinge_rest(q)
        y = q + rng.normal(0, 0.05, 12)
        for project in (True, False):
            a = O.membrane_stencil(x, r, mat, project)
            ha = O.hinge_bending(y, hr, 1e-3, project)
            if have_ref:
                with O.use_backend("reference"):
                    b = O.membrane_stencil(x, r, mat, project)
                    hb = O.hinge_bending(y, hr, 1e-3, project)
                assert abs(a[0] - b[0]) <= 1e-14 * abs(b[0])
                assert np.abs(a[1] - b[1]).max() <= 1e-14 * np.abs(b[1]).max()
                assert np.abs(a[2] - b[2]).max() <= 1e-14 * np.abs(b[2]).max()
                assert ha[0] == hb[0] and np.array_equal(ha[1], hb[1]) and np.array_equal(ha[2], hb[2])
        if t < 8:  # central differences of the raw stencils
            for f, z, n in ((lambda v: O.membrane_stencil(v, r, mat, False), x, 9),
                            (lambda v: O.hinge_bending(v, hr, 1e-3, False), y, 12)):
                _, g, H = f(z)
                eps = 1e-7
                fg = np.array([(f(z + e)[0] - f(z - e)[0]) / (2 * eps) for e in np.eye(n) * eps])
                fh = np.array([(f(z + e)[1] - f(z - e)[1]) / (2 * eps) for e in np.eye(n) * eps]).T
                assert rel_err(g, fg) <= 1e-5
                assert rel_err(H, fh) <= 1e-4
