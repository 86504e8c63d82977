"""Oracle of the contact producers: the restated distance /
barrier stencils (oracle/oracle.hpp) against the reference's own
contact/distance.hpp + contact/barrier.hpp compiled in place (oracle/_ref,
bitwise), and ports of the reference's tests/test_contact.cpp cases on both
backends: classification fixtures (:37-110), finite differences of the
squared-distance derivatives (:112-188), barrier activation / FD / PSD
(:205-264), the ground specialisation (:266-291) and conservative advancement
(:293-339)."""
import numpy as np
import pytest

import oracle_py as O
from contact_cases import make_case


def rel_err(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


def x12(*pts):
    return np.concatenate([np.asarray(p, np.float64) for p in pts])


def test_classification_fixtures(oracle_backend):
    """test_contact.cpp:37-110 (distances of the named configurations)."""
    t0, t1, t2 = [0, 0, 0], [1, 0, 0], [0, 1, 0]
    assert O.pt_dist2(x12([0.25, 0.25, 0.7], t0, t1, t2)) == pytest.approx(0.49)
    assert O.pt_dist2(x12([-1, -1, 0.5], t0, t1, t2)) == pytest.approx(2.25)
    assert O.pt_dist2(x12([0.5, -1, 0], t0, t1, t2)) == pytest.approx(1.0)
    assert O.pt_dist2(x12([1, 1, 0], t0, t1, t2)) == pytest.approx(0.5)
    a0, a1 = [-1, 0, 0], [1, 0, 0]
    assert O.ee_dist2(x12(a0, a1, [0, -1, 0.3], [0, 1, 0.3])) == pytest.approx(0.09)
    assert O.ee_dist2(x12([0, 0, 0], [1, 0, 0], [2, 1, 0], [3, 1, 0])) == pytest.approx(2.0)
    assert O.ee_dist2(x12([0, 0, 0], [1, 0, 0], [0.2, 1, 0], [1.2, 1, 0])) == pytest.approx(1.0)
    rng = np.random.default_rng(11)
    for _ in range(100):  # brute force over a barycentric / parameter sweep can do no better
        p = rng.uniform(-2, 2, 3)
        g = np.linspace(0, 1, 41)
        best = min(np.sum((p - ((1 - u - v) * np.array(t0) + u * np.array(t1) + v * np.array(t2))) ** 2)
                   for u in g for v in g if u + v <= 1 + 1e-12)
        assert O.pt_dist2(x12(p, t0, t1, t2)) <= best + 1e-12


def test_distance_derivatives_finite_differences(oracle_backend):
    """test_contact.cpp:112-188 (region-stable stencils, gradient 2e-6, Hessian 2e-5)."""
    rng = np.random.default_rng(21)
    checked = {"pt": 0, "ee": 0}
    h = 1e-5
    while checked["pt"] < 30 or checked["ee"] < 30:
        x = rng.uniform(-1.5, 1.5, 12)
        for kind, derivs, dist in (("pt", O.pt_dist2_derivs, O.pt_dist2), ("ee", O.ee_dist2_derivs, O.ee_dist2)):
            if checked[kind] >= 30 or dist(x) <= 1e-4:
                continue
            d2, g, H = derivs(x)
            fg, fh = np.empty(12), np.empty((12, 12))
            stable = True
            for k in range(12):
                e = np.zeros(12)
                e[k] = h
                dp, gp, _ = derivs(x + e)
                dm, gm, _ = derivs(x - e)
                # the dual value must stay on one smooth branch (same region)
                if abs((dist(x + e) - dp)) > 1e-12 or abs(dist(x - e) - dm) > 1e-12:
                    stable = False
                fg[k] = (dp - dm) / (2 * h)
                fh[:, k] = (gp - gm) / (2 * h)
            if not stable:
                continue
            assert rel_err(g, fg) < 2e-6
            assert rel_err(H, fh) < 2e-5
            assert np.abs(H - H.T).max() < 1e-10
            checked[kind] += 1


def test_barrier_activation_and_projection(oracle_backend):
    """test_contact.cpp:239-264."""
    dhat, kappa = 0.5, 7.0
    shat = dhat * dhat
    x = x12([0.3, 0.3, 0.2], [0, 0, 0], [1, 0, 0], [0, 1, 0])
    d2, g, H = O.pt_dist2_derivs(x)
    v, bg, bh = O.barrier_pair_derivs(d2, g, H, shat, kappa, project=False)
    eps = 1e-6
    fg = np.array([(O.barrier_pair_derivs(O.pt_dist2_derivs(x + e)[0], g, H, shat, kappa, False)[0] -
                    O.barrier_pair_derivs(O.pt_dist2_derivs(x - e)[0], g, H, shat, kappa, False)[0]) / (2 * eps)
                   for e in np.eye(12) * eps])
    assert rel_err(bg, fg) < 1e-4
    _, _, ph = O.barrier_pair_derivs(d2, g, H, shat, kappa, project=True)
    w = np.linalg.eigvalsh(ph)
    assert w.min() > -1e-8 * np.abs(w).max()
    d2o, go, Ho = O.pt_dist2_derivs(x12([0.3, 0.3, 0.9], [0, 0, 0], [1, 0, 0], [0, 1, 0]))
    vo, gvo, hvo = O.barrier_pair_derivs(d2o, go, Ho, shat, kappa, True)
    assert vo == 0.0 and np.all(gvo == 0) and np.all(hvo == 0)


def test_ground_barrier(oracle_backend):
    """test_contact.cpp:266-291."""
    v, g, H, d = O.ground_barrier_derivs([2, 0.58, -1], [0, 1, 0], 0.5, 0.2, 5.0, project=False)
    assert d == pytest.approx(0.08)
    assert v > 0 and g[1] < 0 and g[0] == 0 and g[2] == 0
    _, _, Hp, _ = O.ground_barrier_derivs([2, 0.58, -1], [0, 1, 0], 0.5, 0.2, 5.0, project=True)
    assert np.linalg.eigvalsh(Hp).min() >= 0
    assert O.ground_barrier_derivs([0, 0.9, 0], [0, 1, 0], 0.5, 0.2, 5.0)[0] == 0.0


def test_restatement_equals_reference_contact_stencils():
    """oracle.hpp vs the reference's distance.hpp / barrier.hpp: bitwise."""
    if not O.reference_available():
        pytest.skip("oracle/_ref not built")
    ci = make_case(seed=4, n_pt=150, n_ee=150, n_ground=30, n_fr4=0, n_fr1=0)
    for kind, st in (("pt", ci.pt), ("ee", ci.ee)):
        derivs = O.pt_dist2_derivs if kind == "pt" else O.ee_dist2_derivs
        for s in st:
            x = ci.pos[s].reshape(-1)
            a = derivs(x)
            with O.use_backend("reference"):
                b = derivs(x)
            assert a[0] == b[0] and np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2])
            if a[0] < ci.dhat ** 2:
                ba = O.barrier_pair_derivs(*a, ci.dhat ** 2, ci.kappa)
                with O.use_backend("reference"):
                    bb = O.barrier_pair_derivs(*a, ci.dhat ** 2, ci.kappa)
                assert ba[0] == bb[0] and np.array_equal(ba[1], bb[1]) and np.array_equal(ba[2], bb[2])
    for v in ci.surf_verts:
        a = O.ground_barrier_derivs(ci.pos[v], ci.ground[0], ci.ground[1], ci.dhat, ci.kappa)
        with O.use_backend("reference"):
            b = O.ground_barrier_derivs(ci.pos[v], ci.ground[0], ci.ground[1], ci.dhat, ci.kappa)
        assert a[0] == b[0] and np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2]) and a[3] == b[3]


def test_conservative_advancement():
    """test_contact.cpp:293-339 through ccd_step on single stencils."""
    g = 0.3
    t = [[-5, 0, -5], [5, 0, -5], [0, 0, 5]]
    pos = np.array([[0.1, g, 0.2], *t])

    def step(disp, ground=None, sv=()):
        ci = O.ContactInput(pos, pt=[[0, 1, 2, 3]], dhat=1.0, kappa=1.0, ground=ground, surf_verts=sv)
        return O.ccd_step(ci, np.asarray(disp, np.float64))

    a = step([[0, -2 * g, 0], [0, 0, 0], [0, 0, 0], [0, 0, 0]])
    assert 0.4 < a <= 0.5
    assert step([[0, 2 * g, 0], [0, 0, 0], [0, 0, 0], [0, 0, 0]]) == 1.0
    assert step([[100, 100, 100]] * 4) == 1.0
    ci = O.ContactInput(np.array([[0, g, 0]]), dhat=1.0, kappa=1.0, ground=([0, 1, 0], 0.0), surf_verts=[0])
    ag = O.ccd_step(ci, np.array([[0, -2 * g, 0]]))
    assert 0.4 < ag <= 0.5
    assert O.ccd_step(ci, np.array([[0, 1.0, 0]])) == 1.0
    rng = np.random.default_rng(41)
    for trial in range(200):  # never tunnels
        x = rng.uniform(-1, 1, (4, 3))
        d = rng.uniform(-1.5, 1.5, (4, 3))
        ee = trial % 2
        dist = O.ee_dist2 if ee else O.pt_dist2
        if dist(x.reshape(-1)) < 1e-8:
            continue
        ci = O.ContactInput(x, pt=[] if ee else [[0, 1, 2, 3]], ee=[[0, 1, 2, 3]] if ee else [], dhat=1.0, kappa=1.0)
        alpha = O.ccd_step(ci, d)
        assert 0 < alpha <= 1
        for k in range(65):
            assert dist((x + alpha * k / 64 * d).reshape(-1)) > 0


def test_contact_assemble_emission_order():
    """assemble_contact's node part: active pairs in candidate order (PT then
    EE, 10 blocks each, emit() canonicalisation), then the ground contacts,
    then the friction constraints; value equals the value path's."""
    ci = make_case(seed=2, n_pt=80, n_ee=80, n_ground=40, n_fr4=10, n_fr1=5)
    dt2 = 1e-4
    val, g, keys, vals = O.contact_assemble(ci, dt2)
    shat = ci.dhat ** 2
    act = [s for s in ci.pt if O.pt_dist2_derivs(ci.pos[s].reshape(-1))[0] < shat]
    act += [s for s in ci.ee if O.ee_dist2_derivs(ci.pos[s].reshape(-1))[0] < shat]
    q = 0
    for s in act:
        for a in range(4):
            for b in range(a, 4):
                r, c = sorted((int(s[a]), int(s[b])))
                assert int(keys[q]) == (r << 32 | c)
                q += 1
    gd = [v for v in ci.surf_verts if 0 < ci.pos[v] @ ci.ground[0] - ci.ground[1] < ci.dhat]
    for v in gd:
        assert int(keys[q]) == (int(v) << 32 | int(v))
        q += 1
    assert len(keys) == q + 10 * 10 + 5
    assert val == pytest.approx(O.contact_value(ci, dt2), rel=1e-12)


def test_broad_phase_equals_brute_force():
    """test_contact.cpp:341-409: the hash-grid candidates equal brute force
    with the same inflation, every truly close pair is found, and the swept
    variant with zero displacement equals the proximity one."""
    from contact_cases import brute_candidates, layered_surface

    pos, verts, edges, tris = layered_surface()
    inflate = 0.11
    pt, ee = O.find_candidates(pos, verts, edges, tris, inflate)
    bpt, bee = brute_candidates(pos, verts, edges, tris, inflate)
    assert np.array_equal(pt, bpt) and np.array_equal(ee, bee)
    assert len(pt) and len(ee)
    found = set(map(tuple, pt.tolist()))
    for vi, v in enumerate(verts):
        for ti, t in enumerate(tris):
            if v in t:
                continue
            if O.pt_dist2(np.concatenate([pos[v], pos[t[0]], pos[t[1]], pos[t[2]]])) < inflate ** 2:
                assert (vi, ti) in found
    spt, see = O.find_candidates(pos, verts, edges, tris, inflate, disp=np.zeros_like(pos))
    assert np.array_equal(spt, pt) and np.array_equal(see, ee)
    # swept boxes: a displacement brings new pairs, a superset
    disp = np.random.default_rng(3).normal(0, 0.05, pos.shape)
    wpt, wee = O.find_candidates(pos, verts, edges, tris, inflate, disp=disp)
    bwpt, bwee = brute_candidates(pos, verts, edges, tris, inflate, disp=disp)
    assert np.array_equal(wpt, bwpt) and np.array_equal(wee, bwee)
    assert set(map(tuple, pt.tolist())) <= set(map(tuple, wpt.tolist()))
