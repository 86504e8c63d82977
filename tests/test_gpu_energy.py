"""GPU parity of the device element-Hessian producer (SURVEY.md §8f #1,
csrc/energy.cu) against the oracle's restatement of IncrementalPotential::
assemble for inertia + tets (incremental_potential.hpp:170-180, 222-239,
scatter12 :310-318, :253-254) with the stable Neo-Hookean stencil
(neo_hookean.hpp:64-104, pinned to the reference's own code in
test_oracle_energy.py) and its PSD projection (psd.hpp:8-14).

Keys (emission order + emit() canonicalisation) are compared bitwise; values
to 1e-10 of the stream's scale (the device builds the 12 x 12 stencil as a
bilinear form in the rows of G^T Dm^-1 and projects in the 9-dimensional
complement of the translations — the same matrix, other rounding), the
gradient and the value to 1e-12."""
import numpy as np
import pytest
import torch

import oracle_py as O
import scenegen as scenes
from paper_2411_06224_b200.context import Context

pytestmark = pytest.mark.gpu
DET = O.ExecPolicy(deterministic=True)
DT2 = 1e-4


@pytest.fixture(scope="module")
def ctx():
    c = Context(0)
    yield c
    c.close()


def device_mesh(sc, dev="cuda:0"):
    inv9, vol = scenes.tet_rest_data(sc.verts, sc.tets)
    return {"mass": torch.from_numpy(sc.mass).to(dev), "tets": torch.from_numpy(sc.tets).to(dev),
            "rest_inv9": torch.from_numpy(inv9).to(dev), "rest_volume": torch.from_numpy(vol).to(dev),
            "tet_begin": [0, len(sc.tets)], "mu": [sc.mu], "lam": [sc.lam]}, inv9, vol


def gpu_emit(ctx, mesh, x, xt, project=True, pinned=None):
    n, nt = mesh["mass"].numel(), mesh["tets"].shape[0]
    T = n + 10 * nt
    keys = torch.empty(T, dtype=torch.int64, device="cuda:0")
    vals = torch.empty((T, 9), dtype=torch.float64, device="cuda:0")
    grad = torch.empty(3 * n, dtype=torch.float64, device="cuda:0")
    dx, dxt = torch.from_numpy(x).cuda(), torch.from_numpy(xt).cuda()
    dpin = None if pinned is None else torch.from_numpy(pinned).cuda()
    val = ctx.fem_emit(mesh, dx, dxt, DT2, keys, vals, grad, project=project, pinned=dpin)
    return val, grad.cpu().numpy(), keys.cpu().numpy().view(np.uint64), vals.cpu().numpy()


def deformed(sc, scale, seed):
    rng = np.random.default_rng(seed)
    h = (sc.verts.max(0) - sc.verts.min(0)).max() / 11.0
    return np.ascontiguousarray((sc.verts + rng.uniform(-scale * h, scale * h, sc.verts.shape)).reshape(-1))


@pytest.mark.parametrize("scale,project", [(0.0, True), (0.05, True), (0.3, True), (0.3, False)])
def test_fem_emit_matches_oracle(ctx, scale, project):
    """At rest (every stencil PSD up to rounding: the fast path), mildly and
    strongly deformed (indefinite stencils: the Jacobi path), and raw."""
    sc = scenes.CONFIGS["cfg1_soft_cube"]()
    mesh, inv9, vol = device_mesh(sc)
    x = deformed(sc, scale, 7)
    xt = scenes.inertial_target(sc)
    pinned = np.zeros(len(sc.mass), np.uint8)
    pinned[:121] = 1
    val, grad, keys, vals = gpu_emit(ctx, mesh, x, xt, project, pinned)
    ov, og, ok, ovals = O.ip_fem_assemble(x, xt, sc.mass, [0, len(sc.tets)], [sc.mu], [sc.lam], sc.tets, inv9, vol,
                                          DT2, pinned, project=project)
    assert np.array_equal(keys, ok), "emission order / canonicalisation differs"
    scale_v = np.abs(ovals).max()
    assert np.abs(vals - ovals).max() <= 1e-10 * scale_v
    assert np.linalg.norm(grad - og) <= 1e-12 * max(np.linalg.norm(og), 1e-300)
    assert abs(val - ov) <= 1e-12 * abs(ov)
    if project:  # every emitted element block set is PSD
        n = len(sc.mass)
        for t in range(0, len(sc.tets), 331):
            H = np.zeros((12, 12))
            q = 0
            te = sc.tets[t]
            for a in range(4):
                for b in range(a, 4):
                    blk = vals[n + 10 * t + q].reshape(3, 3).T
                    if te[a] > te[b]:
                        blk = blk.T
                    H[3 * a:3 * a + 3, 3 * b:3 * b + 3] = blk
                    H[3 * b:3 * b + 3, 3 * a:3 * a + 3] = blk.T
                    q += 1
            assert np.linalg.eigvalsh(H).min() >= -1e-10 * np.abs(H).max()


def test_fem_assemble_pattern_bitwise(ctx):
    """emit + filter_pinned + sort + reduce on the device: rows / cols equal
    the oracle's deterministic sort + hash reduction of the oracle stream;
    values to 1e-10."""
    sc = scenes.CONFIGS["cfg1_soft_cube"]()
    mesh, inv9, vol = device_mesh(sc)
    x = deformed(sc, 0.1, 3)
    xt = scenes.inertial_target(sc)
    pinned = np.zeros(len(sc.mass), np.uint8)
    pinned[:121] = 1
    grad = torch.empty(3 * len(sc.mass), dtype=torch.float64, device="cuda:0")
    val, U = ctx.fem_assemble(mesh, torch.from_numpy(x).cuda(), torch.from_numpy(xt).cuda(), DT2, grad,
                              pinned=torch.from_numpy(pinned).cuda())
    n, rows, cols, blocks = ctx.copy_matrix()
    _, _, ok, ov = O.ip_fem_assemble(x, xt, sc.mass, [0, len(sc.tets)], [sc.mu], [sc.lam], sc.tets, inv9, vol, DT2,
                                     pinned)
    fk, fv = O.filter_pinned(ok, ov, pinned)
    sk, sv = O.sort_stream(fk, fv, DET)
    orow, ocol, oblk = O.fast_hash_reduction(sk, sv, n, DET)
    assert U == len(orow) and np.array_equal(rows, orow) and np.array_equal(cols, ocol)
    assert np.abs(blocks - oblk).max() <= 1e-10 * np.abs(oblk).max()


def test_inverted_element_projects_to_psd(ctx):
    """test_energies.cpp:232-237 on the device: an inverted tet gives a finite
    value and gradient and a PSD Hessian."""
    verts = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], np.float64)
    tets = np.array([[0, 1, 2, 3]], np.int32)
    inv9, vol = scenes.tet_rest_data(verts, tets)
    mesh = {"mass": torch.zeros(4, dtype=torch.float64, device="cuda:0"), "tets": torch.from_numpy(tets).cuda(),
            "rest_inv9": torch.from_numpy(inv9).cuda(), "rest_volume": torch.from_numpy(vol).cuda(),
            "tet_begin": [0, 1], "mu": [1e5], "lam": [4e5]}
    x = verts.copy()
    x[3] = [0, 0, -1]
    x = x.reshape(-1)
    val, grad, keys, vals = gpu_emit(ctx, mesh, x, x.copy())
    assert np.isfinite(val) and np.all(np.isfinite(grad)) and np.all(np.isfinite(vals))
    H = np.zeros((12, 12))
    q = 0
    for a in range(4):
        for b in range(a, 4):
            blk = vals[4 + q].reshape(3, 3).T
            H[3 * a:3 * a + 3, 3 * b:3 * b + 3] = blk
            H[3 * b:3 * b + 3, 3 * a:3 * a + 3] = blk.T
            q += 1
    assert np.linalg.eigvalsh(H).min() >= -1e-8 * np.linalg.norm(H)
    _, _, oh = O.stable_neo_hookean(x, inv9[0], vol[0], 1e5, 4e5, True)
    assert np.abs(H - DT2 * oh).max() <= 1e-10 * np.abs(DT2 * oh).max()


def test_cfg5_device_matrix_equals_streamed_matrix(ctx):
    """Full size (cfg5, 1.9 M tets): the device-produced matrix at rest has the
    pattern of the host-streamed one (scene generator, bitwise) and its values
    to 1e-11; the gradient is -M dt^2 g off the pinned face (the elastic
    forces at rest are rounding: mu F + dJcoef cof = mu I - mu I)."""
    sc = scenes.CONFIGS["cfg5_stiff_box"]()
    mesh, _, _ = device_mesh(sc)
    x = torch.from_numpy(np.ascontiguousarray(sc.verts.reshape(-1))).cuda()
    xt = torch.from_numpy(scenes.inertial_target(sc)).cuda()
    grad = torch.empty_like(x)
    _, U = ctx.fem_assemble(mesh, x, xt, DT2, grad, pinned=torch.from_numpy(sc.pinned).cuda())
    _, rows, cols, blocks = ctx.copy_matrix()
    U2 = ctx.assemble_filtered(sc.keys, sc.vals, sc.n_blocks, sc.pinned)
    _, rows2, cols2, blocks2 = ctx.copy_matrix()
    assert U == U2 and np.array_equal(rows, rows2) and np.array_equal(cols, cols2)
    assert np.abs(blocks - blocks2).max() <= 1e-11 * np.abs(blocks2).max()
    b = scenes.gravity_rhs(sc)
    assert np.abs(-grad.cpu().numpy() - b).max() <= 1e-9 * np.abs(b).max()


def bodies_case(nb, seed):
    rng = np.random.default_rng(seed)
    q = np.zeros((nb, 12))
    q[:, :3] = rng.normal(0, 1, (nb, 3))
    q[:, 3:] = (np.eye(3)[None] + rng.normal(0, 0.05, (nb, 3, 3))).reshape(nb, 9)
    qt = q + rng.normal(0, 1e-3, q.shape)
    L = rng.normal(0, 1, (nb, 12, 12))
    M = L @ L.transpose(0, 2, 1) + 12 * np.eye(12)[None]
    return {"q": q, "q_tilde": qt, "reduced_mass": M, "kappa": rng.uniform(1e6, 1e8, nb),
            "volume": rng.uniform(1e-4, 1e-3, nb)}


def test_fem_emit_with_bodies_and_value(ctx):
    """Inertia + tets + affine bodies (incremental_potential.hpp:170-249):
    body inertia tiles after the vertex inertia, orthogonality tiles
    (abd_energy.hpp:19-42) after the tets; the value-only entry (the line
    search's IncrementalPotential::value, :61-131) equals the emit's value."""
    sc = scenes.CONFIGS["cfg1_soft_cube"]()
    mesh, inv9, vol = device_mesh(sc)
    nb = 7
    bd = bodies_case(nb, 3)
    mesh["bodies"] = {"q": torch.from_numpy(bd["q"]).cuda(), "q_tilde": torch.from_numpy(bd["q_tilde"]).cuda(),
                      "reduced_mass": torch.from_numpy(np.ascontiguousarray(bd["reduced_mass"].transpose(0, 2, 1)))
                      .cuda(), "kappa": torch.from_numpy(bd["kappa"]).cuda(),
                      "volume": torch.from_numpy(bd["volume"]).cuda()}
    n, nt = len(sc.mass), len(sc.tets)
    x = deformed(sc, 0.2, 11)
    xt = scenes.inertial_target(sc)
    pinned = np.zeros(n + 4 * nb, np.uint8)
    pinned[:121] = 1
    pinned[n + 4] = 1  # one body block
    T = n + 10 * nt + 20 * nb
    keys = torch.empty(T, dtype=torch.int64, device="cuda:0")
    vals = torch.empty((T, 9), dtype=torch.float64, device="cuda:0")
    grad = torch.empty(3 * (n + 4 * nb), dtype=torch.float64, device="cuda:0")
    dx, dxt, dpin = torch.from_numpy(x).cuda(), torch.from_numpy(xt).cuda(), torch.from_numpy(pinned).cuda()
    val = ctx.fem_emit(mesh, dx, dxt, DT2, keys, vals, grad, pinned=dpin)
    ov, og, ok, ovals = O.ip_fem_assemble(x, xt, sc.mass, [0, nt], [sc.mu], [sc.lam], sc.tets, inv9, vol, DT2,
                                          pinned, bodies=bd)
    keys = keys.cpu().numpy().view(np.uint64)
    vals = vals.cpu().numpy()
    assert np.array_equal(keys, ok)
    for lo, hi in ((0, n + 10 * nb), (n + 10 * nb, n + 10 * nb + 10 * nt), (n + 10 * nb + 10 * nt, T)):
        assert np.abs(vals[lo:hi] - ovals[lo:hi]).max() <= 1e-10 * np.abs(ovals[lo:hi]).max()
    g = grad.cpu().numpy()
    assert np.linalg.norm(g - og) <= 1e-12 * np.linalg.norm(og)
    assert abs(val - ov) <= 1e-12 * abs(ov)
    g2 = torch.empty_like(grad)
    v2 = ctx.fem_value(mesh, dx, dxt, DT2, g2, pinned=dpin)
    assert abs(v2 - val) <= 1e-13 * abs(val)
    assert torch.allclose(g2, grad, rtol=0, atol=1e-12 * float(torch.abs(grad).max()))


@pytest.mark.parametrize("order", [(0, 1), (1, 0)])
def test_fem_emit_shells_and_solids_in_mesh_order(ctx, order):
    """A cloth patch (membrane triangles + hinges, incremental_potential.hpp:
    190-221, membrane.hpp, bending.hpp) and the soft cube in either scene
    order: the stream follows the mesh order (solid: tets; shell: triangles
    then hinges); keys bitwise, values to 1e-10 of each stencil's scale,
    gradient and value to 1e-12."""
    from contact_cases import cloth_patch

    sc = scenes.CONFIGS["cfg1_soft_cube"]()
    inv9, vol = scenes.tet_rest_data(sc.verts, sc.tets)
    nsol = len(sc.mass)
    first_solid = order[0] == 0
    off = nsol if first_solid else 0
    cl = cloth_patch(20, 3, offset=off)
    ncl = len(cl["mass"])
    sol_off = 0 if first_solid else ncl
    tets = sc.tets + sol_off
    n = nsol + ncl
    x = np.zeros((n, 3))
    mass = np.zeros(n)
    xs = deformed(sc, 0.1, 4).reshape(-1, 3)
    x[sol_off:sol_off + nsol], mass[sol_off:sol_off + nsol] = xs, sc.mass
    x[off:off + ncl], mass[off:off + ncl] = cl["x"], cl["mass"]
    x = np.ascontiguousarray(x.reshape(-1))
    xt = x + np.random.default_rng(1).normal(0, 1e-5, x.shape)
    shells = {"tri_begin": [0, len(cl["tris"])], "hinge_begin": [0, len(cl["hinges"])], "tris": cl["tris"],
              "tri_rest": cl["tri_rest"], "hinges": cl["hinges"], "hinge_rest": cl["hinge_rest"],
              "material": [cl["material"]]}
    kinds = list(order)
    ov, og, ok, ovals = O.ip_fem_assemble(x, xt, mass, [0, len(tets)], [sc.mu], [sc.lam], tets, inv9, vol, DT2,
                                          shells=shells, mesh_kind=kinds)
    t = lambda a, dt=None: torch.from_numpy(np.ascontiguousarray(a, dt)).cuda()  # noqa: E731
    mesh = {"mass": t(mass), "tets": t(tets, np.int32), "rest_inv9": t(inv9), "rest_volume": t(vol),
            "tet_begin": [0, len(tets)], "mu": [sc.mu], "lam": [sc.lam], "mesh_kind": kinds,
            "shells": {"tri_begin": [0, len(cl["tris"])], "hinge_begin": [0, len(cl["hinges"])],
                       "tris": t(cl["tris"], np.int32), "tri_rest": t(cl["tri_rest"]),
                       "hinges": t(cl["hinges"], np.int32), "hinge_rest": t(cl["hinge_rest"]),
                       "material": [cl["material"]]}}
    T = len(ok)
    keys = torch.empty(T, dtype=torch.int64, device="cuda:0")
    vals = torch.empty((T, 9), dtype=torch.float64, device="cuda:0")
    grad = torch.empty(3 * n, dtype=torch.float64, device="cuda:0")
    val = ctx.fem_emit(mesh, t(x), t(xt), DT2, keys, vals, grad)
    keys = keys.cpu().numpy().view(np.uint64)
    assert np.array_equal(keys, ok)
    vals = vals.cpu().numpy()
    diff = np.linalg.norm(vals - ovals, axis=1)
    norm = np.linalg.norm(ovals, axis=1)
    scale = np.max(np.lib.stride_tricks.sliding_window_view(np.pad(norm, 9), 19), axis=1)
    assert np.all(diff <= 1e-10 * scale + 1e-300)
    g = grad.cpu().numpy()
    assert np.linalg.norm(g - og) <= 1e-12 * np.linalg.norm(og)
    assert abs(val - ov) <= 1e-12 * abs(ov)
