"""GPU parity of the device contact producers (SURVEY.md §8f #2,
csrc/contact.cu) against the oracle's restatement (pinned bitwise to the
reference's contact/distance.hpp + barrier.hpp in test_oracle_contact.py):
the node stream of assemble_contact (incremental_potential.hpp:322-384) —
active set, emission order and keys bitwise; block values to 1e-9 of each
block's norm (the projection runs in the 9-dimensional complement of the
translations on the device, Eigen-style Jacobi on the 12 x 12 in the
oracle); node gradient and value to 1e-12 — the line-search value
(:133-157) and the CCD step bound (ccd.hpp:88-110). End to end: device node
stream -> two_level_abd_reduce + sort + reduce on the device against the
oracle's pipeline on an affine-body scene."""
import numpy as np
import pytest
import torch

import oracle_py as O
import scenegen as scenes
from contact_cases import device_dict, make_case
from paper_2411_06224_b200.context import Context

pytestmark = pytest.mark.gpu
DET = O.ExecPolicy(deterministic=True)
DT2 = 1e-4


@pytest.fixture(scope="module")
def ctx():
    c = Context(0)
    yield c
    c.close()


def gpu_emit(ctx, ci, project=True):
    d = device_dict(ci)
    cap = max(ci.max_entries(), 1)
    keys = torch.empty(cap, dtype=torch.int64, device="cuda:0")
    vals = torch.empty((cap, 9), dtype=torch.float64, device="cuda:0")
    g = torch.empty(3 * len(ci.pos), dtype=torch.float64, device="cuda:0")
    val, n = ctx.contact_emit(d, DT2, keys, vals, g, project=project)
    return val, g.cpu().numpy(), keys[:n].cpu().numpy().view(np.uint64), vals[:n].cpu().numpy()


def assert_blocks_close(got, want, tol, group=10):
    """Block differences relative to the scale of the stencil they belong to
    (a stencil's 10 blocks are consecutive; blocks the exact Hessian leaves
    zero come out as rounding after a projection): the largest block norm
    within +-(group - 1) entries."""
    diff = np.linalg.norm(got - want, axis=1)
    norm = np.linalg.norm(want, axis=1)
    pad = np.pad(norm, group - 1)
    scale = np.max(np.lib.stride_tricks.sliding_window_view(pad, 2 * group - 1), axis=1)
    ratio = diff / np.maximum(scale, 1e-300)
    assert np.all(diff <= tol * scale + 1e-300), ratio.max()


@pytest.mark.parametrize("seed,project", [(1, True), (2, True), (3, False)])
def test_contact_emit_matches_oracle(ctx, seed, project):
    ci = make_case(seed=seed)
    val, g, keys, vals = gpu_emit(ctx, ci, project)
    ov, og, ok, ovals = O.contact_assemble(ci, DT2, project)
    assert np.array_equal(keys, ok), "active set / emission order / keys differ"
    assert_blocks_close(vals, ovals, 1e-9)
    gn = np.linalg.norm(og.reshape(-1, 3), axis=1)
    assert np.all(np.linalg.norm((g - og).reshape(-1, 3), axis=1) <= 1e-12 * np.maximum(gn, 1e-300) + 1e-300)
    assert abs(val - ov) <= 1e-12 * abs(ov)


def test_contact_value_and_touch(ctx):
    ci = make_case(seed=5)
    d = device_dict(ci)
    v = ctx.contact_value(d, DT2)
    assert v == pytest.approx(O.contact_value(ci, DT2), rel=1e-12)
    # a stencil in contact: +inf, as the reference's value() returns
    pos = ci.pos.copy()
    s = ci.pt[0]
    pos[s[0]] = pos[s[1]]
    touched = O.ContactInput(pos, ci.pt, ci.ee, ci.dhat, ci.kappa, ci.ground, ci.surf_verts)
    assert O.contact_value(touched, DT2) == np.inf
    assert ctx.contact_value(device_dict(touched), DT2) == np.inf


def test_ccd_step_matches_oracle(ctx):
    ci = make_case(seed=6, n_fr4=0, n_fr1=0)
    rng = np.random.default_rng(7)
    for scale in (1e-3, 1e-2, 0.1):
        disp = rng.normal(0, scale, ci.pos.shape)
        a = ctx.ccd_step(device_dict(ci), torch.from_numpy(disp.reshape(-1)).cuda())
        assert a == pytest.approx(O.ccd_step(ci, disp), rel=1e-12, abs=1e-15)


def test_contact_pipeline_through_two_level_reduction(ctx):
    """Device node stream -> adipc_gpu_assemble_contact_device (two-level ABD
    reduction + append + sort + reduce) against the oracle's node stream ->
    two_level_abd_reduce -> concatenation -> sort -> hash reduction, on the
    affine-body stack (cfg3): PT / EE stencils over body surface nodes, node
    positions from the rest shapes, pattern bitwise, values to 1e-9."""
    sc = scenes.CONFIGS["cfg3_abd_stack"]()
    # contact-node positions of the bodies at rest: J = [I | x_bar (x) I] -> x_bar
    jac = sc.jac36.reshape(-1, 12, 3).transpose(0, 2, 1)  # n x 3 x 12
    xbar = np.stack([jac[:, 0, 3], jac[:, 0, 4], jac[:, 0, 5]], axis=1)
    rng = np.random.default_rng(9)
    n_nodes = len(xbar)
    body = sc.abd_body
    # stencils between nodes of bodies b and b + 1, moved into contact range
    pos = xbar.copy()
    pt, ee = [], []
    for k in range(400):
        b = rng.integers(0, sc.n_bodies - 1)
        na = np.flatnonzero(body == b)
        nb = np.flatnonzero(body == b + 1)
        if k % 2 == 0:
            pt.append([rng.choice(na), *rng.choice(nb, 3, replace=False)])
        else:
            ee.append([*rng.choice(na, 2, replace=False), *rng.choice(nb, 2, replace=False)])
    pos = pos + rng.normal(0, 1e-4, pos.shape)
    ci = O.ContactInput(pos, pt, ee, dhat=0.08, kappa=1e3)
    ov, og, ok, ovals = O.contact_assemble(ci, DT2)
    assert len(ok) > 0
    tk, tv = O.two_level_abd_reduce(ok, ovals, sc.n_fem, sc.n_bodies, sc.abd_body, sc.jac36, DET)
    fk, fv = O.filter_pinned(np.concatenate([sc.keys, tk]), np.concatenate([sc.vals, tv]), sc.pinned)
    sk, sv = O.sort_stream(fk, fv, DET)
    orow, ocol, oblk = O.fast_hash_reduction(sk, sv, sc.n_blocks, DET)
    # device: producer -> node stream -> two-level + global sort / reduce
    _, _, keys, vals = gpu_emit(ctx, ci)
    assert np.array_equal(keys, ok)
    dev = "cuda:0"
    U, _ = ctx.assemble_contact(torch.from_numpy(sc.keys.view(np.int64)).to(dev), torch.from_numpy(sc.vals).to(dev),
                                torch.from_numpy(keys.view(np.int64)).to(dev), torch.from_numpy(vals).to(dev),
                                sc.n_fem, sc.n_bodies, torch.from_numpy(sc.abd_body).to(dev),
                                torch.from_numpy(sc.jac36).to(dev), sc.n_blocks, torch.from_numpy(sc.pinned).to(dev))
    n, rows, cols, blocks = ctx.copy_matrix()
    assert U == len(orow) and np.array_equal(rows, orow) and np.array_equal(cols, ocol)
    assert_blocks_close(blocks, oblk, 1e-9)


@pytest.mark.parametrize("n,swept", [(6, False), (6, True), (40, False), (40, True)])
def test_broad_phase_matches_oracle(ctx, n, swept):
    """Device find_candidates (broad_phase.hpp:143-211) equals the oracle's
    hash grid (itself equal to brute force): pairs bitwise, in order; node
    stencils resolved from the surface."""
    from contact_cases import layered_surface

    pos, verts, edges, tris = layered_surface(n=n, layers=3)
    inflate = 0.11 if n == 6 else 0.03
    disp = np.random.default_rng(n).normal(0, 0.01, pos.shape) if swept else None
    opt, oee = O.find_candidates(pos, verts, edges, tris, inflate, disp=disp)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    ppairs, pst, epairs, est = ctx.broad_phase(t(pos), t(verts), t(edges), t(tris), inflate,
                                               disp=None if disp is None else t(disp))
    assert np.array_equal(ppairs.cpu().numpy(), opt) and np.array_equal(epairs.cpu().numpy(), oee)
    assert len(opt) > 0 and len(oee) > 0
    pst = pst.cpu().numpy()
    assert np.array_equal(pst[:, 0], verts[opt[:, 0]]) and np.array_equal(pst[:, 1:], tris[opt[:, 1]])
    est = est.cpu().numpy()
    assert np.array_equal(est[:, :2], edges[oee[:, 0]]) and np.array_equal(est[:, 2:], edges[oee[:, 1]])


def test_device_contact_chain(ctx):
    """broad phase -> contact producer on the device (no host round trip)
    against the oracle's candidates -> assemble_contact node part."""
    from contact_cases import layered_surface

    pos, verts, edges, tris = layered_surface(n=30, layers=3, noise=0.01)
    dhat = 0.03
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    _, pst, _, est = ctx.broad_phase(t(pos), t(verts), t(edges), t(tris), dhat)
    opt, oee = O.find_candidates(pos, verts, edges, tris, dhat)
    ci = O.ContactInput(pos, np.c_[verts[opt[:, 0]], tris[opt[:, 1]]], np.c_[edges[oee[:, 0]], edges[oee[:, 1]]],
                        dhat=dhat, kappa=1e3)
    ov, og, ok, ovals = O.contact_assemble(ci, DT2)
    cap = 10 * (len(pst) + len(est))
    keys = torch.empty(cap, dtype=torch.int64, device="cuda:0")
    vals = torch.empty((cap, 9), dtype=torch.float64, device="cuda:0")
    g = torch.empty(3 * len(pos), dtype=torch.float64, device="cuda:0")
    d = {"pos": t(pos), "pt": pst, "ee": est, "dhat": dhat, "kappa": 1e3, "ground": None}
    val, nk = ctx.contact_emit(d, DT2, keys, vals, g)
    assert np.array_equal(keys[:nk].cpu().numpy().view(np.uint64), ok) and len(ok) > 0
    assert_blocks_close(vals[:nk].cpu().numpy(), ovals, 1e-9)
    assert abs(val - ov) <= 1e-12 * abs(ov)
