"""Every kernel path behind an ADIPC_OPT_* option solves the same system as
the reference: the PCG on the stiff beam's first Newton matrix and on the soft
cube, for the default solve-order kernels, the generic level kernels (no solve
order / no solve-order kernels) and the preconditioner ring shapes —
iteration counts within +-2 % and solutions within 1e-5 relative L2 of the
oracle, the north-star parity contract. Also a preconditioner apply through
the C ABI in solve order against the reference numbering, and restart
iterations (every 5th, pcg.hpp:69-74) through each path."""
import numpy as np
import pytest

import oracle_py as O
import paper_2411_06224_b200 as P
from paper_2411_06224_b200 import _lib
import scenegen as scenes
from paper_2411_06224_b200.context import Context

pytestmark = pytest.mark.gpu
DET = O.ExecPolicy(deterministic=True)

VARIANTS = {
    "default": {},
    "generic-order": {_lib.OPT_SOLVE_ORDER: 0},
    "generic-kernels": {_lib.OPT_SO_KERNELS: 0},
    "pc-stages3": {_lib.OPT_L0_STAGES: 3},
    "pc-2pairs": {_lib.OPT_PC_PAIRS: 2},
}


def _system(name):
    sc = scenes.CONFIGS[name]()
    fk, fv = O.filter_pinned(sc.keys, sc.vals, sc.pinned)
    sk, sv = O.sort_stream(fk, fv, DET)
    rows, cols, blocks = O.fast_hash_reduction(sk, sv, sc.n_blocks, DET)
    l0 = P.partition_block_graph(sc.n_blocks, sc.rest_edges, 16)
    return sc, rows, cols, blocks, l0


@pytest.fixture(scope="module")
def beam():
    sc, rows, cols, blocks, l0 = _system("stiff_beam")
    b = scenes.gravity_rhs(sc)
    Am = O.Matrix(sc.n_blocks, rows, cols, blocks)
    M = O.MasPreconditioner(Am, O.Hierarchy(l0.part_of, l0.n_parts, 16, O.block_edges(rows, cols), 4))
    xo, ro = O.pcg_solve(Am, b, M, 1e-4, 250, 100000)
    xr, rr = O.pcg_solve(Am, b, M, 1e-4, 5, 100000)  # restart every 5th iteration
    return sc, rows, cols, blocks, l0, b, (xo, ro), (xr, rr)


def _ctx(sc, rows, cols, blocks, l0, opts):
    c = Context(0)
    for k, v in opts.items():
        c.set_option(k, v)
    c.set_matrix(sc.n_blocks, rows, cols, blocks)
    c.set_level0_partition(l0.part_of, l0.n_parts, 16, 4)
    c.build_preconditioner(_lib.PRECOND_MAS)
    return c


@pytest.mark.parametrize("variant", sorted(VARIANTS))
def test_variant_pcg_parity(beam, variant):
    sc, rows, cols, blocks, l0, b, (xo, ro), _ = beam
    c = _ctx(sc, rows, cols, blocks, l0, VARIANTS[variant])
    x, r = c.pcg(b, 1e-4, 250, 100000)
    c.close()
    assert r.converged and ro["converged"]
    assert abs(r.iters - ro["iters"]) <= max(1, 0.02 * ro["iters"]), (variant, r.iters, ro["iters"])
    assert np.linalg.norm(x - xo) <= 1e-5 * np.linalg.norm(xo), variant


@pytest.mark.parametrize("variant", ["default", "generic-order", "generic-kernels"])
def test_variant_restart_iterations(beam, variant):
    """r = b - A x every 5th iteration (pcg.hpp:69-74) through each path."""
    sc, rows, cols, blocks, l0, b, _, (xr, rr) = beam
    c = _ctx(sc, rows, cols, blocks, l0, VARIANTS[variant])
    x, r = c.pcg(b, 1e-4, 5, 100000)
    c.close()
    assert r.converged == rr["converged"]
    assert abs(r.iters - rr["iters"]) <= max(1, 0.02 * rr["iters"]), (variant, r.iters, rr["iters"])
    assert np.linalg.norm(x - xr) <= 1e-5 * np.linalg.norm(xr), variant


@pytest.mark.parametrize("variant", ["default", "generic-kernels"])
def test_variant_cube(variant):
    sc, rows, cols, blocks, l0 = _system("cfg1_soft_cube")
    b = scenes.gravity_rhs(sc)
    Am = O.Matrix(sc.n_blocks, rows, cols, blocks)
    M = O.MasPreconditioner(Am, O.Hierarchy(l0.part_of, l0.n_parts, 16, O.block_edges(rows, cols), 4))
    xo, ro = O.pcg_solve(Am, b, M, 1e-4, 250, 100000)
    c = _ctx(sc, rows, cols, blocks, l0, VARIANTS[variant])
    x, r = c.pcg(b, 1e-4, 250, 100000)
    c.close()
    assert abs(r.iters - ro["iters"]) <= max(1, 0.02 * ro["iters"])
    assert np.linalg.norm(x - xo) <= 1e-5 * np.linalg.norm(xo)


def test_apply_in_solve_order_matches_reference_numbering(beam):
    """MasPreconditioner::apply (mas.hpp:85-99) through the C ABI: the device
    runs in solve order, inputs and outputs are in the reference numbering."""
    sc, rows, cols, blocks, l0, b, _, _ = beam
    Am = O.Matrix(sc.n_blocks, rows, cols, blocks)
    M = O.MasPreconditioner(Am, O.Hierarchy(l0.part_of, l0.n_parts, 16, O.block_edges(rows, cols), 4))
    r = np.random.default_rng(3).standard_normal(3 * sc.n_blocks)
    zo = M.apply(r)
    for order in (1, 0):
        c = _ctx(sc, rows, cols, blocks, l0, {_lib.OPT_SOLVE_ORDER: order})
        z = c.precond_apply(r)
        c.close()
        assert np.linalg.norm(z - zo) <= 1e-10 * np.linalg.norm(zo), order
