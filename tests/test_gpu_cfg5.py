"""Parity on the BENCHMARKED configuration (BASELINE.json config 5, the
985,527-DOF stiff box the bench line is quoted on) against the reference's
own hot-path code compiled in place (oracle/_ref; the restatement when it is
absent):

* assembly (filter_pinned + sort_stream + fast_hash_reduction,
  incremental_potential.hpp:253-257, reduction.hpp:83-107) of the raw
  19.2 M-triplet stream: rows, cols, n_block_rows and every block value
  bit-exact with the reference's deterministic mode;
* the level-0 partition (partition.hpp:88-159) and the MAS hierarchy
  (hierarchy.hpp:30-100): every level's part_of and agg equal;
* PCG (pcg.hpp:34-88, MAS cemas16, rel_tol 1e-4, restart 250) on the gravity
  rhs of the bench and on b = A x*, x* ~ N(0,1) (seed 5):
  iteration counts within +-2 %, solutions within 1e-5 relative L2 of the
  reference's, and the true error |x - x*| / |x*| within 1.25x of the
  reference's own.
The reference runs on all host cores (parallel mode) for the solves; its
assembly runs in deterministic mode, the bitwise contract."""
import numpy as np
import pytest

import oracle_py as O
import paper_2411_06224_b200 as P
import scenegen as scenes
from paper_2411_06224_b200.context import Context

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
DET = O.ExecPolicy(deterministic=True)
PAR = O.ExecPolicy(deterministic=False)
CAP, LEVELS, TOL, RESTART = 16, 4, 1e-4, 250


@pytest.fixture(scope="module")
def cfg5():
    sc = scenes.CONFIGS["cfg5_stiff_box"]()
    backend = "reference" if O.reference_available() else "restated"
    with O.use_backend(backend):
        fk, fv = O.filter_pinned(sc.keys, sc.vals, sc.pinned)  # private in the reference: restated
        sk, sv = O.sort_stream(fk, fv, DET)
        rows, cols, blocks = O.fast_hash_reduction(sk, sv, sc.n_blocks, DET)
        del sk, sv, fk, fv
        part_of, n_parts = O.partition_block_graph(sc.n_blocks, sc.rest_edges, CAP)
        Am = O.Matrix(sc.n_blocks, rows, cols, blocks)
        H = O.Hierarchy(part_of, n_parts, CAP, O.block_edges(rows, cols), LEVELS)
        levels = [dict(L) for L in H.levels]
        M = O.MasPreconditioner(Am, H)
        xstar = np.random.default_rng(5).standard_normal(3 * sc.n_blocks)
        b_star = O.srbk_spmv(sc.n_blocks, rows, cols, blocks, xstar, DET)
        b_grav = scenes.gravity_rhs(sc)
        solves = {"gravity": (b_grav,) + O.pcg_solve(Am, b_grav, M, TOL, RESTART, 100000, PAR),
                  "xstar": (b_star,) + O.pcg_solve(Am, b_star, M, TOL, RESTART, 100000, PAR)}
    return dict(sc=sc, backend=backend, rows=rows, cols=cols, blocks=blocks, part_of=part_of, n_parts=n_parts,
                levels=levels, xstar=xstar, solves=solves)


@pytest.fixture(scope="module")
def gpu(cfg5):
    sc = cfg5["sc"]
    ctx = Context(0)
    U = ctx.assemble_filtered(sc.keys, sc.vals, sc.n_blocks, sc.pinned)
    l0 = P.partition_block_graph(sc.n_blocks, sc.rest_edges, CAP)
    ctx.set_level0_partition(l0.part_of, l0.n_parts, CAP, LEVELS)
    ctx.build_preconditioner(1)
    yield ctx, U, l0
    ctx.close()


def test_cfg5_assembly_bitwise(cfg5, gpu):
    ctx, U, _ = gpu
    n, rows, cols, blocks = ctx.copy_matrix()
    assert n == cfg5["sc"].n_blocks == 328509
    assert U == len(cfg5["rows"])
    assert np.array_equal(rows, cfg5["rows"]) and np.array_equal(cols, cfg5["cols"])
    assert np.array_equal(blocks.view(np.uint8), cfg5["blocks"].view(np.uint8))


def test_cfg5_partition_and_hierarchy(cfg5, gpu):
    ctx, _, l0 = gpu
    assert l0.n_parts == cfg5["n_parts"] and np.array_equal(l0.part_of, cfg5["part_of"])
    levels = ctx.precond_levels()
    assert len(levels) == len(cfg5["levels"]) == LEVELS
    for a, o in zip(levels, cfg5["levels"]):
        assert a["n_nodes"] == o["n_nodes"] and a["n_parts"] == o["n_parts"]
        assert np.array_equal(a["part_of"], o["part_of"]) and np.array_equal(a["agg"], o["agg"])


@pytest.mark.parametrize("rhs", ["gravity", "xstar"])
def test_cfg5_pcg(cfg5, gpu, rhs):
    ctx = gpu[0]
    b, xo, ro = cfg5["solves"][rhs]
    x, r = ctx.pcg(b, TOL, RESTART, 100000)
    assert r.converged and ro["converged"]
    assert abs(r.iters - ro["iters"]) <= max(1, 0.02 * ro["iters"]), (r.iters, ro["iters"])
    rel = np.linalg.norm(x - xo) / np.linalg.norm(xo)
    line = f"cfg5 {rhs}: gpu {r.iters} iters, {cfg5['backend']} {ro['iters']}, |x - x_ref| / |x_ref| = {rel:.2e}"
    if rhs == "xstar":
        xs = cfg5["xstar"]
        eg = np.linalg.norm(x - xs) / np.linalg.norm(xs)
        eo = np.linalg.norm(xo - xs) / np.linalg.norm(xs)
        line += f", true error gpu {eg:.3e} vs reference {eo:.3e}"
        assert eg <= 1.25 * eo
    print(line)
    assert rel <= 1e-5
