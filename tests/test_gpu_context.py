"""Context state rules through the C ABI (the advisor's findings of round 1):
a PCG after a reassembly without a preconditioner rebuild solves the CURRENT
matrix (the reference's pcg_solve always uses the A it is given, pcg.hpp:34);
a new level-0 partition invalidates the preconditioner; vectors of the wrong
length are rejected before any device access; two contexts driven from two
host threads at once give the single-thread results."""
import threading

import numpy as np
import pytest

import oracle_py as O
import paper_2411_06224_b200 as P
from paper_2411_06224_b200 import _lib
import scenegen as scenes
from paper_2411_06224_b200.context import Context, InvalidArgument

pytestmark = pytest.mark.gpu
DET = O.ExecPolicy(deterministic=True)


def _beam():
    sc = scenes.CONFIGS["stiff_beam"]()
    fk, fv = O.filter_pinned(sc.keys, sc.vals, sc.pinned)
    l0 = P.partition_block_graph(sc.n_blocks, sc.rest_edges, 16)
    return sc, fk, fv, l0


@pytest.mark.parametrize("kind", [_lib.PRECOND_MAS, _lib.PRECOND_JACOBI])
def test_pcg_after_reassembly_uses_current_matrix(kind):
    sc, fk, fv, l0 = _beam()
    b = scenes.gravity_rhs(sc)
    c = Context(0)
    c.set_level0_partition(l0.part_of, l0.n_parts, 16, 4)
    c.assemble(fk, fv, sc.n_blocks)
    c.build_preconditioner(kind)
    c.assemble(fk, fv * 3.0, sc.n_blocks)  # new values, same pattern, no rebuild
    x, r = c.pcg(b, 1e-8, 250, 100000)
    assert r.converged
    # the true residual against the NEW matrix
    rows, cols, blocks = O.fast_hash_reduction(*O.sort_stream(fk, fv * 3.0, DET), sc.n_blocks, DET)
    Ax = O.srbk_spmv(sc.n_blocks, rows, cols, blocks, x, DET)
    assert np.linalg.norm(b - Ax) <= 1e-5 * np.linalg.norm(b)
    c.close()


def test_new_partition_invalidates_preconditioner():
    sc, fk, fv, l0 = _beam()
    c = Context(0)
    c.set_level0_partition(l0.part_of, l0.n_parts, 16, 4)
    c.assemble(fk, fv, sc.n_blocks)
    c.build_preconditioner(_lib.PRECOND_MAS)
    c.set_level0_partition(l0.part_of, l0.n_parts, 16, 4)
    with pytest.raises(InvalidArgument):
        c.pcg(scenes.gravity_rhs(sc))
    with pytest.raises(InvalidArgument):
        c.precond_apply(scenes.gravity_rhs(sc))
    c.close()


def test_size_mismatch_rejected():
    sc, fk, fv, l0 = _beam()
    c = Context(0)
    c.assemble(fk, fv, sc.n_blocks)
    c.build_preconditioner(_lib.PRECOND_JACOBI)
    short = np.ones(3 * sc.n_blocks - 1)
    for f in (c.spmv, c.precond_apply, c.pcg):
        with pytest.raises(InvalidArgument):
            f(short)
    # a matrix of another size under the old preconditioner
    c.assemble(np.zeros(0, np.uint64), np.zeros((0, 9)), 7)
    with pytest.raises(InvalidArgument):
        c.pcg(np.ones(21))
    c.close()


def test_two_threads_two_contexts():
    """Distinct contexts on distinct host threads: both
    threads solve concurrently and match a solo solve."""
    sc, fk, fv, l0 = _beam()
    b = scenes.gravity_rhs(sc)
    solo = Context(0)
    solo.set_level0_partition(l0.part_of, l0.n_parts, 16, 4)
    solo.assemble(fk, fv, sc.n_blocks)
    solo.build_preconditioner(_lib.PRECOND_MAS)
    x0, r0 = solo.pcg(b, 1e-4, 250, 100000)
    solo.close()
    out, errs = [None, None], []

    def work(i):
        try:
            c = Context(0)
            c.set_level0_partition(l0.part_of, l0.n_parts, 16, 4)
            for _ in range(3):
                c.assemble(fk, fv, sc.n_blocks)
                c.build_preconditioner(_lib.PRECOND_MAS)
                out[i] = c.pcg(b, 1e-4, 250, 100000)
            c.close()
        except Exception as e:  # pragma: no cover - reported below
            errs.append(e)

    ts = [threading.Thread(target=work, args=(i,)) for i in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs
    for x, r in out:
        assert abs(r.iters - r0.iters) <= max(1, 0.02 * r0.iters)
        assert np.linalg.norm(x - x0) <= 1e-6 * np.linalg.norm(x0)
