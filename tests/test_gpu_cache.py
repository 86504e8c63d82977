"""Hierarchy reuse (ADIPC_OPT_CACHE_HIERARCHY): the MAS hierarchy is a pure
function of (level-0 partition, sparsity pattern, max_levels), so reusing it
while the pattern hash is unchanged must give the identical hierarchy and the
preconditioner a fresh build gives (to rounding); new values with the same pattern must be re-restricted and
re-inverted; a new pattern must trigger a rebuild."""
import numpy as np
import pytest

import paper_2411_06224_b200 as P
from paper_2411_06224_b200 import _lib
import scenegen as scenes
from paper_2411_06224_b200.context import Context

pytestmark = pytest.mark.gpu


def _setup(ctx, sc, scale=1.0, drop_pin=False):
    pinned = sc.pinned.copy()
    if drop_pin:
        pinned[np.flatnonzero(pinned)[:10]] = 0  # changes the pattern
    fk, fv = ctx.filter_pinned(sc.keys, sc.vals * scale, pinned)
    ctx.assemble(fk, fv, sc.n_blocks)


def test_cache_reuse_is_exact():
    sc = scenes.CONFIGS["stiff_beam"]()
    l0 = P.partition_block_graph(sc.n_blocks, sc.rest_edges, 16)
    b = scenes.gravity_rhs(sc)
    fresh, cached = Context(0), Context(0)
    for c in (fresh, cached):
        c.set_level0_partition(l0.part_of, l0.n_parts, 16, 4)
    cached.set_option(_lib.OPT_CACHE_HIERARCHY, 1)
    for scale, drop in ((1.0, False), (1.7, False), (1.7, True), (1.0, False)):
        outs = []
        for c in (fresh, cached):
            _setup(c, sc, scale, drop)
            c.build_preconditioner(_lib.PRECOND_MAS)
            outs.append((c.precond_levels(), c.precond_apply(b), c.pcg(b, 1e-4, 250, 10000)))
        (lf, zf, (xf, rf)), (lc, zc, (xc, rc)) = outs
        assert len(lf) == len(lc)
        for a, o in zip(lf, lc):
            assert np.array_equal(a["agg"], o["agg"]) and np.array_equal(a["part_of"], o["part_of"])
        # coarse restrictions accumulate with fp64 atomics, so two builds agree
        # to rounding, not bitwise
        assert np.linalg.norm(zf - zc) <= 1e-10 * np.linalg.norm(zf)
        # ... and so can converged iteration counts: the contract is +-2 %
        assert abs(rf.iters - rc.iters) <= max(1, 0.02 * rc.iters)
        assert np.linalg.norm(xf - xc) <= 1e-6 * np.linalg.norm(xf)
    fresh.close()
    cached.close()
