"""Restatement (oracle/oracle.hpp) against the reference's own hot-path code
compiled in place (oracle/_ref, oracle/ref_capi.cpp + the Eigen subset in
oracle/eigen_shim) on the scene configs, outputs compared directly:
integer outputs and deterministic-mode sums bit-exact, Eigen-internal
arithmetic (LLT solves) to rounding. Skipped when neither oracle/_ref nor
/root/reference is present."""
import numpy as np
import pytest

import oracle_py as O
import scenegen as scenes

DET = O.ExecPolicy(deterministic=True)
PAR = O.ExecPolicy(deterministic=False, threads=4)

pytestmark = pytest.mark.skipif(not O.reference_available(), reason="oracle/_ref unavailable")


def both(fn):
    with O.use_backend("restated"):
        a = fn()
    with O.use_backend("reference"):
        b = fn()
    return a, b


def bits(x):
    x = np.asarray(x)
    return x.view(np.uint8) if x.dtype == np.float64 else x


def assert_same(a, b):
    if isinstance(a, (tuple, list)):
        assert len(a) == len(b)
        for u, v in zip(a, b):
            assert_same(u, v)
    else:
        assert np.array_equal(bits(a), bits(b))


def assembled(sc):
    fk, fv = O.filter_pinned(sc.keys, sc.vals, sc.pinned)
    sk, sv = O.sort_stream(fk, fv, DET)
    return O.fast_hash_reduction(sk, sv, sc.n_blocks, DET)


@pytest.mark.parametrize("name", ["cfg1_soft_cube", "stiff_beam", "cfg2_cloth"])
def test_assembly_bitwise(name):
    sc = scenes.CONFIGS[name]()
    a, b = both(lambda: (O.sort_stream(sc.keys, sc.vals, DET), assembled(sc)))
    assert_same(a, b)


@pytest.mark.parametrize("name", ["cfg3_abd_stack", "cfg4_hybrid"])
def test_two_level_bitwise(name):
    sc = scenes.CONFIGS[name]()
    args = (sc.node_keys, sc.node_vals, sc.n_fem, sc.n_bodies, sc.abd_body, sc.jac36)
    a, b = both(lambda: O.two_level_abd_reduce(*args, DET))
    assert_same(a, b)


def test_spmv_deterministic_bitwise_parallel_close():
    sc = scenes.CONFIGS["cfg1_soft_cube"]()
    rows, cols, blocks = assembled(sc)
    x = np.random.default_rng(3).standard_normal(3 * sc.n_blocks)
    a, b = both(lambda: O.srbk_spmv(sc.n_blocks, rows, cols, blocks, x, DET))
    assert_same(a, b)
    a, b = both(lambda: O.srbk_spmv(sc.n_blocks, rows, cols, blocks, x, PAR))
    assert np.allclose(a, b, rtol=1e-12, atol=1e-12 * np.abs(a).max())


@pytest.mark.parametrize("name", ["cfg1_soft_cube", "stiff_beam"])
def test_partition_hierarchy_mas_pcg(name):
    import paper_2411_06224_b200 as P

    sc = scenes.CONFIGS[name]()
    rows, cols, blocks = assembled(sc)
    b = scenes.gravity_rhs(sc)

    def run():
        part, n_parts = O.partition_block_graph(sc.n_blocks, sc.rest_edges, 16)
        E = O.block_edges(rows, cols)
        H = O.Hierarchy(part, n_parts, 16, E, 4)
        A = O.Matrix(sc.n_blocks, rows, cols, blocks)
        M = O.MasPreconditioner(A, H)
        mats = [M.level_matrix(l, s) for l in range(M.n_levels()) for s in (0, H.levels[l]["n_parts"] - 1)]
        z = M.apply(b)
        x, info = O.pcg_solve(A, b, M, 1e-4, 250, 2000, DET)
        J = O.BlockJacobiPreconditioner(A)
        zj = J.apply(b)
        hier = [(L["n_nodes"], L["n_parts"], L["part_of"], L["agg"]) for L in H.levels]
        return part, E, hier, mats, z, x, info, zj

    ra, rb = both(run)
    # integer outputs + galerkin sums (reference loop order) + Eigen 3x3 inverse: exact
    assert_same(ra[0], rb[0])
    assert_same(ra[1], rb[1])
    assert_same(ra[2], rb[2])
    assert_same(ra[3], rb[3])
    assert_same(ra[7], rb[7])
    # LLT solves: Eigen-internal arithmetic, to rounding
    assert np.linalg.norm(ra[4] - rb[4]) <= 1e-12 * np.linalg.norm(rb[4])
    assert ra[6]["iters"] == rb[6]["iters"] and ra[6]["converged"] and rb[6]["converged"]
    assert np.linalg.norm(ra[5] - rb[5]) <= 1e-9 * np.linalg.norm(rb[5])
    # the product's host partition follows the same rules (host_precond.cpp)
    l0 = P.partition_block_graph(sc.n_blocks, sc.rest_edges, 16)
    assert np.array_equal(l0.part_of, rb[0])


def test_dump_block_coo_text_identical():
    """api.dump_block_coo (the --dump-hessian wire format, srbk_spmv.hpp:52-60)
    is byte-identical to the reference's own dump, including exponents,
    negative zeros and values needing more than 6 significant digits."""
    import io

    from paper_2411_06224_b200 import api as P

    rows, cols, blocks = assembled(scenes.CONFIGS["cfg1_soft_cube"]())
    blocks = blocks.copy()
    blocks[0, :4] = [-0.0, 1e-300, 123456789.0, -2.5e17]
    want = O.reference_dump_block_coo(1728, rows, cols, blocks)
    f = io.StringIO()
    P.dump_block_coo(P.SortedSymBlockCoo(1728, rows, cols, blocks), f)
    assert f.getvalue() == want
    assert want.splitlines()[0] == f"1728 {len(rows)}"
