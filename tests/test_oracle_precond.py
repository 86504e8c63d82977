"""Pins the oracle's partition / hierarchy / MAS / block-Jacobi / PCG
restatement against the reference's own tests: proj/tests/test_precond.cpp,
the PCG section of proj/tests/test_solver.cpp:79-130 and
tools/verify_suites.hpp:645-667 (mas_fixture)."""
import numpy as np
import pytest

import oracle_py as O
from helpers import chain_spd_system, dense_from, make_spd_system, restriction_matrix, sixteen_slot_graph_edges

# every test runs on the restatement and on the compiled reference (conftest)
pytestmark = pytest.mark.usefixtures("oracle_backend")


def test_subdomain_count():  # test_precond.cpp:71-78
    assert O.subdomain_count(100, 16, 1) == 7
    assert O.subdomain_count(100, 16, 0) == 7
    assert O.subdomain_count(16, 16, 0) == 1
    assert O.subdomain_count(17, 16, 0) == 2
    assert O.subdomain_count(100, 32, 0) == 4
    assert O.subdomain_count(1, 16, 0) == 1


def test_chunk_partition():  # :80-86
    part, n = O.chunk_partition(10, 4)
    assert n == 3 and list(part) == [0, 0, 0, 0, 1, 1, 1, 1, 2, 2]
    assert O.chunk_partition(16, 4)[1] == 4
    assert O.chunk_partition(0, 4)[1] == 0


def test_graph_partition_fixtures():  # :88-128
    part, n = O.partition_block_graph(16, sixteen_slot_graph_edges(), 4)
    assert n == 4
    for s in (0, 13, 15, 2):
        assert part[s] == 0
    for s in (1, 3, 5, 7):
        assert part[s] == 1
    assert part[4] == 2 and part[8] == 3
    pairs = [(2 * i, 2 * i + 1) for i in range(7)]
    q, nq = O.partition_block_graph(14, pairs, 4)
    assert nq == 4 and list(np.bincount(q)) == [4, 4, 4, 2]
    path = [(i, i + 1) for i in range(99)]
    r, nr = O.partition_block_graph(100, path, 16)
    assert nr == O.subdomain_count(100, 16, 0)
    assert np.all(np.diff(r) >= 0)
    sizes = np.bincount(r)
    assert sizes.max() <= 16 and sizes.min() >= 14


EXPECT_L1 = [0, 1, 2, 1, 3, 4, 5, 4, 6, 6, 6, 6, 7, 8, 7, 8]
EXPECT_L2 = [0, 1, 0, 1, 2, 1, 2, 1, 3, 3, 3, 3, 2, 0, 2, 0]


def test_hierarchy_fixtures():  # :130-177
    edges = sixteen_slot_graph_edges()
    part, n = O.chunk_partition(16, 4)
    h = O.Hierarchy(part, n, 4, edges, 8)
    assert h.n_levels() == 3
    assert h.levels[1]["n_nodes"] == 9 and h.levels[1]["n_parts"] == 3
    assert list(h.levels[1]["agg"]) == EXPECT_L1
    assert h.levels[2]["n_nodes"] == 4 and h.levels[2]["n_parts"] == 1
    assert list(h.levels[2]["agg"]) == EXPECT_L2

    part, n = O.partition_block_graph(16, edges, 4)
    h = O.Hierarchy(part, n, 4, edges, 8)
    assert h.n_levels() == 2
    assert h.levels[1]["n_nodes"] == 4 and h.levels[1]["n_parts"] == 1
    assert list(h.levels[1]["agg"]) == EXPECT_L2

    part, n = O.chunk_partition(16, 4)
    assert O.Hierarchy(part, n, 4, edges, 2).n_levels() == 2
    assert O.Hierarchy(part, n, 4, [], 8).n_levels() == 1


def test_mas_fixture_suite():  # verify_suites.hpp:645-667 (acceptance #5)
    edges = sixteen_slot_graph_edges()
    part, n = O.partition_block_graph(16, edges, 4)
    hc = O.Hierarchy(part, n, 4, edges, 4)
    assert hc.n_levels() == 2 and hc.levels[-1]["n_parts"] == 1
    part, n = O.chunk_partition(16, 4)
    hm = O.Hierarchy(part, n, 4, edges, 4)
    assert hm.n_levels() == 3


def _random_edges(rng, v, count):
    pick = O.UniformInt(0, v - 1)
    edges = []
    for _ in range(count):
        a, b = pick(rng), pick(rng)
        if a == b:
            continue
        edges.append((min(a, b), max(a, b)))
    return sorted(set(edges))


def test_level_matrices_and_apply():  # :179-226
    rng = O.Rng(71)
    v = 30
    edges = _random_edges(rng, v, 70)
    rows, cols, blocks = make_spd_system(v, edges, rng)
    Ad = dense_from(v, rows, cols, blocks)
    np.linalg.cholesky(Ad)
    be = O.block_edges(rows, cols)
    part, n = O.partition_block_graph(v, be, 8)
    h = O.Hierarchy(part, n, 8, be, 4)
    A = O.Matrix(v, rows, cols, blocks)
    M = O.MasPreconditioner(A, h)
    assert M.n_levels() == h.n_levels()
    for l in range(h.n_levels()):
        for s in range(h.levels[l]["n_parts"]):
            R = restriction_matrix(h.levels, v, l, s)
            expect = R @ Ad @ R.T
            got = M.level_matrix(l, s)
            assert got.shape == expect.shape
            assert np.linalg.norm(got - expect) <= 1e-12 * (1 + np.linalg.norm(expect))
    u = O.UniformReal(-1, 1)
    r = u.fill(rng, 3 * v)
    z = M.apply(r)
    expect = np.zeros(3 * v)
    for l in range(h.n_levels()):
        for s in range(h.levels[l]["n_parts"]):
            R = restriction_matrix(h.levels, v, l, s)
            D = R @ Ad @ R.T
            expect += R.T @ np.linalg.solve(D, R @ r)
    assert np.linalg.norm(z - expect) <= 1e-10 * np.linalg.norm(expect)


def test_apply_symmetric_positive():  # :228-253
    rng = O.Rng(81)
    edges = [(i, i + 1) for i in range(19)]
    rows, cols, blocks = make_spd_system(20, edges, rng)
    be = O.block_edges(rows, cols)
    part, n = O.partition_block_graph(20, be, 6)
    h = O.Hierarchy(part, n, 6, be, 4)
    M = O.MasPreconditioner(O.Matrix(20, rows, cols, blocks), h)
    u = O.UniformReal(-1, 1)
    for _ in range(20):
        r1 = np.empty(60)
        r2 = np.empty(60)
        for i in range(60):
            r1[i] = u(rng)
            r2[i] = u(rng)
        z1, z2 = M.apply(r1), M.apply(r2)
        assert abs(r2 @ z1 - r1 @ z2) <= 1e-10 * (abs(r1 @ z1) + abs(r2 @ z2))
        assert r1 @ z1 > 0


def test_single_covering_subdomain_exact():  # :255-274
    rng = O.Rng(91)
    edges = [(i, i + 1) for i in range(9)]
    rows, cols, blocks = make_spd_system(10, edges, rng)
    be = O.block_edges(rows, cols)
    part, n = O.partition_block_graph(10, be, 16)
    h = O.Hierarchy(part, n, 16, be, 4)
    assert h.n_levels() == 1 and h.levels[0]["n_parts"] == 1
    M = O.MasPreconditioner(O.Matrix(10, rows, cols, blocks), h)
    Ad = dense_from(10, rows, cols, blocks)
    u = O.UniformReal(-1, 1)
    x = u.fill(rng, 30)
    z = M.apply(Ad @ x)
    assert np.linalg.norm(z - x) <= 1e-10 * np.linalg.norm(x)


def test_block_jacobi_exact():  # :276-293
    rng = O.Rng(101)
    rows, cols, blocks = make_spd_system(4, [(0, 1), (1, 2), (0, 3)], rng)
    M = O.BlockJacobiPreconditioner(O.Matrix(4, rows, cols, blocks))
    Ad = dense_from(4, rows, cols, blocks)
    u = O.UniformReal(-1, 1)
    r = u.fill(rng, 12)
    z = M.apply(r)
    for i in range(4):
        expect = np.linalg.solve(Ad[3 * i:3 * i + 3, 3 * i:3 * i + 3], r[3 * i:3 * i + 3])
        assert np.linalg.norm(z[3 * i:3 * i + 3] - expect) <= 1e-12 * np.linalg.norm(expect)


def test_indefinite_subdomain_raises():  # mas.hpp:66-81 retry rule
    rows = np.array([0], np.uint32)
    cols = np.array([0], np.uint32)
    blocks = np.array([np.diag([-1.0, 1.0, 1.0]).T.reshape(-1)])
    part, n = O.chunk_partition(1, 4)
    h = O.Hierarchy(part, n, 4, [], 4)
    with pytest.raises(RuntimeError, match="indefinite"):
        O.MasPreconditioner(O.Matrix(1, rows, cols, blocks), h)
    # a singular (PSD) diagonal is rescued by the first shift
    blocks = np.array([np.diag([0.0, 1.0, 1.0]).T.reshape(-1)])
    M = O.MasPreconditioner(O.Matrix(1, rows, cols, blocks), h)
    assert M.shifts() == (1 if O.backend() == "restated" else -1)  # the reference does not count shifts


# ------------------------------------------------------------------ PCG ----
@pytest.fixture
def chain():  # test_solver.cpp:79-88
    rng = O.Rng(11)
    v = 20
    rows, cols, blocks = chain_spd_system(v, rng)
    Ad = dense_from(v, rows, cols, blocks)
    u = O.UniformReal(-1, 1)
    b = u.fill(rng, 3 * v)
    return v, rows, cols, blocks, Ad, b


def test_pcg_block_jacobi(chain):  # :90-97
    v, rows, cols, blocks, Ad, b = chain
    A = O.Matrix(v, rows, cols, blocks)
    x, r = O.pcg_solve(A, b, O.BlockJacobiPreconditioner(A), 1e-8, 250, 10000)
    assert r["converged"]
    assert np.linalg.norm(Ad @ x - b) <= 1e-6 * np.linalg.norm(b)


def test_pcg_exact_mas_one_iteration(chain):  # :99-111
    v, rows, cols, blocks, Ad, b = chain
    be = O.block_edges(rows, cols)
    part, n = O.partition_block_graph(v, be, 64)
    h = O.Hierarchy(part, n, 64, be, 4)
    assert h.levels[0]["n_parts"] == 1
    A = O.Matrix(v, rows, cols, blocks)
    x, r = O.pcg_solve(A, b, O.MasPreconditioner(A, h), 1e-4, 250, 10000)
    assert r["converged"] and r["iters"] == 1
    assert np.linalg.norm(Ad @ x - b) <= 1e-8 * np.linalg.norm(b)


def test_pcg_restart_path(chain):  # :113-120
    v, rows, cols, blocks, Ad, b = chain
    A = O.Matrix(v, rows, cols, blocks)
    x, r = O.pcg_solve(A, b, O.BlockJacobiPreconditioner(A), 1e-8, 1, 10000)
    assert r["converged"]
    assert np.linalg.norm(Ad @ x - b) <= 1e-6 * np.linalg.norm(b)


def test_pcg_zero_rhs(chain):  # :122-129
    v, rows, cols, blocks, Ad, b = chain
    A = O.Matrix(v, rows, cols, blocks)
    x, r = O.pcg_solve(A, np.zeros(3 * v), O.BlockJacobiPreconditioner(A), 1e-4, 250, 100)
    assert r["converged"] and r["iters"] == 0 and np.linalg.norm(x) == 0


def test_stiff_beam_cemas_vs_jacobi_ratio():
    """Acceptance #6 (acceptance.cpp:121-164) analogue on the
    beam's first Newton system (rest state, pinned x=0 face, b = M dt^2 g):
    cemas16 needs <= 0.6x the block-Jacobi PCG iterations. Also pins the
    hierarchy sizes of SURVEY.md Appendix B (371/62/34/17, 513 L1 nodes)."""
    import paper_2411_06224_b200 as P
    import scenegen as scenes

    sc = scenes.CONFIGS["stiff_beam"]()
    det = O.ExecPolicy(deterministic=True)
    fk, fv = O.filter_pinned(sc.keys, sc.vals, sc.pinned)
    sk, sv = O.sort_stream(fk, fv, det)
    rows, cols, blocks = O.fast_hash_reduction(sk, sv, sc.n_blocks, det)
    A = O.Matrix(sc.n_blocks, rows, cols, blocks)
    l0 = P.partition_block_graph(sc.n_blocks, sc.rest_edges, 16)
    H = O.Hierarchy(l0.part_of, l0.n_parts, 16, O.block_edges(rows, cols), 4)
    assert [(L["n_nodes"], L["n_parts"]) for L in H.levels] == [(5040, 371), (513, 62), (197, 34), (169, 17)]
    b = scenes.gravity_rhs(sc)
    _, rm = O.pcg_solve(A, b, O.MasPreconditioner(A, H), 1e-4, 250, 100000, det)
    _, rj = O.pcg_solve(A, b, O.BlockJacobiPreconditioner(A), 1e-4, 250, 100000, det)
    assert rm["converged"] and rj["converged"]
    assert rm["iters"] / rj["iters"] <= 0.6, (rm["iters"], rj["iters"])
