"""Pins the oracle (oracle/oracle.hpp) against the reference's own sparse
tests: proj/tests/test_block_sparse.cpp (each case cites its lines) with the
same seeds and the same libstdc++ std::mt19937 draw sequences."""
import numpy as np
import pytest

import oracle_py as O
from helpers import Stream, abd_jacobian, cm, dense_from, map_accumulate, nat, vec3_draw

# every test runs on the restatement and on the compiled reference (conftest)
pytestmark = pytest.mark.usefixtures("oracle_backend")

DET = O.ExecPolicy(deterministic=True)


def test_key_round_trip():  # test_block_sparse.cpp:61-70
    vals = [0, 1, 77, 0x7FFFFFFF, 0xFFFFFFFF]
    for r in vals:
        for c in vals:
            k = O.make_block_key(r, c)
            assert k >> 32 == r and k & 0xFFFFFFFF == c
    assert O.make_block_key(0, 1) < O.make_block_key(1, 0)


def test_emission_canonicalizes_and_sort_is_stable():  # :72-91
    B1 = np.array([[1, 2, 3], [4, 5, 6], [7, 8, 9]], float)
    B2 = 2 * np.eye(3)
    B3 = np.array([[0, 1, 0], [1, 0, 2], [0, 2, 0]], float)
    s = Stream()
    s.emit(2, 1, B1)
    s.emit(1, 2, B2)
    s.emit(1, 1, B3)
    keys, vals = O.sort_stream(*s.arrays())
    assert list(keys) == [O.make_block_key(1, 1), O.make_block_key(1, 2), O.make_block_key(1, 2)]
    assert np.array_equal(vals[0], cm(B3))
    assert np.array_equal(vals[1], cm(B1.T))
    assert np.array_equal(vals[2], cm(B2))


def test_radix_sort_stable_and_ordered():  # :93-101
    rng = O.Rng(7)
    keys, vals = O.random_stream(rng, 40, 5000)
    sk, sv = O.sort_stream(keys, vals)
    assert np.all(sk[1:] >= sk[:-1])
    assert np.array_equal(sk, np.sort(keys))
    # stability: the permutation of equal keys preserves emission order
    k2, perm = O.radix_sort_keys(keys)
    assert np.array_equal(k2, sk)
    order = np.lexsort((np.arange(len(keys)), keys))
    assert np.array_equal(perm, order)


def test_hash_reduction_matches_map_oracle_bitwise():  # :103-123
    rng = O.Rng(11)
    for _ in range(20):
        keys, vals = O.random_stream(rng, 12, 400)
        oracle = map_accumulate(keys, vals)
        sk, sv = O.sort_stream(keys, vals, DET)
        rows, cols, blocks = O.fast_hash_reduction(sk, sv, 12, DET)
        assert len(blocks) == len(oracle)
        for r, c, b in zip(rows, cols, blocks):
            k = (int(r) << 32) | int(c)
            assert np.array_equal(b, oracle[k])  # bitwise
        kk = (rows.astype(np.uint64) << np.uint64(32)) | cols
        assert np.all(kk[1:] > kk[:-1])


def test_parallel_hash_reduction_within_1e12():  # :125-139
    rng = O.Rng(13)
    keys, vals = O.random_stream(rng, 20, 3000)
    oracle = map_accumulate(keys, vals)
    par = O.ExecPolicy(threads=4, lane_width=8)
    sk, sv = O.sort_stream(keys, vals, par)
    rows, cols, blocks = O.fast_hash_reduction(sk, sv, 20, par)
    assert len(blocks) == len(oracle)
    for r, c, b in zip(rows, cols, blocks):
        want = oracle[(int(r) << 32) | int(c)]
        assert np.linalg.norm(b - want) <= 1e-12 * max(1.0, np.linalg.norm(want))


def test_lane_walkthrough():  # :141-153
    Oseg = [0, 0, 0, 1, 1, 1, 2, 2]
    V = np.ones(8)
    for det in (True, False):
        pol = O.ExecPolicy(deterministic=det, lane_width=8, threads=2)
        R = O.fast_segment_reduction(Oseg, V, 3, pol)
        assert list(R) == [3.0, 3.0, 2.0]


def test_segment_spanning_lane_groups():  # :155-164
    R = O.fast_segment_reduction([0] * 12, np.ones(12), 1, O.ExecPolicy(lane_width=4, threads=3))
    assert list(R) == [12.0]


def test_segment_size_mismatch_raises():  # reduction.hpp:34
    import pytest

    with pytest.raises(ValueError):
        O.fast_segment_reduction([0, 0, 1], np.ones(2), 2)


def test_lane_width_invariance():  # :166-194
    rng = O.Rng(17)
    val = O.Normal(0.0, 1.0)
    adv = O.UniformInt(0, 4)
    n = 4000
    Oseg = np.empty(n, np.int32)
    V = np.empty(n)
    seg = 0
    for i in range(n):
        if i > 0 and adv(rng) == 0:
            seg += 1
        Oseg[i] = seg
        V[i] = val(rng)
    ref = O.fast_segment_reduction(Oseg, V, seg + 1, DET)
    for w in (4, 8, 32):
        R = O.fast_segment_reduction(Oseg, V, seg + 1, O.ExecPolicy(lane_width=w, threads=4))
        assert np.all(np.abs(R - ref) <= 1e-12 * np.maximum(1.0, np.abs(ref)))
    again = O.fast_segment_reduction(Oseg, V, seg + 1, DET)
    assert np.array_equal(again, ref)


def test_spmv_two_row_fixture():  # :196-211
    rows = np.array([0, 0, 1], np.uint32)
    cols = np.array([0, 1, 1], np.uint32)
    blocks = np.array([cm(2 * np.eye(3)), cm(np.eye(3)), cm(2 * np.eye(3))])
    for det in (True, False):
        y = O.srbk_spmv(2, rows, cols, blocks, np.ones(6), O.ExecPolicy(deterministic=det, threads=2))
        assert np.array_equal(y, np.full(6, 3.0))


def test_spmv_dense_mirror():  # :213-237
    rng = O.Rng(23)
    for trial in range(10):
        keys, vals = O.random_stream(rng, 15, 800)
        pol = O.ExecPolicy(threads=4 if trial % 2 else 1, lane_width=4)
        sk, sv = O.sort_stream(keys, vals, pol)
        rows, cols, blocks = O.fast_hash_reduction(sk, sv, 15, pol)
        D = dense_from(15, rows, cols, blocks)
        val = O.Normal(0.0, 1.0)
        x = val.fill(rng, 45)
        y = O.srbk_spmv(15, rows, cols, blocks, x, pol)
        yd = D @ x
        for i in range(15):
            assert np.linalg.norm(y[3 * i:3 * i + 3] - yd[3 * i:3 * i + 3]) <= 1e-12 * max(1.0, np.linalg.norm(yd))


def test_split_fixture():  # :239-264
    H = np.array([[100.0 * i + j for j in range(12)] for i in range(12)])
    keys, vals = O.split(O.SPLIT_12x12, 4, 8, H)
    assert len(keys) == 16
    for ti in range(4):
        for tj in range(4):
            e = 4 * ti + tj
            assert keys[e] >> 32 == 4 + ti and keys[e] & 0xFFFFFFFF == 8 + tj
            assert np.array_equal(vals[e], cm(H[3 * ti:3 * ti + 3, 3 * tj:3 * tj + 3]))
    C = np.random.default_rng(0).uniform(-1, 1, (12, 3))
    keys, vals = O.split(O.SPLIT_12x3, 4, 2, C)
    assert len(keys) == 4
    for t in range(4):
        assert keys[t] >> 32 == 2 and keys[t] & 0xFFFFFFFF == 4 + t
        assert np.array_equal(vals[t], cm(C[3 * t:3 * t + 3, :].T))
    keys, vals = O.split(O.SPLIT_SYM_12x12, 4, 0, H)
    assert len(keys) == 10
    keys, vals = O.split(O.SPLIT_3x12, 9, 4, C.T)
    assert [int(k >> 32) for k in keys] == [4, 5, 6, 7]  # below diagonal -> transposed


def make_test_map(n_fem, n_bodies, vpb, rng):  # :268-283
    val = O.Normal(0.0, 1.0)
    body, jac = [], []
    for b in range(n_bodies):
        for _ in range(vpb):
            rest = vec3_draw(val, rng)
            body.append(b)
            jac.append(abd_jacobian(rest))
    return body, jac


def node_jacobian_matrix(n_fem, body, jac, n_nodes, n_blocks):
    dofJ = np.zeros((3 * n_nodes, 3 * n_blocks))
    for i in range(n_nodes):
        if i < n_fem:
            dofJ[3 * i:3 * i + 3, 3 * i:3 * i + 3] = np.eye(3)
        else:
            base = n_fem + 4 * body[i - n_fem]
            dofJ[3 * i:3 * i + 3, 3 * base:3 * base + 12] = jac[i - n_fem]
    return dofJ


def jac36(jac):
    return np.array([np.ascontiguousarray(J.T).reshape(-1) for J in jac]) if jac else np.zeros((0, 36))


def test_two_level_equals_naive_sandwich():  # :287-334
    rng = O.Rng(31)
    n_fem, n_bodies, vpb = 6, 2, 5
    body, jac = make_test_map(n_fem, n_bodies, vpb, rng)
    n_nodes = n_fem + n_bodies * vpb
    n_blocks = n_fem + 4 * n_bodies
    val = O.Normal(0.0, 1.0)
    pick = O.UniformInt(0, n_nodes - 1)
    s = Stream()
    naive = np.zeros((3 * n_blocks, 3 * n_blocks))
    dofJ = node_jacobian_matrix(n_fem, body, jac, n_nodes, n_blocks)
    for _ in range(60):
        nd = sorted(pick(rng) for _ in range(4))
        if len(set(nd)) != 4:
            continue
        L = val.fill(rng, 144).reshape(12, 12).T  # L.data()[k] column-major
        H = L + L.T
        sel = np.zeros((12, 3 * n_nodes))
        for a in range(4):
            sel[3 * a:3 * a + 3, 3 * nd[a]:3 * nd[a] + 3] = np.eye(3)
            for b in range(a, 4):
                s.emit(nd[a], nd[b], H[3 * a:3 * a + 3, 3 * b:3 * b + 3])
        S = sel @ dofJ
        naive += S.T @ H @ S
    keys, vals = s.arrays()
    for det in (True, False):
        pol = O.ExecPolicy(deterministic=det, threads=1 if det else 4)
        tk, tv = O.two_level_abd_reduce(keys, vals, n_fem, n_bodies, body, jac36(jac), pol)
        sk, sv = O.sort_stream(tk, tv, pol)
        rows, cols, blocks = O.fast_hash_reduction(sk, sv, n_blocks, pol)
        D = dense_from(n_blocks, rows, cols, blocks)
        assert np.linalg.norm(D - naive) / np.linalg.norm(naive) <= 1e-10


def test_filter_pinned():  # incremental_potential.hpp:410-425
    s = Stream()
    s.emit(0, 0, np.eye(3) * 5)
    s.emit(0, 1, np.ones((3, 3)))
    s.emit(1, 2, np.ones((3, 3)) * 2)
    s.emit(2, 2, np.eye(3) * 7)
    keys, vals = s.arrays()
    fk, fv = O.filter_pinned(keys, vals, np.array([0, 1, 0], np.uint8))
    assert [(int(k >> 32), int(k & 0xFFFFFFFF)) for k in fk] == [(0, 0), (2, 2), (1, 1)]
    assert np.array_equal(fv[2], cm(np.eye(3)))
