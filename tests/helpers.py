"""Shared test helpers: dense mirrors and brute-force oracles restated from
the reference tests (proj/tests/test_block_sparse.cpp:18-38,
test_precond.cpp:26-67, tools/verify_suites.hpp:95-134)."""
import numpy as np

import oracle_py as O


def cm(M):
    """natural 3x3 -> 9 doubles column-major (Eigen Mat3::data())."""
    return np.ascontiguousarray(np.asarray(M, np.float64).T).reshape(-1)


def nat(v9):
    """9 doubles column-major -> natural 3x3."""
    return np.asarray(v9, np.float64).reshape(3, 3).T


def dense_from(n_block_rows, rows, cols, blocks):
    """test_block_sparse.cpp:30-38: dense symmetric mirror of an upper-stored matrix."""
    D = np.zeros((3 * n_block_rows, 3 * n_block_rows))
    for r, c, b in zip(rows, cols, blocks):
        B = nat(b)
        D[3 * r:3 * r + 3, 3 * c:3 * c + 3] += B
        if r != c:
            D[3 * c:3 * c + 3, 3 * r:3 * r + 3] += B.T
    return D


def map_accumulate(keys, vals):
    """test_block_sparse.cpp:18-28: left-to-right per-key accumulation."""
    acc = {}
    for k, v in zip(keys.tolist(), vals):
        if k in acc:
            acc[k] = acc[k] + v
        else:
            acc[k] = v.copy()
    return acc


class Stream:
    """BlockTripletStream (block_coo.hpp:25-51) built through the oracle's emit."""

    def __init__(self):
        self.keys = []
        self.vals = []

    def emit(self, r, c, M):
        k, v = O.emit(int(r), int(c), cm(M))
        self.keys.append(k)
        self.vals.append(v)

    def arrays(self):
        if not self.keys:
            return np.zeros(0, np.uint64), np.zeros((0, 9))
        return np.array(self.keys, np.uint64), np.array(self.vals, np.float64)


def make_spd_system(v, edges, rng, policy=None):
    """test_precond.cpp:26-40 (graph-Laplacian SPD block system)."""
    s = Stream()
    for a, b in edges:
        k = nat(O.random_spd3(rng, 0.1))
        s.emit(a, a, k)
        s.emit(b, b, k)
        s.emit(a, b, -k)
    for i in range(v):
        s.emit(i, i, nat(O.random_spd3(rng, 2.0)))
    keys, vals = s.arrays()
    keys, vals = O.sort_stream(keys, vals, policy)
    return O.fast_hash_reduction(keys, vals, v, policy)


def chain_spd_system(v, rng, policy=None):
    """test_solver.cpp:23-35."""
    s = Stream()
    for i in range(v - 1):
        k = nat(O.random_spd3(rng, 0.1))
        s.emit(i, i, k)
        s.emit(i + 1, i + 1, k)
        s.emit(i, i + 1, -k)
    for i in range(v):
        s.emit(i, i, nat(O.random_spd3(rng, 2.0)))
    keys, vals = s.arrays()
    keys, vals = O.sort_stream(keys, vals, policy)
    return O.fast_hash_reduction(keys, vals, v, policy)


def restriction_matrix(levels, n_slots, level, sub):
    """test_precond.cpp:54-67."""
    hl = levels[level]
    pos_of = -np.ones(hl["n_nodes"], np.int64)
    m = 0
    for node in range(hl["n_nodes"]):
        if hl["part_of"][node] == sub:
            pos_of[node] = m
            m += 1
    R = np.zeros((3 * m, 3 * n_slots))
    for slot in range(n_slots):
        node = hl["agg"][slot]
        if pos_of[node] < 0:
            continue
        for k in range(3):
            R[3 * pos_of[node] + k, 3 * slot + k] = 1
    return R


def abd_jacobian(rest):
    """scene/mesh.hpp:196-201: J = [I3 | diag-rows rest^T] (3x12)."""
    J = np.zeros((3, 12))
    J[:, :3] = np.eye(3)
    for r in range(3):
        J[r, 3 + 3 * r:6 + 3 * r] = rest
    return J


def sixteen_slot_graph_edges():
    """precond/fixture_graph.hpp:12-15."""
    return [(0, 13), (1, 3), (2, 15), (3, 5), (4, 12), (5, 7),
            (6, 14), (8, 9), (9, 10), (10, 11), (12, 14), (13, 15)]


def vec3_draw(dist, rng):
    """`Vec3 rest(val(rng), val(rng), val(rng))` as g++ compiles it: the
    constructor arguments are evaluated right to left (checked with g++ 13 on
    this image), so the first draw lands in z."""
    d1 = dist(rng)
    d2 = dist(rng)
    d3 = dist(rng)
    return np.array([d3, d2, d1])
