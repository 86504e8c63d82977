"""Input generators of `adipc verify kernel-oracles`
(tools/verify_suites.hpp:140-343), consuming the shared std::mt19937 in the
reference's exact order. Shared by the oracle pin tests and the GPU parity
tests (which run the same 1000-case suites through the C-ABI)."""
import numpy as np

import oracle_py as O
from helpers import Stream, abd_jacobian, vec3_draw


def segment_cases(rng, trials=1000):  # :161-191
    length = O.UniformInt(1, 400)
    adv = O.UniformInt(0, 3)
    val = O.Normal(0.0, 1.0)
    for _ in range(trials):
        n = length(rng)
        Oseg = np.empty(n, np.int32)
        V = np.empty(n)
        seg = 0
        for i in range(n):
            if i > 0 and adv(rng) == 0:
                seg += 1
            Oseg[i] = seg
            V[i] = val(rng)
        yield Oseg, V, seg + 1


def hash_cases(rng, trials=1000):  # :192-215
    nb = O.UniformInt(2, 24)
    ne = O.UniformInt(1, 240)
    for _ in range(trials):
        n_blocks = nb(rng)
        keys, vals = O.random_stream(rng, n_blocks, ne(rng))
        yield n_blocks, keys, vals


def spmv_cases(rng, trials=1000):  # :217-252
    nb = O.UniformInt(1, 16)
    ne = O.UniformInt(1, 150)
    val = O.Normal(0.0, 1.0)
    det = O.ExecPolicy(deterministic=True)
    for _ in range(trials):
        n_blocks = nb(rng)
        keys, vals = O.random_stream(rng, n_blocks, ne(rng))
        sk, sv = O.sort_stream(keys, vals, det)
        rows, cols, blocks = O.fast_hash_reduction(sk, sv, n_blocks, det)
        x = val.fill(rng, 3 * n_blocks)
        yield n_blocks, rows, cols, blocks, x


def abd_cases(rng, trials=1000):  # :254-343
    nf = O.UniformInt(0, 5)
    nbod = O.UniformInt(0, 2)
    vpb = O.UniformInt(1, 4)
    nc = O.UniformInt(1, 12)
    val = O.Normal(0.0, 1.0)
    for _ in range(trials):
        while True:
            n_fem = nf(rng)
            n_bodies = nbod(rng)
            body, jac = [], []
            for b in range(n_bodies):
                nv = vpb(rng)
                for _v in range(nv):
                    rest = vec3_draw(val, rng)
                    body.append(b)
                    jac.append(abd_jacobian(rest))
            if n_fem + len(body) >= 4:
                break
        n_nodes = n_fem + len(body)
        n_blocks = n_fem + 4 * n_bodies
        dofJ = np.zeros((3 * n_nodes, 3 * n_blocks))
        for i in range(n_nodes):
            if i < n_fem:
                dofJ[3 * i:3 * i + 3, 3 * i:3 * i + 3] = np.eye(3)
            else:
                base = n_fem + 4 * body[i - n_fem]
                dofJ[3 * i:3 * i + 3, 3 * base:3 * base + 12] = jac[i - n_fem]
        pick = O.UniformInt(0, n_nodes - 1)
        s = Stream()
        naive = np.zeros((3 * n_blocks, 3 * n_blocks))
        made, guard = 0, 0
        while made < nc(rng) and guard < 200:
            guard += 1
            nd = sorted(pick(rng) for _ in range(4))
            if len(set(nd)) != 4:
                continue
            L = val.fill(rng, 144).reshape(12, 12).T
            H = L + L.T
            sel = np.zeros((12, 3 * n_nodes))
            for a in range(4):
                sel[3 * a:3 * a + 3, 3 * nd[a]:3 * nd[a] + 3] = np.eye(3)
                for b in range(a, 4):
                    s.emit(nd[a], nd[b], H[3 * a:3 * a + 3, 3 * b:3 * b + 3])
            S = sel @ dofJ
            naive += S.T @ H @ S
            made += 1
        if not s.keys:
            continue
        keys, vals = s.arrays()
        jac36 = np.array([np.ascontiguousarray(J.T).reshape(-1) for J in jac]) if jac else np.zeros((0, 36))
        yield dict(n_fem=n_fem, n_bodies=n_bodies, body=np.array(body, np.int32), jac36=jac36,
                   n_nodes=n_nodes, n_blocks=n_blocks, keys=keys, vals=vals, naive=naive)
