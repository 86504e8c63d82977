"""Seeded contact inputs for the contact-producer parity tests: stencils whose
closest features cover every region of contact/distance.hpp (vertex, edge
and interior of a triangle; endpoint / interior pairs of two segments, near
parallel segments), distances spread around dhat, ground contacts and lagged
friction constraints (friction.hpp:38-44) with orthonormal tangent frames."""
import numpy as np

import oracle_py as O


def make_case(seed=1, n_pt=600, n_ee=600, n_ground=200, n_fr4=150, n_fr1=60, dhat=1e-2):
    rng = np.random.default_rng(seed)
    pos, pt, ee = [], [], []

    def add(p):
        pos.append(np.asarray(p, np.float64))
        return len(pos) - 1

    for _ in range(n_pt):
        c = rng.normal(0, 1, 3)
        t = [c + rng.normal(0, 0.05, 3) for _ in range(3)]
        n = np.cross(t[1] - t[0], t[2] - t[0])
        n /= np.linalg.norm(n)
        # barycentric target, possibly outside (edge / vertex regions)
        w = rng.uniform(-0.5, 1.2, 3)
        w /= w.sum()
        q = w[0] * t[0] + w[1] * t[1] + w[2] * t[2]
        p = q + n * rng.uniform(0.1, 1.6) * dhat * rng.choice([-1, 1]) + rng.normal(0, 0.3 * dhat, 3)
        pt.append([add(p), add(t[0]), add(t[1]), add(t[2])])
    for k in range(n_ee):
        c = rng.normal(0, 1, 3)
        a0 = c + rng.normal(0, 0.05, 3)
        da = rng.normal(0, 0.05, 3)
        db = da + rng.normal(0, 0.05 if k % 7 else 1e-9, 3)  # a few near-parallel pairs
        s, t = rng.uniform(-0.3, 1.3, 2)
        off = np.cross(da, db)
        off = off / max(np.linalg.norm(off), 1e-30) if np.linalg.norm(off) > 1e-12 else rng.normal(0, 1, 3)
        off /= np.linalg.norm(off)
        pa = a0 + s * da
        b0 = pa + off * rng.uniform(0.1, 1.6) * dhat - t * db + rng.normal(0, 0.2 * dhat, 3)
        ee.append([add(a0), add(a0 + da), add(b0), add(b0 + db)])
    normal = np.array([0.0, 1.0, 0.0])
    height = -5.0
    surf = []
    for _ in range(n_ground):
        p = rng.normal(0, 1, 3)
        p[1] = height + rng.uniform(0.05, 1.8) * dhat
        surf.append(add(p))
    pos = np.array(pos)
    base = pos + rng.normal(0, 0.3 * dhat, pos.shape)
    fr = {"nodes": [], "n": [], "coeff": [], "t1": [], "t2": [], "lam": []}
    for k in range(n_fr4 + n_fr1):
        four = k < n_fr4
        st = pt[k % len(pt)] if four else [surf[k % len(surf)], 0, 0, 0]
        nrm = rng.normal(0, 1, 3)
        nrm /= np.linalg.norm(nrm)
        ref = np.array([0, 1.0, 0]) if abs(nrm[0]) > 0.9 else np.array([1.0, 0, 0])  # friction.hpp:46-50
        t1 = np.cross(nrm, ref)
        t1 /= np.linalg.norm(t1)
        t2 = np.cross(nrm, t1)
        b = rng.uniform(0, 1, 3)
        b /= b.sum()
        fr["nodes"].append(list(st))
        fr["n"].append(4 if four else 1)
        fr["coeff"].append([1, -b[0], -b[1], -b[2]] if four else [1, 0, 0, 0])
        fr["t1"].append(t1)
        fr["t2"].append(t2)
        fr["lam"].append(rng.uniform(0.1, 10.0))
    # a few constraints with (numerically) zero tangential slip
    if fr["nodes"]:
        base[fr["nodes"][0]] = pos[fr["nodes"][0]]
    return O.ContactInput(pos, pt, ee, dhat=dhat, kappa=1e4, ground=(normal, height), surf_verts=surf, friction=fr,
                          fr_base=base, mu=0.3, fr_eps=1e-3 * dhat)


def device_dict(ci, dev="cuda:0"):
    import torch

    t = lambda a, dt=None: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    d = {"pos": t(ci.pos), "pt": t(ci.pt), "ee": t(ci.ee), "dhat": ci.dhat, "kappa": ci.kappa, "ground": ci.ground,
         "surf_verts": t(ci.surf_verts), "mu": ci.mu, "fr_eps": ci.fr_eps}
    if len(ci.fr_n):
        d.update(fr_nodes=t(ci.fr_nodes), fr_n=t(ci.fr_n), fr_coeff=t(ci.fr_coeff), fr_t1=t(ci.fr_t1),
                 fr_t2=t(ci.fr_t2), fr_lambda=t(ci.fr_lambda), fr_base=t(ci.fr_base))
    return d


def make_grid(nx, ny, sx, sy):
    """geometry/shapes.hpp:22-44 (make_grid): vertex id = j nx + i, the
    diagonal alternating with (i + j) parity."""
    verts = np.array([[sx * i / (nx - 1), sy * j / (ny - 1), 0.0] for j in range(ny) for i in range(nx)])
    tris = []
    for j in range(ny - 1):
        for i in range(nx - 1):
            a, b, c, d = j * nx + i, j * nx + i + 1, (j + 1) * nx + i + 1, (j + 1) * nx + i
            if (i + j) % 2 == 0:
                tris += [[a, b, c], [a, c, d]]
            else:
                tris += [[a, b, d], [b, c, d]]
    return verts, np.array(tris, np.int32)


def edges_of(tris):
    """scene/mesh.hpp:84-95 (extract_edges): sorted unique (min, max) pairs."""
    e = np.concatenate([tris[:, [0, 1]], tris[:, [1, 2]], tris[:, [2, 0]]])
    e = np.sort(e, axis=1)
    return np.unique(e, axis=0).astype(np.int32)


def layered_surface(n=6, layers=2, seed=51, noise=0.02):
    """test_contact.cpp:341-360: interleaved cloth patches (shells: every
    vertex, edge and triangle is on the contact surface) plus noise."""
    rng = np.random.default_rng(seed)
    P, T, E = [], [], []
    off = 0
    for layer in range(layers):
        v, t = make_grid(n, n, 1, 1)
        v = v + np.array([0.3 * layer, 0.05 * layer, 0.2 * layer])
        P.append(v)
        T.append(t + off)
        E.append(edges_of(t) + off)
        off += len(v)
    pos = np.concatenate(P) + noise * rng.uniform(-1, 1, (off, 3))
    return pos, np.arange(off, dtype=np.int32), np.concatenate(E), np.concatenate(T)


def brute_candidates(pos, verts, edges, tris, inflate, disp=None):
    """test_contact.cpp:362-389: every overlapping pair, brute force."""
    half = inflate / 2

    def box(nodes):
        pts = pos[nodes]
        if disp is not None:
            pts = np.concatenate([pts, pos[nodes] + disp[nodes]])
        return pts.min(0) - half, pts.max(0) + half

    def ov(a, b):
        return bool(np.all(a[0] <= b[1]) and np.all(b[0] <= a[1]))

    tb = [box(t) for t in tris]
    pt = [(vi, ti) for vi, v in enumerate(verts) for ti, t in enumerate(tris)
          if v not in t and ov(box([v]), tb[ti])]
    eb = [box(e) for e in edges]
    ee = [(i, j) for i in range(len(edges)) for j in range(i + 1, len(edges))
          if not set(edges[i]) & set(edges[j]) and ov(eb[i], eb[j])]
    return np.array(pt, np.int32).reshape(-1, 2), np.array(ee, np.int32).reshape(-1, 2)


def build_hinges(tris):
    """scene/mesh.hpp:98-121: interior edges shared by two triangles ->
    (e0, e1, w0, w1), w0 the wing of the triangle running e0 -> e1."""
    half, hinges = {}, []
    for t in tris:
        for a in range(3):
            u, v, w = int(t[a]), int(t[(a + 1) % 3]), int(t[(a + 2) % 3])
            key = (min(u, v), max(u, v))
            if key not in half:
                half[key] = (w, 0 if u == key[0] else 1)
            else:
                w0, d = half[key]
                hinges.append([key[0], key[1], w0, w] if d == 0 else [key[0], key[1], w, w0])
    return np.array(hinges, np.int32).reshape(-1, 4)


def cloth_patch(n=20, seed=1, offset=0):
    """A shell mesh (make_grid n x n) with its rest data from the oracle
    (membrane_rest / hinge_rest) and a deformed state; node ids shifted by
    `offset` (its position in the scene's slots)."""
    rng = np.random.default_rng(seed)
    verts, tris = make_grid(n, n, 1.0, 1.0)
    verts[:, 2] = 0.02 * np.sin(3 * verts[:, 0]) * np.cos(2 * verts[:, 1])
    hinges = build_hinges(tris)
    tri_rest = np.array([O.membrane_rest(verts[t].reshape(-1)) for t in tris])
    hinge_rest = np.array([O.hinge_rest(verts[h].reshape(-1)) for h in hinges])
    x = verts * np.array([1.05, 0.98, 1.0]) + rng.normal(0, 0.01, verts.shape)
    mass = rng.uniform(1e-4, 2e-4, len(verts))
    return {"verts": verts, "x": x, "mass": mass, "tris": tris + offset, "hinges": hinges + offset,
            "tri_rest": tri_rest, "hinge_rest": hinge_rest, "material": [1e-3, 5e4, 5e6, 0.3, 1e-3]}
