"""Profiling aid: the element producer (fem_emit) on the cfg5 mesh at rest and
under random vertex perturbations (the PSD projection's Jacobi path), and the
contact pass on the geometric hybrid scene. Usage: python tools/producer_deformed.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import scenegen as S  # noqa: E402
from paper_2411_06224_b200.context import Context  # noqa: E402

sc = S.cfg5_batch_scene(5)
inv9, vol = S.tet_rest_data(sc.verts, sc.tets)
n, nt = len(sc.mass), len(sc.tets)
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
mesh = {"mass": t(sc.mass), "tets": t(sc.tets), "rest_inv9": t(inv9), "rest_volume": t(vol), "tet_begin": [0, nt],
        "mu": [sc.mu], "lam": [sc.lam]}
ctx = Context(0)
xt = t(S.inertial_target(sc))
keys = torch.empty(n + 10 * nt, dtype=torch.int64, device="cuda")
vals = torch.empty((n + 10 * nt, 9), dtype=torch.float64, device="cuda")
g = torch.empty(3 * n, dtype=torch.float64, device="cuda")
h = float(np.abs(sc.verts[1] - sc.verts[0]).max())
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for amp in (0.0, 0.01, 0.1, 0.3):
    x = t((sc.verts + np.random.default_rng(1).uniform(-amp * h, amp * h, sc.verts.shape)).reshape(-1))
    ctx.fem_emit(mesh, x, xt, 1e-4, keys, vals, g)
    torch.cuda.synchronize()
    ev0.record()
    for _ in range(5):
        ctx.fem_emit(mesh, x, xt, 1e-4, keys, vals, g)
    ev1.record()
    torch.cuda.synchronize()
    print(f"fem_emit perturbation {amp} h: {ev0.elapsed_time(ev1) / 5:.2f} ms", flush=True)
