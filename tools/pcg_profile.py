"""Profiling aid: one cfg5 Newton solve per option set, with the per-kernel-class
CUDA-event breakdown of the PCG iteration (us per iteration) and the graph-mode
PCG time. Usage: python tools/pcg_profile.py 'so=1,l0=3,pairs=4' 'so=0' ..."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_06224_b200 import _lib  # noqa: E402
import scenegen as scenes  # noqa: E402
from paper_2411_06224_b200 import api as P  # noqa: E402
from paper_2411_06224_b200.context import Context  # noqa: E402

OPTS = {"so": _lib.OPT_SO_KERNELS, "l0": _lib.OPT_L0_STAGES, "order": _lib.OPT_SOLVE_ORDER, "pairs": _lib.OPT_PC_PAIRS}
sc = scenes.CONFIGS[os.environ.get("CFG", "cfg5_stiff_box")]()
ctx = Context(0)
l0 = P.partition_block_graph(sc.n_blocks, sc.rest_edges, 16)
ctx.set_level0_partition(l0.part_of, l0.n_parts, 16, 4)
fk, fv = ctx.filter_pinned(sc.keys, sc.vals, sc.pinned)
ctx.assemble(fk, fv, sc.n_blocks)
n, U = ctx.matrix_info()
b = torch.from_numpy(scenes.gravity_rhs(sc)).cuda()
x = torch.empty_like(b)
res_ref = None
for spec in sys.argv[1:] or ["so=1"]:
    for kv in spec.split(","):
        k, v = kv.split("=")
        ctx.set_option(OPTS[k], int(v))
    ctx.build_preconditioner(_lib.PRECOND_MAS)
    out = {"spec": spec}
    for prof in (0, 1):
        ctx.set_option(_lib.OPT_PROFILE, prof)
        best = None
        for _ in range(1 if prof else 3):  # graph mode: best of 3 solves
            _, res = ctx.pcg(b, 1e-4, 250, int(os.environ.get("MAXIT", "100000")), x=x)
            t = ctx.timings()
            if best is None or t["pcg_ms"] < best[1]["pcg_ms"]:
                best = (res, t)
        res, t = best
        if prof:
            pr = ctx.pcg_profile()
            it = max(pr["iters"], 1)
            out["class_us"] = {k: round(pr[k + "_ms"] / it * 1000, 1) for k in ("spmv", "update", "precond", "final")}
        else:
            out["iters"] = res.iters
            out["pcg_ms"] = round(t["pcg_ms"], 3)
            out["us_per_iter"] = round(t["pcg_ms"] / max(res.iters, 1) * 1000, 1)
            xs = x.cpu().numpy()
            if res_ref is None:
                res_ref = xs
            out["rel_vs_first"] = float(np.linalg.norm(xs - res_ref) / np.linalg.norm(res_ref))
    ctx.set_option(_lib.OPT_PROFILE, 0)
    print(json.dumps(out), flush=True)
