"""Profiling aid: one Newton linear solve of the hybrid 1M-DOF scene
(cfg4_hybrid_1m) through the device path — two-level contact assembly, cold
MAS build, PCG — for an ncu launch list. Usage: python tools/hybrid_profile.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_06224_b200 import _lib  # noqa: E402
from paper_2411_06224_b200 import api as P  # noqa: E402
from paper_2411_06224_b200.context import Context  # noqa: E402
import scenegen as scenes  # noqa: E402

sc = scenes.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg4_hybrid_1m"]()
ctx = Context(0)
ctx.set_option(_lib.OPT_CACHE_HIERARCHY, 0)
l0 = P.partition_block_graph(sc.n_blocks, sc.rest_edges, 16)
ctx.set_level0_partition(l0.part_of, l0.n_parts, 16, 4)
d = {k: torch.from_numpy(v).cuda() for k, v in dict(keys=sc.keys.view(np.int64), vals=sc.vals,
                                                    nk=sc.node_keys.view(np.int64), nv=sc.node_vals, body=sc.abd_body,
                                                    jac=sc.jac36, pin=sc.pinned).items()}
xs = torch.from_numpy(scenes.ballistic_direction(sc)).cuda()
b = torch.empty_like(xs)
for it in range(int(os.environ.get("REPS", "2"))):
    U, nt = ctx.assemble_contact(d["keys"], d["vals"], d["nk"], d["nv"], sc.n_fem, sc.n_bodies, d["body"], d["jac"],
                                 sc.n_blocks, d["pin"])
    t_asm = ctx.timings()["assemble_ms"]
    if it == 0:
        ctx.spmv(xs, b)
    ctx.build_preconditioner(_lib.PRECOND_MAS)
    t = ctx.timings()
    x, res = ctx.pcg(b, 1e-4, 250, 100000, x=torch.empty_like(b))
    print(f"rep {it}: assembly {t_asm:.2f} ms (U {U}, tiles {nt}), build {t['build_ms']:.2f} ms "
          f"(host {t['build_host_ms']:.2f}), pcg {ctx.timings()['pcg_ms']:.2f} ms, {res.iters} iterations", flush=True)
