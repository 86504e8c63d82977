"""Profiling aid: cfg5 PCG per-iteration kernel-class times under different
options (L2 evict-last fraction of A for the SpMV). Prints one JSON line per
setting."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_06224_b200 as P  # noqa: E402
from paper_2411_06224_b200 import _lib, scenes  # noqa: E402
from paper_2411_06224_b200.context import Context  # noqa: E402

sc = scenes.CONFIGS["cfg5_stiff_box"]()
ctx = Context(0)
ctx.set_option(_lib.OPT_PROFILE, 1)
fk, fv = ctx.filter_pinned(sc.keys, sc.vals, sc.pinned)
ctx.assemble(fk, fv, sc.n_blocks)
l0 = P.partition_block_graph(sc.n_blocks, sc.rest_edges, 16)
ctx.set_level0_partition(l0.part_of, l0.n_parts, 16, 4)
ctx.build_preconditioner(_lib.PRECOND_MAS)
b = torch.from_numpy(scenes.gravity_rhs(sc)).cuda()
x = torch.empty_like(b)
fracs = [int(v) for v in sys.argv[1:]] or [0, 256, 384, 512, 640]
for frac in fracs:
    ctx.set_option(_lib.OPT_L2_PERSIST, frac)
    for rep in range(3):
        _, r = ctx.pcg(b, 1e-4, 250, 100000, x=x)
    t = ctx.timings()
    p = ctx.pcg_profile()
    it = max(p["iters"], 1)
    print(json.dumps({"persist_1024": frac, "iters": r.iters, "pcg_ms": round(t["pcg_ms"], 3),
                      "us_per_iter": round(1000 * t["pcg_ms"] / r.iters, 2),
                      **{k: round(1000 * v / it, 2) for k, v in p.items() if k.endswith("_ms")}}), flush=True)
