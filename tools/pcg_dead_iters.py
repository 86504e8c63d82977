import os, sys, torch
sys.path.insert(0, '/root/repo')
from paper_2411_06224_b200 import _lib
import scenegen as scenes
from paper_2411_06224_b200 import api as P
from paper_2411_06224_b200.context import Context
sc = scenes.CONFIGS["cfg5_stiff_box"]()
ctx = Context(0)
l0 = P.partition_block_graph(sc.n_blocks, sc.rest_edges, 16)
ctx.set_level0_partition(l0.part_of, l0.n_parts, 16, 4)
fk, fv = ctx.filter_pinned(sc.keys, sc.vals, sc.pinned)
ctx.assemble(fk, fv, sc.n_blocks)
ctx.build_preconditioner(_lib.PRECOND_MAS)
b = torch.from_numpy(scenes.gravity_rhs(sc)).cuda(); x = torch.empty_like(b); torch.cuda.synchronize()
for mi in [int(a) for a in (sys.argv[1:] or ["100000", "340", "339", "100000", "340"])]:
    best = 1e9
    for _ in range(3):
        _, r = ctx.pcg(b, 1e-4, 250, mi, x=x)
        best = min(best, ctx.timings()["pcg_ms"])
    print(mi, r.iters, r.converged, "%.3f ms" % best, flush=True)
