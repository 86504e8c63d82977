"""Profiling aid: cold MAS builds (hierarchy from the pattern every time) of
one scene with the host-side phase split (ADIPC_DEBUG_HIER=1 prints it to
stderr). Usage: ADIPC_DEBUG_HIER=1 python tools/hier_profile.py [config]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_06224_b200 import _lib  # noqa: E402
from paper_2411_06224_b200 import api as P  # noqa: E402
from paper_2411_06224_b200.context import Context  # noqa: E402
import scenegen as scenes  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4_hybrid_1m"
sc = scenes.CONFIGS[name]()
ctx = Context(0)
ctx.set_option(_lib.OPT_CACHE_HIERARCHY, 0)
t0 = time.perf_counter()
l0 = P.partition_block_graph(sc.n_blocks, sc.rest_edges, 16)
print(f"level-0 partition (once per scene) {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)
ctx.set_level0_partition(l0.part_of, l0.n_parts, 16, 4)
if len(sc.node_keys):
    ctx.assemble_contact(sc.keys, sc.vals, sc.node_keys, sc.node_vals, sc.n_fem, sc.n_bodies, sc.abd_body, sc.jac36,
                         sc.n_blocks, sc.pinned)
else:
    ctx.assemble_filtered(sc.keys, sc.vals, sc.n_blocks, sc.pinned)
for i in range(3):
    ctx.build_preconditioner(_lib.PRECOND_MAS)
    t = ctx.timings()
    print(f"build {i}: {t['build_ms']:.1f} ms (host {t['build_host_ms']:.1f})", flush=True)
print("levels", [(L["n_nodes"], L["n_parts"]) for L in ctx.precond_levels()])
