"""Regression aid: repeated cold MAS rebuilds (alternating sparsity patterns)
must not grow device memory use. Prints free device memory after each build
and the cold build times (ms)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_06224_b200 import _lib  # noqa: E402
import scenegen as scenes  # noqa: E402
from paper_2411_06224_b200 import api as P  # noqa: E402
from paper_2411_06224_b200.context import Context  # noqa: E402

sc = scenes.CONFIGS[os.environ.get("CFG", "cfg5_stiff_box")]()
ctx = Context(0)
ctx.set_option(_lib.OPT_CACHE_HIERARCHY, 1)
l0 = P.partition_block_graph(sc.n_blocks, sc.rest_edges, 16)
ctx.set_level0_partition(l0.part_of, l0.n_parts, 16, 4)
pins = [sc.pinned.copy(), sc.pinned.copy()]
pins[1][np.flatnonzero(pins[1])[:50]] = 0  # a second pattern
free = []
for i in range(8):
    fk, fv = ctx.filter_pinned(sc.keys, sc.vals, pins[i % 2])
    ctx.assemble(fk, fv, sc.n_blocks)
    ctx.build_preconditioner(_lib.PRECOND_MAS)
    torch.cuda.synchronize()
    free.append(torch.cuda.mem_get_info()[0] / 2**20)
    print(f"build {i}: {ctx.timings()['build_ms']:.1f} ms, free {free[-1]:.0f} MiB", flush=True)
print("growth after the first two builds: %.0f MiB" % (free[1] - free[-1]))
