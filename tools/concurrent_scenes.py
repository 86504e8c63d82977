"""Experiment: K independent cfg5 scenes solved concurrently on one GPU (one
context and stream per scene, one host thread each; ctypes releases the GIL
during the C-ABI calls). Prints the aggregate PCG iterations/s vs K."""
import os
import sys
import threading
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_06224_b200 import _lib  # noqa: E402
import scenegen as scenes  # noqa: E402
from paper_2411_06224_b200 import api as P  # noqa: E402
from paper_2411_06224_b200.context import Context  # noqa: E402

sc = scenes.CONFIGS["cfg5_stiff_box"]()
l0 = P.partition_block_graph(sc.n_blocks, sc.rest_edges, 16)
b_host = torch.from_numpy(scenes.gravity_rhs(sc))
d_keys = torch.from_numpy(sc.keys.view("int64")).cuda()
d_vals = torch.from_numpy(sc.vals).cuda()
d_pin = torch.from_numpy(sc.pinned).cuda()
torch.cuda.synchronize()


def make():
    c = Context(0)
    c.set_option(_lib.OPT_CACHE_HIERARCHY, 1)
    c.set_level0_partition(l0.part_of, l0.n_parts, 16, 4)
    c.assemble_filtered(d_keys, d_vals, sc.n_blocks, d_pin)
    c.build_preconditioner(_lib.PRECOND_MAS)
    b = b_host.cuda()
    x = torch.empty_like(b)
    torch.cuda.synchronize()
    c.pcg(b, 1e-4, 250, 100000, x=x)  # warm (graphs, splits)
    return c, b, x


for K in [int(a) for a in (sys.argv[1:] or ["1", "2", "3", "4"])]:
    ctxs = [make() for _ in range(K)]
    iters = [0] * K
    reps = 4

    def run(i):
        c, b, x = ctxs[i]
        for _ in range(reps):
            _, r = c.pcg(b, 1e-4, 250, 100000, x=x)
            iters[i] += r.iters

    ths = [threading.Thread(target=run, args=(i,)) for i in range(K)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"K={K}: {sum(iters)} iterations in {dt * 1e3:.1f} ms -> {sum(iters) / dt:.0f} it/s aggregate", flush=True)
    for c, _, _ in ctxs:
        c.close()
