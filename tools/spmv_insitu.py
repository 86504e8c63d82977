"""Profiling aid: the SpMV in situ vs in isolation. Runs one cfg5 Newton solve
(assembly, MAS build, PCG with per-kernel-class events), then times the SpMV
kernels alone on the solve-order matrix with the PCG's final p as input, and on
the reference-order matrix with a random x."""
import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_06224_b200 import _lib, scenes  # noqa: E402
from paper_2411_06224_b200 import api as P  # noqa: E402
from paper_2411_06224_b200.context import Context  # noqa: E402

sc = scenes.CONFIGS["cfg5_stiff_box"]()
ctx = Context(0)
l0 = P.partition_block_graph(sc.n_blocks, sc.rest_edges, 16)
ctx.set_level0_partition(l0.part_of, l0.n_parts, 16, 4)
fk, fv = ctx.filter_pinned(sc.keys, sc.vals, sc.pinned)
ctx.assemble(fk, fv, sc.n_blocks)
n, U = ctx.matrix_info()
b = torch.from_numpy(scenes.gravity_rhs(sc)).cuda()
x = torch.empty_like(b)
out = {"n": n, "U": U}
for variant in [int(a) for a in (sys.argv[1:] or ["0", "3"])]:
    if variant == 8:  # sliced-ELL copy built from the current matrix (ADIPC_SELL_REF: reference order)
        ctx.set_option(_lib.OPT_SPMV_VARIANT, 8)
    ctx.set_option(_lib.OPT_SPMV_VARIANT, variant)
    ctx.build_preconditioner(_lib.PRECOND_MAS)
    ctx.set_option(_lib.OPT_PROFILE, 1)
    _, res = ctx.pcg(b, 1e-4, 250, 100000, x=x)
    prof = ctx.pcg_profile()
    ctx.set_option(_lib.OPT_PROFILE, 0)
    it = max(prof["iters"], 1)
    out[f"v{variant}_pcg"] = {k: round(prof[k + "_ms"] / it * 1000, 1) for k in ("spmv", "update", "precond", "final")}
    L = _lib.gpu()
    if variant == 8:
        ctx._check(L.adipc_gpu_debug_build_sell(ctx.h))
    xr = torch.randn(3 * n, dtype=torch.float64, device="cuda")
    yr = torch.zeros_like(xr)
    for mode, name in ((256, "insitu_warm"), (256 | 8, "insitu_cold"), (256 | 512, "insitu_dot_warm"),
                       (256 | 512 | 8, "insitu_dot_cold"), (0, "ref_warm"), (8, "ref_cold")):
        ms = C.c_float()
        ctx._check(L.adipc_gpu_debug_spmv_time(ctx.h, xr.data_ptr(), yr.data_ptr(), mode | (variant << 4), 20, C.byref(ms)))
        out[f"v{variant}_{name}_us"] = round(ms.value * 1000, 1)
print(json.dumps(out))
