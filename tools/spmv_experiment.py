"""Profiling aid: time SpMV kernels on the cfg5 matrix (the LDG-streamed and
the TMA-staged variants; normal, without atomics, warm or cold L2) to attribute
the SpMV time. Modes without atomics compute wrong results by construction."""
import ctypes as C
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_06224_b200 import _lib, scenes  # noqa: E402
from paper_2411_06224_b200.context import Context  # noqa: E402

sc = scenes.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg5_stiff_box"]()
ctx = Context(0)
fk, fv = ctx.filter_pinned(sc.keys, sc.vals, sc.pinned)
ctx.assemble(fk, fv, sc.n_blocks)
n, U = ctx.matrix_info()
x = torch.randn(3 * n, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
out = {"n": n, "U": U, "bytes": 80 * U + 48 * n}
L = _lib.gpu()
modes = [0, 2, 8, 10]
for v in (2, 3, 4):
    modes += [(v << 4), (v << 4) | 8, (v << 4) | 10]
for mode in modes:  # +8: L2 evicted before every launch (cold); >>4: variant
    ms = C.c_float()
    ctx._check(L.adipc_gpu_debug_spmv_time(ctx.h, x.data_ptr(), y.data_ptr(), mode, 30, C.byref(ms)))
    out[f"mode{mode}_us"] = round(ms.value * 1000, 2)
    out[f"mode{mode}_gbs"] = round(out["bytes"] / (ms.value / 1000) / 1e9, 1)
print(json.dumps(out))
