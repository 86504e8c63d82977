"""Profiling aid: the cfg5 assembly (filter_pinned + sort + reduce) from a
device-resident stream, timed with CUDA events; run under ncu for the kernel
breakdown. Usage: python tools/asm_profile.py [reps]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import scenegen as scenes  # noqa: E402
from paper_2411_06224_b200.context import Context  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
sc = scenes.CONFIGS[os.environ.get("CFG", "cfg5_stiff_box")]()
ctx = Context(0)
dk = torch.from_numpy(sc.keys.view(np.int64)).cuda()
dv = torch.from_numpy(sc.vals).cuda()
dp = torch.from_numpy(sc.pinned).cuda()
torch.cuda.synchronize()
ts = []
for i in range(reps):
    ctx.assemble_filtered(dk, dv, sc.n_blocks, dp)
    ts.append(ctx.timings()["assemble_ms"])
print("assemble_ms", ["%.3f" % t for t in ts], "U", ctx.matrix_info())
