"""Profiling aid: assemble_filtered (filter_pinned + sort + reduce) on the cfg5
stream resident in HBM, CUDA-event timed. Usage: python tools/assembly_time.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import scenegen as S  # noqa: E402
from paper_2411_06224_b200.context import Context  # noqa: E402

sc = S.cfg5_batch_scene(5)
ctx = Context(0)
k = torch.from_numpy(sc.keys.view(np.int64)).cuda()
v = torch.from_numpy(sc.vals).cuda()
p = torch.from_numpy(sc.pinned).cuda()
for _ in range(3):
    ctx.assemble_filtered(k, v, sc.n_blocks, p)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    ctx.assemble_filtered(k, v, sc.n_blocks, p)
e1.record()
torch.cuda.synchronize()
print(f"assemble_filtered cfg5 ({len(sc.keys)} triplets): {e0.elapsed_time(e1) / 10:.3f} ms")
