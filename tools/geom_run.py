"""Run only the geometric hybrid Newton-iteration leg of bench.py (GPU),
optionally the CPU leg too: python tools/geom_run.py [--cpu] [--steps K]."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--warmup", type=int, default=2)
ap.add_argument("--cpu", action="store_true")
a = ap.parse_args()
out = {"gpu": bench.geom_gpu(a, 0)}
print(json.dumps(out), flush=True)
if a.cpu:
    out["cpu"] = bench.geom_cpu()
    print(json.dumps(out["cpu"]), flush=True)
