#!/bin/bash
# Profiling recipe (B200_PROFILING.md), run on the GPU box from the repo root:
#   bash profiles/run_profiles.sh <tag>
# 1. launch list: every kernel of one warm bench step with its device time
# 2. ncu --set full on the hot kernels of the PCG iteration and the build
set -u
TAG=${1:-r01}
OUT=gpurun_out
mkdir -p $OUT
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv $CMD > $OUT/ncu_launch_$TAG.log 2>&1
echo "launch list rc=$?"
ncu --set full --clock-control none --import-source on \
    -k regex:'k_spmv|k_mas_level|k_mas_final|k_restrict|k_invert|k_reduce_rows' -s 40 -c 12 \
    -o $OUT/prof_$TAG -f $CMD > $OUT/ncu_full_$TAG.log 2>&1
echo "ncu full rc=$?"
