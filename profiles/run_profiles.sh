#!/bin/bash
# Profiling recipe (/opt/skills/guides/B200_PROFILING.md), on the GPU box from
# the repo root:   bash profiles/run_profiles.sh <tag>
# 1. launch list: every kernel of one warm bench step with its device time
#    (cold-cache, serialised: compare shares, not absolutes)
# 2. ncu --set full on the PCG-iteration kernels, the assembly kernels and
#    the MAS build kernels (one capture each; never multi-rank)
set -u
TAG=${1:-r01}
OUT=gpurun_out
mkdir -p $OUT
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv $CMD \
    > $OUT/ncu_launch_$TAG.log 2>&1
echo "launch list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:'k_spmv|k_update_so|k_precond_so|k_final_so' -s 300 -c 8 \
    -o $OUT/prof_pcg_$TAG -f $CMD > $OUT/ncu_pcg_$TAG.log 2>&1
echo "ncu pcg rc=$?"
ncu --set full --clock-control none --import-source on -k regex:'k_reduce_rows|k_row_scatter|k_sort_rows|k_pin_' \
    -c 8 -o $OUT/prof_build_$TAG -f $CMD > $OUT/ncu_build_$TAG.log 2>&1
echo "ncu assembly rc=$?"
ncu --set full --clock-control none --import-source on -k regex:'k_restrict|k_invert|k_solve_gather|k_graph' \
    -c 6 -o $OUT/prof_mas_$TAG -f $CMD > $OUT/ncu_mas_$TAG.log 2>&1
echo "ncu mas build rc=$?"
