# Round-end validation on one B200 (from the repo root): GPU tests, smoke,
# both bench arms (reference first, as the driver runs them), launch list.
set -u
OUT=gpurun_out; TAG=${1:-r02j}
python -m pytest tests -m gpu -x -q > $OUT/gputest_$TAG.txt 2>&1; echo "gpu tests rc=$?"; tail -n 2 $OUT/gputest_$TAG.txt
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.txt 2>&1; echo "smoke rc=$?"; tail -n 2 $OUT/smoke_$TAG.txt
python bench.py --impl reference > $OUT/bench_${TAG}_ref.json 2> $OUT/bench_${TAG}_ref.err; echo "ref rc=$?"
python bench.py > $OUT/bench_${TAG}.json 2> $OUT/bench_${TAG}.err; echo "bench rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-geom > $OUT/ncu_launch_$TAG.log 2>&1; echo "launch list rc=$?"
