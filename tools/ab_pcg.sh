# A/B of the PCG iteration on one box: ADIPC_GPU_LIB=tools/bin/libadipc_gpu_old.so (a build of another commit) vs the in-tree build
for r in 1 2; do
  ADIPC_GPU_LIB=$PWD/tools/bin/libadipc_gpu_old.so python tools/pcg_profile.py so=1 2>&1 | tail -n 1 | sed 's/^/old /'
  python tools/pcg_profile.py so=1 2>&1 | tail -n 1 | sed 's/^/new /'
done
