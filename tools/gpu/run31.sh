make -j16 > gpurun_out/make.log 2>&1 || { tail -30 gpurun_out/make.log; exit 1; }
mkdir -p gpurun_out/prof
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"jacobi|chol_warp" -c 2 -o gpurun_out/prof/small_c2b python bench.py --config C2 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_small.log 2>&1; echo "ncu rc=$?"
