# LU profiling: per-kernel sweep + one full ncu capture of the C4-sized leaf
make -j16 > gpurun_out/make.log 2>&1 || { tail -30 gpurun_out/make.log; exit 1; }
timeout 300 python tools/gpu/lu_micro.py 22,42,52,64 > gpurun_out/lu_micro.log 2>&1; echo "micro rc=$?"; cat gpurun_out/lu_micro.log
mkdir -p gpurun_out/prof
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"lu_select" -c 1 -o gpurun_out/prof/lu_leaf56 python tools/gpu/lu_one.py 2000000 52 > gpurun_out/ncu_leaf56.log 2>&1; echo "ncu rc=$?"
