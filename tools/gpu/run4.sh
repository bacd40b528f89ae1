make -j16 > gpurun_out/make.log 2>&1 || { tail -30 gpurun_out/make.log; exit 1; }
timeout 900 ncu --set full --import-source on --clock-control none -k regex:lu_select -s 30 -c 3 -o gpurun_out/lu_c2 python bench.py --config C2 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_lu.log 2>&1; echo ncu rc=$?
tail -3 gpurun_out/ncu_lu.log
