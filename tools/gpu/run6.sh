make -j16 > gpurun_out/make.log 2>&1 || { tail -30 gpurun_out/make.log; exit 1; }
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"f32_tc" -c 2 -o gpurun_out/c4_tc python bench.py --config C4 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_c4.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/ncu_c4.log
