make -j16 > gpurun_out/make.log 2>&1 || { tail -30 gpurun_out/make.log; exit 1; }
mkdir -p gpurun_out/prof
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"aty_f32_tc" -c 1 -o gpurun_out/prof/c4_aty_ts python bench.py --config C4 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_c4aty.log 2>&1; echo "ncu rc=$?"
