make -j16 > gpurun_out/make.log 2>&1 || { tail -30 gpurun_out/make.log; exit 1; }
mkdir -p gpurun_out/prof
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"ax_f64_emu" -c 1 -o gpurun_out/prof/c3_emu python bench.py --config C3 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_c3emu.log 2>&1; echo "ncu rc=$?"
