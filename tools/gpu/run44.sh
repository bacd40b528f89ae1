make -j16 > gpurun_out/make.log 2>&1 || { tail -30 gpurun_out/make.log; exit 1; }
mkdir -p gpurun_out/prof
timeout 600 python bench.py --config C3 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/prof/plain_C3.log 2>&1; echo "plain rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"ax_f64_emu_kernel" -c 1 -o gpurun_out/prof/C3_emu python bench.py --config C3 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/prof/ncu_C3emu.log 2>&1; echo "ncu rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/C3_launches.csv python bench.py --config C3 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/prof/ncu_C3_list.log 2>&1; echo "list rc=$?"
