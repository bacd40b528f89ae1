make -j16 > gpurun_out/make.log 2>&1 || { tail -30 gpurun_out/make.log; exit 1; }
python tools/gpu/prof_overhead.py C2
python tools/gpu/prof_overhead.py C1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c2_launches.csv python bench.py --config C2 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_c2.log 2>&1; echo ncu rc=$?
