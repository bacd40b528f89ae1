make -j16 > gpurun_out/make.log 2>&1 || { tail -30 gpurun_out/make.log; exit 1; }
timeout 600 python bench.py --config C4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/b4.log 2>&1 || { tail gpurun_out/b4.log; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:lu_select --csv --log-file gpurun_out/c4_lu_launches.csv python bench.py --config C4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu4.log 2>&1; echo ncu rc=$?
