make -j16 > gpurun_out/make.log 2>&1 || { tail -30 gpurun_out/make.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "all tests rc=$?"; tail -1 gpurun_out/gpu_tests.log
mkdir -p gpurun_out/prof
timeout 600 python bench.py --config C5 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/prof/plain_C5.log 2>&1; echo "plain C5 rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"csr_spmm_pair" -c 2 -o gpurun_out/prof/C5_csr2 python bench.py --config C5 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/prof/ncu_C5b.log 2>&1; echo "ncu C5 rc=$?"
timeout 600 python bench.py --config C4 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/prof/plain_C4.log 2>&1; echo "plain C4 rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"ax_f32_tc_kernel" -c 1 -o gpurun_out/prof/C4_ax2 python bench.py --config C4 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/prof/ncu_C4b.log 2>&1; echo "ncu C4 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/C5_launches.csv python bench.py --config C5 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/prof/ncu_C5_list.log 2>&1; echo "C5 list rc=$?"
