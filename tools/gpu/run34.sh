make -j16 > gpurun_out/make.log 2>&1 || { tail -30 gpurun_out/make.log; exit 1; }
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "f32 or c4 or C4 or fp32 or float" > gpurun_out/gpu_tests_f32.log 2>&1; echo "f32 tests rc=$?"; tail -1 gpurun_out/gpu_tests_f32.log
C=C4 NK=3 bash tools/gpu/run30.sh 2>&1 | grep -v "^$"
timeout 900 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:"aty_f32_tc" -c 1 python bench.py --config C4 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline 2>&1 | grep -E "dram__bytes|gpu__time|hit_rate"
