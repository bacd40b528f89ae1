make -j16 > gpurun_out/make.log 2>&1 || { tail -30 gpurun_out/make.log; exit 1; }
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "f32 or c4 or C4 or fp32 or float" > gpurun_out/gpu_tests_f32.log 2>&1; echo "f32 tests rc=$?"; tail -3 gpurun_out/gpu_tests_f32.log
timeout 600 python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q -p no:cacheprovider -k "c4" > gpurun_out/gpu_tests_c4full.log 2>&1; echo "c4 full rc=$?"; tail -3 gpurun_out/gpu_tests_c4full.log
timeout 900 python bench.py --config C4 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_C4.log 2>&1; echo "C4 rc=$?"; tail -1 gpurun_out/bench_C4.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('ms', round(d['ms_per_step'],3), 'roof', d['roofline']['kernel'], d['roofline']['achieved'], d['roofline']['frac'], {k:round(v['ms_per_step'],3) for k,v in list(d['kernels'].items())[:8]})"
