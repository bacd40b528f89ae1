make -j16 > gpurun_out/make.log 2>&1 || { tail -30 gpurun_out/make.log; exit 1; }
timeout 300 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "f32 or fp32 or centered" > gpurun_out/gpu_tests_f32.log 2>&1; echo "f32 tests rc=$?"; tail -15 gpurun_out/gpu_tests_f32.log
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "all tests rc=$?"; tail -3 gpurun_out/gpu_tests.log
timeout 600 python bench.py --config C4 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_C4.log 2>&1; echo "C4 rc=$?"; tail -1 gpurun_out/bench_C4.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['config']['workload'][:3], 'ms', round(d['ms_per_step'],3), 'frac', d['roofline']['frac'], {k:round(v['ms_per_step'],3) for k,v in d['kernels'].items()})"
