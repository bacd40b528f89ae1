make -j16 > gpurun_out/make.log 2>&1 || { tail -30 gpurun_out/make.log; exit 1; }
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "emu or eigens" > gpurun_out/gpu_tests_emu.log 2>&1; echo "emu tests rc=$?"; tail -3 gpurun_out/gpu_tests_emu.log
timeout 900 python bench.py --config C3 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_C3.log 2>&1; echo "C3 rc=$?"; tail -1 gpurun_out/bench_C3.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('ms', round(d['ms_per_step'],3), 'roof', d['roofline']['kernel'], d['roofline']['achieved'], d['roofline']['frac'], {k:round(v['ms_per_step'],3) for k,v in list(d['kernels'].items())[:6]})"
