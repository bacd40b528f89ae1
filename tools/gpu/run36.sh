make -j16 > gpurun_out/make.log 2>&1 || { tail -30 gpurun_out/make.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py -m gpu -x -q -p no:cacheprovider -k "eigens or nystrom or Nystrom or c3 or C3" > gpurun_out/gpu_tests_emu.log 2>&1; echo "eigens tests rc=$?"; tail -15 gpurun_out/gpu_tests_emu.log
timeout 600 python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q -p no:cacheprovider -k "c3" > gpurun_out/gpu_tests_c3.log 2>&1; echo "c3 full rc=$?"; tail -15 gpurun_out/gpu_tests_c3.log
timeout 900 python bench.py --config C3 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_C3.log 2>&1; echo "C3 rc=$?"; tail -1 gpurun_out/bench_C3.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('ms', round(d['ms_per_step'],3), 'roof', d['roofline']['kernel'], d['roofline']['achieved'], d['roofline']['frac'], {k:round(v['ms_per_step'],3) for k,v in list(d['kernels'].items())[:8]})"
RPCA_NO_EMU=1 timeout 900 python bench.py --config C3 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_C3_noemu.log 2>&1; echo "C3 noemu rc=$?"; tail -1 gpurun_out/bench_C3_noemu.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('ms', round(d['ms_per_step'],3), 'roof', d['roofline']['kernel'], d['roofline']['achieved'], d['roofline']['frac'])"
