make -j16 > gpurun_out/make.log 2>&1 || { tail -30 gpurun_out/make.log; exit 1; }
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "all tests rc=$?"; tail -1 gpurun_out/gpu_tests.log
for c in ${CONFIGS:-C1 C2}; do
timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$c.log 2>&1; echo "$c rc=$?"; tail -1 gpurun_out/bench_$c.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('ms', round(d['ms_per_step'],3), 'roof', d['roofline']['kernel'], d['roofline']['achieved'], d['roofline']['frac'], {k:round(v['ms_per_step'],3) for k,v in list(d['kernels'].items())[:10]})"
done
