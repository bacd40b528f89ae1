make -j16 > gpurun_out/make.log 2>&1 || { tail -30 gpurun_out/make.log; exit 1; }
timeout 400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "all tests rc=$?"; tail -2 gpurun_out/gpu_tests.log
for c in C2 C1 C3 C4 C5; do
  extra="--no-cpu-baseline --no-e2e"; [ $c = C2 ] && extra=""
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 $extra > gpurun_out/bench_$c.log 2>&1; echo "$c rc=$?"; tail -1 gpurun_out/bench_$c.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['config']['workload'][:3], 'ms', round(d['ms_per_step'],3), 'roof', d['roofline']['kernel'], d['roofline']['achieved'], d['roofline']['frac'], 'e2e', (d.get('e2e') or {}).get('value'), 'cpu', (d.get('cpu_baseline') or {}).get('value'), {k:round(v['ms_per_step'],3) for k,v in list(d['kernels'].items())[:8]})"
done
