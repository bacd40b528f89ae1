make -j16 > gpurun_out/make.log 2>&1 || { tail -30 gpurun_out/make.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "all tests rc=$?"; tail -1 gpurun_out/gpu_tests.log
for c in C4; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$c.log 2>&1
  tail -1 gpurun_out/bench_$c.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); k=d['kernels']; print('$c', round(d['ms_per_step'],3)); [print('   %-22s %5.1f %8.3f' % (n, v['launches_per_step'], v['ms_per_step'])) for n,v in sorted(k.items(), key=lambda x:-x[1]['ms_per_step'])[:10]]"
done
