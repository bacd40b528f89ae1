# GPU tests + quick benches (no CPU baseline / e2e) for the configs given as args
make -j16 > gpurun_out/make.log 2>&1 || { tail -30 gpurun_out/make.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"
tail -15 gpurun_out/gpu_tests.log
for c in "$@"; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1; echo "$c rc=$?"; tail -1 gpurun_out/bench_$c.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['config']['workload'][:3], 'ms', round(d['ms_per_step'],3), 'frac', d['roofline']['frac'], {k:round(v['ms_per_step'],3) for k,v in d['kernels'].items()})"; done
