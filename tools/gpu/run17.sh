# full default bench line (C2 with e2e + CPU baseline) and the other configs
make -j16 > gpurun_out/make.log 2>&1 || { tail -30 gpurun_out/make.log; exit 1; }
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo "default rc=$?"; tail -1 gpurun_out/bench_default.log
for c in C1 C3 C4 C5; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-e2e > gpurun_out/bench_full_$c.log 2>&1; echo "$c rc=$?"; tail -1 gpurun_out/bench_full_$c.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['config']['workload'][:3], 'ms', round(d['ms_per_step'],3), 'roof', d['roofline']['kernel'], d['roofline']['achieved'], d['roofline']['frac'], 'cpu', d.get('cpu_baseline'))"
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/bench_ref.log
