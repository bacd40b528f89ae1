# full GPU tests, launch lists of every config, all bench lines (session refresh)
set -u
make -j16 > gpurun_out/make.log 2>&1 || { tail -30 gpurun_out/make.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "all tests rc=$?"; tail -1 gpurun_out/gpu_tests.log
mkdir -p gpurun_out/prof
for c in C1 C2 C3 C4 C5; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/${c}_launches.csv python bench.py --config $c --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/prof/ncu_${c}_list.log 2>&1; echo "$c list rc=$?"
done
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo "default rc=$?"; tail -1 gpurun_out/bench_default.log
for c in C1 C3 C4 C5; do
  timeout 900 python bench.py --config $c > gpurun_out/bench_full_$c.log 2>&1; echo "$c rc=$?"; tail -1 gpurun_out/bench_full_$c.log | cut -c1-200
done
