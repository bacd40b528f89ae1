make -j16 > gpurun_out/make.log 2>&1 || { tail -30 gpurun_out/make.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "all tests rc=$?"; tail -1 gpurun_out/gpu_tests.log
for c in C3 C2; do
for v in cols rows; do
  if [ $v = cols ]; then export RPCA_JACOBI_COLS=1; else unset RPCA_JACOBI_COLS; fi
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_${c}_$v.log 2>&1
  tail -1 gpurun_out/bench_${c}_$v.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$c $v ms', round(d['ms_per_step'],3), 'jacobi', d['kernels']['jacobi'])"
done; done
