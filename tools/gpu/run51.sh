make -j16 > gpurun_out/make.log 2>&1 || { tail -30 gpurun_out/make.log; exit 1; }
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "small_svd or pca" > gpurun_out/svd_tests.log 2>&1; echo "svd tests rc=$?"; tail -3 gpurun_out/svd_tests.log
for c in C1 C2 C5; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$c.log 2>&1
  tail -1 gpurun_out/bench_$c.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$c ms', round(d['ms_per_step'],3), 'jacobi', d['kernels'].get('jacobi'))"
done
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "all tests rc=$?"; tail -1 gpurun_out/gpu_tests.log
