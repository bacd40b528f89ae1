set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
make -j16 > gpurun_out/make.log 2>&1 || exit 1
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"
tail -30 gpurun_out/gpu_tests.log
for c in C2 C4 C3 C5 C1; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench_$c.log 2>&1; echo "$c rc=$?"; tail -2 gpurun_out/bench_$c.log; done
