make -j16 > gpurun_out/make.log 2>&1 || { tail -30 gpurun_out/make.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "all tests rc=$?"; tail -1 gpurun_out/gpu_tests.log
timeout 600 python bench.py --config C4 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/b4.log 2>&1
tail -1 gpurun_out/b4.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); k=d['kernels']; print('C4', round(d['ms_per_step'],2), 'misc', k['misc'])"
