make -j16 > gpurun_out/make.log 2>&1 || { tail -30 gpurun_out/make.log; exit 1; }
timeout 300 python tools/gpu/debug_aty.py 2>&1 | grep -v "^ \|z\["
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "all tests rc=$?"; tail -3 gpurun_out/gpu_tests.log
timeout 600 python bench.py --config C4 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_C4.log 2>&1; echo "C4 rc=$?"; tail -1 gpurun_out/bench_C4.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['config']['workload'][:3], 'ms', round(d['ms_per_step'],3), 'frac', d['roofline']['frac'], {k:round(v['ms_per_step'],3) for k,v in d['kernels'].items()})"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"f32_tc" -c 2 -o gpurun_out/c4_tc3 python bench.py --config C4 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_c4.log 2>&1; echo ncu rc=$?
