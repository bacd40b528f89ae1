# A/B: AtY A_lo TMEM slots 2 vs 4 on C4 (plus the f32 GPU tests for each)
for ns in 2 4; do
  touch paper_1412_3510_b200/csrc/dense_f32_tc.cu
  make -j16 NVCC="nvcc -DATY_SLOTS=$ns" > gpurun_out/make.log 2>&1 || { tail -30 gpurun_out/make.log; exit 1; }
  timeout 120 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "f32 or fp32" 2>&1 | tail -1
  timeout 600 python bench.py --config C4 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_C4_ns$ns.log 2>&1; echo "C4 ns=$ns rc=$?"; tail -1 gpurun_out/bench_C4_ns$ns.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['config']['workload'][:3], 'ms', round(d['ms_per_step'],3), 'frac', d['roofline']['frac'], {k:round(v['ms_per_step'],3) for k,v in list(d['kernels'].items())[:6]})"
done
