make -j16 > gpurun_out/make.log 2>&1 || { tail -30 gpurun_out/make.log; exit 1; }
VARIANTS="s2:-DATY_SLOTS=2 s3:-DATY_SLOTS=3 s4:-DATY_SLOTS=4" bash tools/gpu/variants.sh > gpurun_out/variants.log 2>&1 || { tail gpurun_out/variants.log; exit 1; }
for v in s2 s3 s4; do
  RPCA_LIB_PATH=/tmp/rpca_var/$v/librpca.so timeout 900 python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_C4_$v.log 2>&1; echo "$v rc=$?"; tail -1 gpurun_out/bench_C4_$v.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('ms', round(d['ms_per_step'],3), {k:round(v['ms_per_step'],3) for k,v in list(d['kernels'].items())[:3]})"
done
