# Aᵀ·Y A-slot count (2 slots + 3 accumulators vs 3-4 slots + 2 accumulators)
make -j16 > gpurun_out/make.log 2>&1 || { tail -30 gpurun_out/make.log; exit 1; }
VARIANTS="s3:-DATY_SLOTS=3 s4:-DATY_SLOTS=4" bash tools/gpu/variants.sh > gpurun_out/var.log 2>&1 || { tail gpurun_out/var.log; exit 1; }
for v in base s3 s4 base s3 s4; do
  if [ $v = base ]; then unset RPCA_LIB_PATH; else export RPCA_LIB_PATH=/tmp/rpca_var/$v/librpca.so; fi
  timeout 600 python bench.py --config C4 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/b_$v.log 2>&1
  tail -1 gpurun_out/b_$v.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); k=d['kernels']; print('$v', round(d['ms_per_step'],2), 'aty', round(k['aty_f32_tc']['ms_per_step']/5,3), 'reduce', round(k.get('aty_reduce',{}).get('ms_per_step',0),3))" 2>&1 | tail -1
done
