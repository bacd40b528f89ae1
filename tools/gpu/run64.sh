make -j16 > gpurun_out/make.log 2>&1 || { tail -30 gpurun_out/make.log; exit 1; }
VARIANTS="st10:-DATY_MAX_STAGES=10 st6:-DATY_MAX_STAGES=6" bash tools/gpu/variants.sh > gpurun_out/var.log 2>&1 || { tail gpurun_out/var.log; exit 1; }
for v in base st10 st6 base st10; do
  if [ $v = base ]; then unset RPCA_LIB_PATH; else export RPCA_LIB_PATH=/tmp/rpca_var/$v/librpca.so; fi
  timeout 600 python bench.py --config C4 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/b_$v.log 2>&1
  tail -1 gpurun_out/b_$v.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); k=d['kernels']; print('$v', round(d['ms_per_step'],2), 'aty', round(k['aty_f32_tc']['ms_per_step']/5,3), 'ax', round(k['ax_f32_tc']['ms_per_step']/5,3))"
done
