# Aᵀ·Y (fp32, C4 shape) ablations: per-pass times from bench's kernel table
make -j16 > gpurun_out/make.log 2>&1 || { tail -30 gpurun_out/make.log; exit 1; }
VARIANTS="nomma:-DATY_NO_MMA nost:-DATY_NO_TMEM_ST both:-DATY_NO_MMA,-DATY_NO_TMEM_ST" bash tools/gpu/variants.sh > gpurun_out/var.log 2>&1 || { tail gpurun_out/var.log; exit 1; }
for v in base nomma nost both base; do
  if [ $v = base ]; then unset RPCA_LIB_PATH; else export RPCA_LIB_PATH=/tmp/rpca_var/$v/librpca.so; fi
  timeout 600 python bench.py --config C4 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/b_$v.log 2>&1
  tail -1 gpurun_out/b_$v.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); k=d['kernels']; print('$v aty', round(k['aty_f32_tc']['ms_per_step']/5,3), 'ax', round(k['ax_f32_tc']['ms_per_step']/5,3))" 2>&1 | tail -1
done
