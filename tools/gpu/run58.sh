make -j16 > gpurun_out/make.log 2>&1 || { tail -30 gpurun_out/make.log; exit 1; }
VARIANTS="r2:-DLU_LEAF_R24=2,-DLU_LEAF_R32=2" bash tools/gpu/variants.sh > gpurun_out/var.log 2>&1 || { tail gpurun_out/var.log; exit 1; }
for v in base r2; do
  if [ $v = base ]; then unset RPCA_LIB_PATH; else export RPCA_LIB_PATH=/tmp/rpca_var/$v/librpca.so; fi
  for c in C2 C5; do
    timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_${c}_$v.log 2>&1
    tail -1 gpurun_out/bench_${c}_$v.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); k=d['kernels']; print('$v $c', round(d['ms_per_step'],3), 'leaf', round(k['lu_leaf']['ms_per_step'],3), 'tree', round(k['lu_tree']['ms_per_step'],3))"
  done
done
unset RPCA_LIB_PATH
