make -j16 > gpurun_out/make.log 2>&1 || { tail -30 gpurun_out/make.log; exit 1; }
if [ -n "$VARIANTS" ]; then bash tools/gpu/variants.sh > gpurun_out/variants.log 2>&1 || { tail gpurun_out/variants.log; exit 1; }; fi
C=${C:-C4}
run() {
  timeout 900 python bench.py --config $C --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_${C}_$1.log 2>&1; echo "$1 rc=$?"; tail -1 gpurun_out/bench_${C}_$1.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('ms', round(d['ms_per_step'],3), {k:round(v['ms_per_step'],3) for k,v in list(d['kernels'].items())[:${NK:-4}]})"
}
run default
for spec in $VARIANTS; do v=${spec%%:*}; RPCA_LIB_PATH=/tmp/rpca_var/$v/librpca.so run $v; done
run default2
