make -j16 > gpurun_out/make.log 2>&1 || { tail -30 gpurun_out/make.log; exit 1; }
VARIANTS="sb4:-DEMU_SB=4 sb6:-DEMU_SB=6 sb10:-DEMU_SB=10" bash tools/gpu/variants.sh > gpurun_out/variants.log 2>&1 || { tail gpurun_out/variants.log; exit 1; }
for v in default sb4 sb6 sb10; do
  if [ $v = default ]; then L=""; else L=/tmp/rpca_var/$v/librpca.so; fi
  RPCA_LIB_PATH=$L timeout 300 python bench.py --config C3 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/bench_C3_$v.log 2>&1; echo "$v rc=$?"
  tail -1 gpurun_out/bench_C3_$v.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); k=d['kernels']['ax_f64_emu']; print('step', round(d['ms_per_step'],3), 'emu ms/launch', round(k['ms_per_step']/k['launches_per_step'],3))" 2>&1 | tail -1
done
