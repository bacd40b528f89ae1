make -j16 > gpurun_out/make.log 2>&1 || { tail -30 gpurun_out/make.log; exit 1; }
mkdir -p gpurun_out/prof
for spec in C2:aty_f64_tma_kernel C2:ax_f64_tma_kernel C4:aty_f32_tc_kernel C4:ax_f32_tc_kernel C4:lu_select_kernel C2:lu_select_kernel; do
  c=${spec%%:*}; k=${spec#*:}
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$k" -c 1 -o gpurun_out/prof/${c}_$k python bench.py --config $c --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/prof/ncu_${c}_$k.log 2>&1; echo "$c $k rc=$?"
done
