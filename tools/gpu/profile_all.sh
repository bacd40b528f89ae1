# ncu evidence for profiles/: launch lists of one bench step per config and
# --set full captures of the pass kernels of C2, C3, C4, C5 and of the C4 LU
# leaf (each after the same bench command exited 0 without ncu).
set -u
make -j16 > gpurun_out/make.log 2>&1 || exit 1
mkdir -p gpurun_out/prof
for c in C1 C2 C3 C4 C5; do
  timeout 600 python bench.py --config $c --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/prof/plain_$c.log 2>&1 || { echo "plain $c failed"; continue; }
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/${c}_launches.csv python bench.py --config $c --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/prof/ncu_${c}_list.log 2>&1; echo "$c list rc=$?"
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"_f64_tma" -c 2 -o gpurun_out/prof/C2_passes python bench.py --config C2 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/prof/ncu_C2.log 2>&1; echo "C2 full rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"ax_f64_tma" -c 1 -o gpurun_out/prof/C3_pass python bench.py --config C3 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/prof/ncu_C3.log 2>&1; echo "C3 full rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"f32_tc_kernel|lu_select" -c 3 -o gpurun_out/prof/C4_passes python bench.py --config C4 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/prof/ncu_C4.log 2>&1; echo "C4 full rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"csr_spmm_kernel" -c 2 -o gpurun_out/prof/C5_passes python bench.py --config C5 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/prof/ncu_C5.log 2>&1; echo "C5 full rc=$?"
ls -la gpurun_out/prof
