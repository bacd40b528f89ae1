# ncu evidence for profiles/: launch lists of one bench step per config and
# --set full captures of the pass kernels of C2, C3, C4, C5 and of the C4 LU
# nomination leaf (each after the same bench command exited 0 without ncu).
# usage: bash tools/gpu/profile_all.sh [outdir]
set -u
OUT=${1:-gpurun_out/prof}
make -j16 > $OUT.make.log 2>&1 || exit 1
mkdir -p $OUT
for c in C1 C2 C3 C4 C5; do
  timeout 600 python bench.py --config $c --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/plain_$c.log 2>&1 || { echo "plain $c failed"; continue; }
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/${c}_launches.csv python bench.py --config $c --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/ncu_${c}_list.log 2>&1; echo "$c list rc=$?"
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"_f64_tma" -c 2 -o $OUT/C2_passes python bench.py --config C2 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > $OUT/ncu_C2.log 2>&1; echo "C2 full rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"ax_f64_emu_kernel" -c 1 -o $OUT/C3_pass python bench.py --config C3 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > $OUT/ncu_C3.log 2>&1; echo "C3 full rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"f32_tc_kernel|lu_nominate" -c 3 -o $OUT/C4_passes python bench.py --config C4 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > $OUT/ncu_C4.log 2>&1; echo "C4 full rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"csr_spmm" -c 2 -o $OUT/C5_passes python bench.py --config C5 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > $OUT/ncu_C5.log 2>&1; echo "C5 full rc=$?"
ls -la $OUT
