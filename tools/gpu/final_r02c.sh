# round-2 close after the fp32 race fix and the rolled nomination: full GPU suite, smoke, bench lines, C4 capture of the fixed Aᵀ·Y
set -x
OUT=gpurun_out/fin2; mkdir -p $OUT
make -j16 > $OUT/make.log 2>&1 || exit 1
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $OUT/smoke.log 2>&1; echo smoke rc=$?
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo pytest rc=$?
timeout 600 python bench.py > $OUT/bench_C2.log 2>&1; echo bench C2 rc=$?
timeout 600 python bench.py --config C3 --no-cpu-baseline > $OUT/bench_C3.log 2>&1; echo bench C3 rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/C2_launches.csv python bench.py --config C2 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/ncu_C2_list.log 2>&1; echo C2 list rc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"aty_f32_tc_kernel|lu_nominate" -c 3 -o $OUT/C4_aty python bench.py --config C4 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > $OUT/ncu_C4_full.log 2>&1; echo C4 full rc=$?
