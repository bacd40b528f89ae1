# round-2 closing check: full GPU suite, smoke, bench lines (C2 default, C5),
# the C5 launch list and one --set full capture of its SpMM kernels
set -x
OUT=gpurun_out/fin; mkdir -p $OUT
make -j16 > $OUT/make.log 2>&1 || exit 1
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $OUT/smoke.log 2>&1; echo smoke rc=$?
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo pytest rc=$?
timeout 600 python bench.py > $OUT/bench_C2.log 2>&1; echo bench C2 rc=$?
timeout 600 python bench.py --config C5 --no-cpu-baseline > $OUT/bench_C5.log 2>&1; echo bench C5 rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/C5_launches.csv python bench.py --config C5 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/ncu_C5_list.log 2>&1; echo C5 list rc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"csr_spmm_pair" -c 2 -o $OUT/C5_spmm python bench.py --config C5 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > $OUT/ncu_C5_full.log 2>&1; echo C5 full rc=$?
