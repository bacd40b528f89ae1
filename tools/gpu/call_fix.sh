# the fp32 Aᵀ·Y stage-release fix: corruption stress, determinism, full GPU suite, C4/C2 bench
timeout 300 python tools/gpu/aty_f32_diag.py - 40 > gpurun_out/fix_diag.log 2>&1; echo diag rc=$?
timeout 600 python tools/gpu/determinism.py 10 > gpurun_out/fix_det.log 2>&1; echo det rc=$?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/fix_pytest.log 2>&1; echo pytest rc=$?
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/fix_smoke.log 2>&1; echo smoke rc=$?
timeout 600 python bench.py --config C4 --no-cpu-baseline > gpurun_out/fix_bench_c4.log 2>&1; echo c4 rc=$?
timeout 600 python bench.py > gpurun_out/fix_bench_c2.log 2>&1; echo c2 rc=$?
