make -j16 > gpurun_out/make.log 2>&1 || { tail -30 gpurun_out/make.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "all tests rc=$?"; tail -1 gpurun_out/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo "default rc=$?"; tail -1 gpurun_out/bench_default.log | cut -c1-400
timeout 900 python bench.py --config C4 > gpurun_out/bench_full_C4.log 2>&1; echo "C4 rc=$?"; tail -1 gpurun_out/bench_full_C4.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('C4', d['ms_per_step'], d['roofline']['frac'], d['e2e'])"
