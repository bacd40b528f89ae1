make -j16 > gpurun_out/make.log 2>&1 || { tail -30 gpurun_out/make.log; exit 1; }
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "f32 or c4 or C4 or fp32 or float" > gpurun_out/gpu_tests_f32.log 2>&1; echo "f32 tests rc=$?"; tail -1 gpurun_out/gpu_tests_f32.log
C=C4 NK=3 bash tools/gpu/run30.sh 2>&1 | grep -v "^$"
VARIANTS="lu24:-DLU_TWO_BLOCK_MAX=24" C=C5 NK=4 bash tools/gpu/run30.sh 2>&1 | grep -v "^$"
