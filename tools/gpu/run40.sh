make -j16 > gpurun_out/make.log 2>&1 || { tail -30 gpurun_out/make.log; exit 1; }
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "emu or eigens" > gpurun_out/gpu_tests_emu.log 2>&1; echo "emu tests rc=$?"; tail -1 gpurun_out/gpu_tests_emu.log
VARIANTS="w8:-DEMU_SPLIT_WARPS=8 w32:-DEMU_SPLIT_WARPS=32" C=C3 NK=2 bash tools/gpu/run30.sh 2>&1 | grep -v "^$"
