make -j16 > gpurun_out/make.log 2>&1 || { tail -30 gpurun_out/make.log; exit 1; }
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "emu" > gpurun_out/gpu_tests_emu.log 2>&1; echo "emu tests rc=$?"; tail -15 gpurun_out/gpu_tests_emu.log
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "all tests rc=$?"; tail -2 gpurun_out/gpu_tests.log
