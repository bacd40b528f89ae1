make -j16 > gpurun_out/make.log 2>&1 || { tail -30 gpurun_out/make.log; exit 1; }
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "csr or CSR or sparse or c5" > gpurun_out/gpu_tests_csr.log 2>&1; echo "csr tests rc=$?"; tail -1 gpurun_out/gpu_tests_csr.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q -p no:cacheprovider -k "c5" > gpurun_out/gpu_tests_c5.log 2>&1; echo "c5 full rc=$?"; tail -1 gpurun_out/gpu_tests_c5.log
C=C5 NK=5 bash tools/gpu/run30.sh 2>&1 | grep -E "ms|rc=" | head -2
