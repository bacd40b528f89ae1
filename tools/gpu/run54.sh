make -j16 > gpurun_out/make.log 2>&1 || { tail -30 gpurun_out/make.log; exit 1; }
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "small_svd or pca" > gpurun_out/svd_tests.log 2>&1; echo "svd tests rc=$?"; tail -3 gpurun_out/svd_tests.log
python tools/gpu/svd_micro.py
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "all tests rc=$?"; tail -1 gpurun_out/gpu_tests.log
