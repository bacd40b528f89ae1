make -j16 > gpurun_out/make.log 2>&1 || { tail -30 gpurun_out/make.log; exit 1; }
timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py -m gpu -x -q -p no:cacheprovider -k "lu or LU or shard" > gpurun_out/gpu_tests_lu.log 2>&1; echo "lu tests rc=$?"; tail -15 gpurun_out/gpu_tests_lu.log
timeout 300 python tools/gpu/lu_micro.py 22,42,52,64 > gpurun_out/lu_micro.log 2>&1; echo "micro rc=$?"; cat gpurun_out/lu_micro.log
