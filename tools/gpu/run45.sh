make -j16 > gpurun_out/make.log 2>&1 || { tail -30 gpurun_out/make.log; exit 1; }
timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py -m gpu -x -q -p no:cacheprovider -k "lu or LU or shard" > gpurun_out/gpu_tests_lu.log 2>&1; echo "lu tests rc=$?"; tail -1 gpurun_out/gpu_tests_lu.log
for c in C5 C2; do C=$c NK=4 bash tools/gpu/run30.sh 2>&1 | grep -E "ms|rc=" | head -2; done
