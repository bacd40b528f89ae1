make -j16 > gpurun_out/make.log 2>&1 || { tail -30 gpurun_out/make.log; exit 1; }
bash tools/gpu/variants.sh > gpurun_out/variants.log 2>&1 || { tail gpurun_out/variants.log; exit 1; }
RPCA_LIB_PATH=/tmp/rpca_var/r2/librpca.so timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "lu" 2>&1 | tail -1
for c in C5 C2; do VARIANTS="r2:-DLU_LEAF_R_MID=2" C=$c NK=4 bash tools/gpu/run30.sh 2>&1 | grep -E "ms|rc=" | head -4; done
