make -j16 > gpurun_out/make.log 2>&1 || { tail -30 gpurun_out/make.log; exit 1; }
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "int8emu" > gpurun_out/gpu_tests_emu.log 2>&1; echo "emu tests rc=$?"; tail -15 gpurun_out/gpu_tests_emu.log
if [ -n "$VARIANTS" ]; then bash tools/gpu/variants.sh > gpurun_out/variants.log 2>&1 || { tail gpurun_out/variants.log; exit 1; }; fi
echo "== default"; timeout 300 python tools/gpu/emu_micro.py > gpurun_out/emu_micro.log 2>&1; tail -8 gpurun_out/emu_micro.log
for spec in $VARIANTS; do v=${spec%%:*}; echo "== $v"; RPCA_LIB_PATH=/tmp/rpca_var/$v/librpca.so timeout 300 python tools/gpu/emu_micro.py > gpurun_out/emu_micro_$v.log 2>&1; grep -E "ax_f64_emu|int8emu " gpurun_out/emu_micro_$v.log; done
