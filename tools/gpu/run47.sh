make -j16 > gpurun_out/make.log 2>&1 || { tail -30 gpurun_out/make.log; exit 1; }
if [ -n "$VARIANTS" ]; then bash tools/gpu/variants.sh > gpurun_out/variants.log 2>&1 || { tail gpurun_out/variants.log; exit 1; }; fi
echo "== default"; timeout 300 python tools/gpu/pass_micro.py > gpurun_out/pm_default.log 2>&1; tail -12 gpurun_out/pm_default.log
for spec in $VARIANTS; do v=${spec%%:*}; echo "== $v"; RPCA_LIB_PATH=/tmp/rpca_var/$v/librpca.so timeout 300 python tools/gpu/pass_micro.py > gpurun_out/pm_$v.log 2>&1; tail -8 gpurun_out/pm_$v.log; done
