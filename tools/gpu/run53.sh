make -j16 > gpurun_out/make.log 2>&1 || { tail -30 gpurun_out/make.log; exit 1; }
VARIANTS="smem:-DJACOBI_NO_WARP" bash tools/gpu/variants.sh > gpurun_out/var.log 2>&1 || { tail gpurun_out/var.log; exit 1; }
echo "== warp"; python tools/gpu/svd_micro.py
echo "== smem"; RPCA_LIB_PATH=/tmp/rpca_var/smem/librpca.so python tools/gpu/svd_micro.py
