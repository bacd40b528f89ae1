# ncu --set full of the C5 Cholesky-QR Gram (gram_dmma_kernel<4, true>, 1e7×32)
make -j16 > gpurun_out/make.log 2>&1 || { tail -30 gpurun_out/make.log; exit 1; }
timeout 600 python bench.py --config C5 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/b5.log 2>&1 || { tail -3 gpurun_out/b5.log; exit 1; }
mkdir -p gpurun_out/prof
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gram_dmma -c 1 -o gpurun_out/prof/r01d_c5_gram python bench.py --config C5 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/prof/ncu_gram.log 2>&1; echo "ncu rc=$?"
