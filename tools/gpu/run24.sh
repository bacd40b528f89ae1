make -j16 > gpurun_out/make.log 2>&1 || { tail -30 gpurun_out/make.log; exit 1; }
mkdir -p gpurun_out/prof
timeout 300 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "qr or svd or pca or orth or chol" > gpurun_out/gpu_tests_small.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gpu_tests_small.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"jacobi|chol_kernel" -c 5 -o gpurun_out/prof/small_c2 python bench.py --config C2 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_small.log 2>&1; echo "ncu rc=$?"
