# rolled Cholesky-QR warp kernel vs the unrolled build: bitwise (all cases), whole-PCA A/B on C2/C5, C2 launch list
N=paper_1412_3510_b200/librpca.so; B=.scratch/var/base/librpca.so
timeout 900 python tools/gpu/bitwise_ab.py $N $B > gpurun_out/ch_bitwise.log 2>&1; echo bw rc=$?
for c in C2 C5; do timeout 900 python tools/gpu/ab_pass.py pca:$c 11 $N $B > gpurun_out/ch_ab_$c.log 2>&1; echo ab $c rc=$?; done
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ch_C2_launches.csv python bench.py --config C2 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ch_ncu.log 2>&1; echo ncu rc=$?
timeout 900 python -m pytest tests -m gpu -x -q -k "qr or orthonormal or chol or pca_c2 or breakdown" > gpurun_out/ch_tests.log 2>&1; echo tests rc=$?
