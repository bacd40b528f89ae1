# rolled LU nomination panels vs the unrolled build: bitwise (twice), whole-PCA A/B, C2 launch list
N=paper_1412_3510_b200/librpca.so; B=.scratch/var/base/librpca.so
timeout 900 python tools/gpu/bitwise_ab.py $N $B > gpurun_out/rl_bitwise1.log 2>&1; echo bw1 rc=$?
timeout 900 python tools/gpu/bitwise_ab.py $N $B > gpurun_out/rl_bitwise2.log 2>&1; echo bw2 rc=$?
for c in C2 C4 C5; do timeout 900 python tools/gpu/ab_pass.py pca:$c 9 $N $B > gpurun_out/rl_ab_$c.log 2>&1; echo ab $c rc=$?; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/rl_C2_launches.csv python bench.py --config C2 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/rl_ncu.log 2>&1; echo ncu rc=$?
