make -j16 > gpurun_out/make.log 2>&1 || { tail -30 gpurun_out/make.log; exit 1; }
for o in 0 1 2 3 7; do
  echo "== opts leaf=$o tree=$((o & 3))"
  RPCA_LU_OPTS_LEAF=$o RPCA_LU_OPTS_TREE=$((o & 3)) timeout 300 python tools/gpu/lu_micro.py 22,52,64 2>&1 | grep -v "m=     256"
done
