# build library variants: VARIANTS="name:-DFLAG=v ..." → /tmp/rpca_var/<name>/librpca.so
set -e
for spec in $VARIANTS; do
  name=${spec%%:*}; flags=${spec#*:}; flags=${flags//,/ }
  d=${VAR_DIR:-/tmp/rpca_var}/$name; mkdir -p $d/obj
  for f in paper_1412_3510_b200/csrc/*.cu; do
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr $flags -Iinclude -c $f -o $d/obj/$(basename $f .cu).o &
  done
  wait
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $d/librpca.so $d/obj/*.o -lcudart -ldl
done
