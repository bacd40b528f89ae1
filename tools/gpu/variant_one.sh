# one-file library variants: FILE=<csrc file stem> VARIANTS="name:-DFLAG=v,..." →
# ${VAR_DIR:-.scratch/var}/<name>/librpca.so (the other objects from build/; run `make` first)
set -e
for spec in $VARIANTS; do
  name=${spec%%:*}; flags=${spec#*:}; flags=${flags//,/ }
  d=${VAR_DIR:-.scratch/var}/$name; mkdir -p $d
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
    -Xptxas -warn-spills $flags -Iinclude -c paper_1412_3510_b200/csrc/$FILE.cu -o $d/$FILE.o
  objs=$(ls build/*.o | grep -v "/$FILE.o")
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $d/librpca.so $objs $d/$FILE.o -lcudart -ldl
done
