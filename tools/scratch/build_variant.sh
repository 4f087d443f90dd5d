# Build a diagnostics variant of libhodlr2d.so: build_variant.sh OUT.so -DNAME=VALUE ...
# (apply.cu recompiled with the defines, linked with the in-tree objects of the other sources)
set -e
out=$1; shift
B=paper_2204_05536_b200/_build
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr "$@" \
  -c paper_2204_05536_b200/csrc/apply.cu -o /tmp/apply_variant.o
objs=$(ls $B/*.o | grep -v apply.o)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -Xlinker \
  --version-script=paper_2204_05536_b200/csrc/exports.map -o "$out" /tmp/apply_variant.o $objs
