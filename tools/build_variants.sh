# Compile-time variants of libfde.so for tools/ab_lib.sh (dev tool).
# usage: bash tools/build_variants.sh "name:-DFOO=1 -DBAR=2" ...
mkdir -p paper_1808_02937_b200/variants
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  (cd paper_1808_02937_b200/csrc && /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
     -Xcompiler -fPIC -cudart static -shared $flags -o ../variants/libfde_$name.so libfde.cu api.cpp tables.cpp -ldl) &
done
wait
ls -la paper_1808_02937_b200/variants
