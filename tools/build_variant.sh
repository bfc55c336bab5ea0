#!/bin/bash
# Experimental build of the library with extra preprocessor flags, for A/B
# timing on the GPU box:  tools/build_variant.sh NAME -DFOO=1 ...
# -> variants/NAME/libtcsparse_b200.so ; load it with TCS_LIB_PATH=<that path>.
set -e
name=$1; shift
cd "$(dirname "$0")/.."
out=variants/$name
mkdir -p $out/obj
for f in paper_2412_11007_b200/csrc/*.cu; do
  b=$(basename $f .cu)
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    -Iinclude --expt-relaxed-constexpr "$@" -c $f -o $out/obj/$b.o &
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/libtcsparse_b200.so $out/obj/*.o
rm -rf $out/obj
echo "$out/libtcsparse_b200.so"
