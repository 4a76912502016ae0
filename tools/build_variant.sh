#!/bin/bash
# Build an A/B variant of the library with extra nvcc flags:
#   tools/build_variant.sh NAME [-DKNOB=VALUE ...]   ->  abso/NAME.so
set -e
name=$1; shift
d=abso/$name; mkdir -p $d
for src in runtime gemm kernels attention cnn; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I include \
    --expt-relaxed-constexpr "$@" -c paper_2505_05856_b200/csrc/$src.cu -o $d/$src.o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o abso/$name.so $d/*.o -lcudart
rm -rf $d
echo abso/$name.so
