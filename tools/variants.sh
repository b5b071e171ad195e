#!/bin/bash
# build libagr variants: name "flags" ...
set -e
cd /root/repo
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr"
while [ $# -gt 0 ]; do
  name=$1; flags=$2; shift 2
  mkdir -p build/var/$name
  $NV $flags -c paper_2503_01471_b200/csrc/cast.cu -o build/var/$name/cast.o
  $NV -gencode arch=compute_100a,code=sm_100a -shared -o build/var/$name/libagr.so build/blas.o build/tlas.o build/var/$name/cast.o build/checksum.o build/sim.o build/abi.o -lcudart_static -lrt -ldl -lpthread
  echo built $name
done
