#!/bin/bash
# Build tuning variants of libmt.so into variants/ (git-ignored *.so).
# usage: tools/build_variants.sh name "-DFLAG=..." [name "-D..."]...
cd "$(dirname "$0")/.."
SRC=$(ls paper_2603_28907_b200/csrc/*.cu)
while [ $# -gt 1 ]; do
  name=$1; flags=$2; shift 2
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -ftz=true \
    -Xcompiler -fPIC -Xcompiler -O2 --expt-relaxed-constexpr $flags -shared \
    -o variants/libmt_$name.so $SRC -lcudart -ldl &
done
wait
ls -la variants
