#!/bin/bash
# Build a tuning variant of the library: tools/build_variant.sh NAME "-DFLAG=.. ..."
set -e
cd "$(dirname "$0")/.."
mkdir -p build_variants
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared -Xcompiler -fPIC \
  -prec-div=false -prec-sqrt=false -ftz=true $2 -o build_variants/lib_$1.so paper_2212_02224_b200/csrc/bd_api.cu
echo built build_variants/lib_$1.so
