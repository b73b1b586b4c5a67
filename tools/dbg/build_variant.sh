#!/bin/bash
# build a variant of the engine library with extra nvcc defines:
#   tools/dbg/build_variant.sh NAME "-DFOO=1 -DBAR=2"
set -e
cd "$(dirname "$0")/../.."
mkdir -p tools/dbg/variants /tmp/variant_$1
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC $2"
for f in elementwise gemm deal layers; do nvcc $F -c -o /tmp/variant_$1/$f.o paper_2104_10949_b200/csrc/$f.cu; done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o tools/dbg/variants/lib_$1.so /tmp/variant_$1/*.o
