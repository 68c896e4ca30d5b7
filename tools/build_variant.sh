#!/bin/bash
# bash tools/build_variant.sh NAME [-DFLAG=V ...]: the library with extra defines into build/ab/NAME.so (for tools/ab_multi.sh)
name=$1; shift
mkdir -p build/ab
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v "$@" \
  -shared -o build/ab/$name.so paper_1011_0093_b200/csrc/capi.cu 2> build/ab/$name.ptxas.log || { tail -20 build/ab/$name.ptxas.log; exit 1; }
