#!/bin/bash
# Build A/B variants of the library into tools/_ab/<name>.so with extra nvcc
# defines (experiment builds; the product .so is built by __graft_entry__).
#   tools/build_ab.sh <name> [-DMACRO=value ...]
set -eu
NAME=$1; shift
mkdir -p tools/_ab
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false \
  -Xcompiler -fPIC -shared -cudart static "$@" -I include -o tools/_ab/$NAME.so paper_2401_01728_b200/csrc/ravnest_b200.cu
echo "built tools/_ab/$NAME.so $*"
