#!/bin/bash
# Build A/B variants of libpastis_sw.so: tools/build_var.sh NAME "-DFLAG=.." ...
# Output var/NAME.so (git-ignored; travels to the GPU box). Load with PASTIS_SW_LIB.
set -e
cd "$(dirname "$0")/.."
mkdir -p var
name=$1; shift
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
  -Xcompiler -fPIC -shared "$@" -o var/$name.so paper_2303_01845_b200/csrc/sw_engine.cu
