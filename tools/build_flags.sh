#!/bin/bash
# Build the working tree's library with extra nvcc flags into lib/alt_NAME.so:
#   tools/build_flags.sh NAME -DFOO=1 ...
NAME=$1; shift
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
  -fmad=false -prec-div=true -prec-sqrt=true -ftz=false -Xcompiler -fPIC,-ffp-contract=off,-O2 \
  -shared "$@" -I include -o paper_1505_08023_b200/lib/alt_$NAME.so \
  paper_1505_08023_b200/csrc/api.cu paper_1505_08023_b200/csrc/kernels.cu \
  paper_1505_08023_b200/csrc/plan.cpp -lcudart -ldl && echo paper_1505_08023_b200/lib/alt_$NAME.so
