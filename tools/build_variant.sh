#!/bin/bash
# Build the library of git revision REV into paper_1505_08023_b200/lib/alt_NAME.so (A/B runs
# load it with MINIFE_LIB_PATH).  Usage: tools/build_variant.sh REV NAME
set -e
REV=$1; NAME=$2
T=$(mktemp -d)
git archive "$REV" paper_1505_08023_b200/csrc include | tar -x -C "$T"
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
  -fmad=false -prec-div=true -prec-sqrt=true -ftz=false -Xcompiler -fPIC,-ffp-contract=off,-O2 \
  -shared -I "$T/include" -o paper_1505_08023_b200/lib/alt_$NAME.so \
  "$T"/paper_1505_08023_b200/csrc/api.cu "$T"/paper_1505_08023_b200/csrc/kernels.cu \
  "$T"/paper_1505_08023_b200/csrc/plan.cpp -lcudart -ldl
rm -rf "$T"
echo paper_1505_08023_b200/lib/alt_$NAME.so
