#!/bin/bash
# experiment build of the Horner translation unit only:
#   tools/mkvariant.sh NAME [-DHX_... flags]  ->  variants/NAME.so
# (order-4 instantiations only; the other objects come from the last full build)
set -e
N=$1; shift
P=paper_2202_04140_b200
mkdir -p variants /tmp/hv
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 -diag-suppress 550 \
  -Xptxas -v -DACEDAG_HORNER_FAST "$@" -c -o /tmp/hv/$N.o $P/csrc/horner.cu 2> /tmp/hv/$N.ptxas
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o variants/$N.so $P/build/capi.o /tmp/hv/$N.o $P/build/graph.o \
  $P/build/graph_io.o $P/build/plan.o
grep -A2 "k2_hornerILi4EdLb1" /tmp/hv/$N.ptxas | grep -E "spill|Used" | tr '\n' ' '; echo " <- $N"
