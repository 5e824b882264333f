#!/bin/bash
# registers / spills of every kernel in one CUDA source: tools/ptxas_check.sh file.cu [regex]
f=$1; pat=${2:-.}
cd /root/repo/paper_1903_12294_b200/csrc && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false \
  -Xcompiler -fPIC,-ffp-contract=off --expt-relaxed-constexpr -Xptxas -v -c $f -o /tmp/ptxas_check.o 2>&1 \
  | grep -E "error|Compiling entry|registers|spill" | grep -E "error|$pat" -A2 | grep -E "error|Compiling|registers|spill"
