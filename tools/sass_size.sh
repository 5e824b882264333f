#!/bin/bash
# SASS instruction count per kernel of one CUDA source: tools/sass_size.sh file.cu
cd /root/repo/paper_1903_12294_b200/csrc && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -fmad=false \
  -Xcompiler -fPIC,-ffp-contract=off --expt-relaxed-constexpr -cubin -o /tmp/sass_size.cubin $1 2>/dev/null && \
  cuobjdump -sass /tmp/sass_size.cubin | awk '/Function :/{f=$3} /^ +\/\*[0-9a-f]+\*\//{n[f]++} END{for (k in n) print n[k], k}' | sort -k2
