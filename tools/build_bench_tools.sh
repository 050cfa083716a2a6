#!/bin/bash
# Build the development micro-benchmarks (not part of the library) with absolute paths.
set -e
B=/root/repo/paper_1811_01201_b200/csrc/bench
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xptxas -v \
  -o $B/p3_variants $B/p3_variants.cu > /tmp/ptx_p3v.log 2>&1 || { grep -i error /tmp/ptx_p3v.log; exit 1; }
grep -A2 "Compiling entry function" /tmp/ptx_p3v.log | grep -E "Compiling|spill" | paste - - \
  | sed -E "s/.*function .//; s/' for 'sm_100a'//" | awk '{print $1, $2, $3, $6, $7}' | grep -v " 0 bytes spill" || true
