#!/bin/bash
# Build the development micro-benchmarks (not part of the library) with absolute paths.
set -e
B=/root/repo/paper_1811_01201_b200/csrc/bench
P=/root/repo/paper_1811_01201_b200/csrc/probe
NVCC="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17"
$NVCC -o $B/p3x $B/p3x.cu             # phase-3 tile-shape / pipeline explorer
$NVCC -o $B/mix_probe $B/mix_probe.cu # register- and smem-fed relaxation mix
$NVCC -o $P/isa_probe $P/isa_probe.cu # L0 instruction throughput probe
$NVCC -o $P/nvls_probe $P/nvls_probe.cu -L/usr/local/cuda/lib64/stubs -lcuda   # NVLS multicast probe
$NVCC -o $P/pdl_probe $P/pdl_probe.cu   # programmatic dependent launch probe
