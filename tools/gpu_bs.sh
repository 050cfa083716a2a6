#!/bin/bash
mkdir -p gpurun_out
for b in 64 32; do
  timeout 900 python bench.py --block $b --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_c4_bs$b.json 2> gpurun_out/bench_c4_bs$b.err
done
