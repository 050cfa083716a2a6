#!/bin/bash
# C5 launch list (1 solve) and BS sweep at C4.
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_c5.csv python tools/solve_once.py --config C5 > gpurun_out/ncu_c5.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_c5.log
for b in 64 32; do
  timeout 900 python bench.py --block $b --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_c4_bs$b.json 2> gpurun_out/bench_c4_bs$b.err
done
