#!/bin/bash
# Bench lines of the configs whose inputs fit in L2 (L2 flushed before every timed step).
O=gpurun_out/small
mkdir -p $O
timeout 600 python bench.py --config C2 --no-cpu --e2e-steps 3 --steps 20 > $O/bench_c2.json 2> $O/bench_c2.err
timeout 600 python bench.py --config C1 --no-cpu --e2e-steps 3 --steps 20 > $O/bench_c1.json 2> $O/bench_c1.err
