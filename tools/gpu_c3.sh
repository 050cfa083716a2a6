#!/bin/bash
mkdir -p gpurun_out
timeout 600 python bench.py --config C3 --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 600 python bench.py --config C2 --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_c4.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu.log 2>&1
