#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:phase1 -c 20 --csv --log-file gpurun_out/p1_launches.csv python tools/solve_once.py --config C4 > gpurun_out/ncu_p1l.log 2>&1
