#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:resolve --csv --log-file gpurun_out/resolve_c5.csv python tools/solve_once.py --config C5 > gpurun_out/ncu_resolve.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:resolve --csv --log-file gpurun_out/resolve_c2.csv python tools/solve_once.py --config C2 > gpurun_out/ncu_resolve2.log 2>&1
timeout 600 python bench.py --config C2 --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
