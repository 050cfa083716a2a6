#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:phase1 -c 20 --csv --log-file gpurun_out/p1_c4.csv python tools/solve_once.py --config C4 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:phase1 -c 20 --csv --log-file gpurun_out/p1_c2.csv python tools/solve_once.py --config C2 > /dev/null 2>&1
timeout 600 python bench.py --no-cpu --no-e2e > gpurun_out/b_c4.json 2> gpurun_out/b_c4.err
timeout 600 python bench.py --config C2 --no-cpu --no-e2e > gpurun_out/b_c2.json 2> gpurun_out/b_c2.err
timeout 600 python bench.py --config C3 --no-cpu --no-e2e > gpurun_out/b_c3.json 2> gpurun_out/b_c3.err
