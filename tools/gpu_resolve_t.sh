#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:resolve --csv --log-file gpurun_out/resolve_c5.csv python tools/solve_once.py --config C5 > gpurun_out/ncu_resolve.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:resolve --csv --log-file gpurun_out/resolve_c2.csv python tools/solve_once.py --config C2 > gpurun_out/ncu_resolve2.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "real or C2 or lastk or mixed" > gpurun_out/pytest_res.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_res.log
