#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -m gpu -x -q -k "real or C2 or tags or lastk or C5 or loopback" > gpurun_out/pytest_resolve.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_resolve.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:resolve --csv --log-file gpurun_out/resolve_c5.csv python tools/solve_once.py --config C5 > gpurun_out/ncu_resolve.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_resolve.log
