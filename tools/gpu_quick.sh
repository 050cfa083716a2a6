#!/bin/bash
# tests + bench (C4) + launch list
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "bench rc=$?" >> gpurun_out/bench_c4.err
FW_LOOKAHEAD=0 timeout 600 python bench.py --no-cpu --no-e2e > gpurun_out/bench_c4_nola.json 2> gpurun_out/bench_c4_nola.err
