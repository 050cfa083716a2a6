#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "n65536" --durations=3 > gpurun_out/pytest_65536.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_65536.log
timeout 1200 python bench.py --n 65536 --steps 1 --warmup 1 --no-e2e > gpurun_out/bench_n65536.json 2> gpurun_out/bench_n65536.err; echo "rc=$?" >> gpurun_out/bench_n65536.err
