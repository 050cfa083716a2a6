#!/bin/bash
mkdir -p gpurun_out
timeout 600 python bench.py --no-cpu --no-e2e > gpurun_out/b_c4.json 2> gpurun_out/b_c4.err
timeout 900 python bench.py --config C5 --no-cpu --no-e2e --steps 2 --warmup 3 > gpurun_out/b_c5.json 2> gpurun_out/b_c5.err
timeout 600 python bench.py --config C3 --no-cpu --no-e2e > gpurun_out/b_c3.json 2> gpurun_out/b_c3.err
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "C1 or C2 or complete or ring or mixed or lastk or keyed" > gpurun_out/pytest_some.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_some.log
