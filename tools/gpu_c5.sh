#!/bin/bash
mkdir -p gpurun_out
free -g > gpurun_out/mem.txt; nproc >> gpurun_out/mem.txt; lscpu | grep "Model name" >> gpurun_out/mem.txt
python tools/mc_probe.py > gpurun_out/mc.txt 2>&1
nvidia-smi topo -m >> gpurun_out/mc.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "C5" --durations=5 > gpurun_out/pytest_c5.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_c5.log
timeout 900 python bench.py --config C5 --steps 2 --warmup 3 --no-cpu > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "rc=$?" >> gpurun_out/bench_c5.err
