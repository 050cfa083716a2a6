#!/bin/bash
# full GPU suite + smoke + default bench line
mkdir -p gpurun_out/ft
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/ft/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ft/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ft/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/ft/smoke.log
timeout 900 python bench.py > gpurun_out/ft/bench_default.json 2> gpurun_out/ft/bench_default.err
