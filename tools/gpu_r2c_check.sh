#!/bin/bash
# Round-2 re-entry (session 3) check of HEAD: GPU suite, smoke, C4 + C2 bench lines.
O=gpurun_out/r2c
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py --no-cpu --e2e-steps 3 > $O/bench_c4.json 2> $O/bench_c4.err
timeout 600 python bench.py --config C2 --no-cpu --e2e-steps 3 --steps 20 > $O/bench_c2.json 2> $O/bench_c2.err
