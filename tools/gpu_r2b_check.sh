#!/bin/bash
# Round-2 re-entry check: GPU suite, smoke, C2 (persistent path) and C4 bench lines.
O=gpurun_out/r2b
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 600 python bench.py --config C2 --no-cpu --e2e-steps 3 --steps 20 > $O/bench_c2.json 2> $O/bench_c2.err
timeout 600 python tools/ab_options.py --config C2 --sets "persistent=0;persistent=1" --reps 9 > $O/ab_c2.jsonl 2>&1
timeout 900 python bench.py --no-cpu --e2e-steps 3 > $O/bench_c4.json 2> $O/bench_c4.err
