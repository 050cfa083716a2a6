#!/bin/bash
mkdir -p gpurun_out/pipe
O=gpurun_out/pipe
timeout 900 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_parity.py -m gpu -x -q -k "pipeline or pair or C4 or C2 or keyed" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
timeout 600 python tools/pipe_probe.py --config C4 --chunks=-1 --reps 3 > $O/probe_c4.log 2>&1
timeout 600 python tools/pipe_probe.py --config C3 --chunks=-1 --reps 3 > $O/probe_c3.log 2>&1
timeout 900 python bench.py --config C5 --no-cpu --no-e2e --steps 2 --warmup 1 > $O/bench_c5.json 2>/dev/null
