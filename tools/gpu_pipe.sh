#!/bin/bash
mkdir -p gpurun_out/pipe
O=gpurun_out/pipe
timeout 900 python -m pytest tests/test_gpu_pipeline.py -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
timeout 600 python tools/pipe_probe.py --config C4 --chunks=-1 --reps 3 > $O/probe_c4.log 2>&1
timeout 600 python tools/pipe_probe.py --config C3 --chunks=-1 --reps 3 > $O/probe_c3.log 2>&1
