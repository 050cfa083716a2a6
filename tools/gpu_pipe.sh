#!/bin/bash
# Host pipeline: its GPU tests, then the e2e probes (C4 pinned/pageable, C5, C3).
mkdir -p gpurun_out/pipe
O=gpurun_out/pipe
timeout 900 python -m pytest tests/test_gpu_pipeline.py -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
timeout 600 python tools/pipe_probe.py --config C4 --chunks -1 --reps 3 > $O/probe_c4.log 2>&1
timeout 900 python tools/pipe_probe.py --config C4 --chunks 0,-1 --reps 2 --pageable > $O/probe_c4_pageable.log 2>&1
timeout 600 python tools/pipe_probe.py --config C3 --chunks -1 --reps 3 > $O/probe_c3.log 2>&1
timeout 900 python tools/pipe_probe.py --config C5 --chunks -1 --reps 2 > $O/probe_c5.log 2>&1
