#!/bin/bash
# Host pipeline: its GPU tests, the chunk-size probe, then the C4 bench line.
mkdir -p gpurun_out/pipe
O=gpurun_out/pipe
timeout 900 python -m pytest tests/test_gpu_pipeline.py -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
timeout 600 python tools/pipe_probe.py --chunks 0,-1,16,32 > $O/probe_c4.log 2>&1; echo "probe rc=$?" >> $O/probe_c4.log
timeout 600 python bench.py --no-cpu --e2e-steps 3 > $O/bench_c4.json 2> $O/bench_c4.err; echo "bench rc=$?" >> $O/bench_c4.err
