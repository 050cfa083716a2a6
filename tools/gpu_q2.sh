#!/bin/bash
O=gpurun_out/q2
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py tests/test_gpu_fuzz.py -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
timeout 600 python bench.py --config C2 --no-cpu --e2e-steps 3 --steps 20 > $O/bench_c2.json 2> $O/bench_c2.err
