#!/bin/bash
# Panel transpose (TAG post-pass): dist + pipeline + parity tests; C2 / C5 A-B numbers.
O=gpurun_out/panels
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_dist.py tests/test_gpu_pipeline.py tests/test_gpu_parity.py -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
timeout 300 python tools/ab_options.py --config C2 --sets "pairs=1;pairs=1" --reps 9 > $O/ab_c2.jsonl 2>&1
timeout 600 python tools/ab_options.py --config C5 --sets "pairs=1" --reps 2 > $O/ab_c5.jsonl 2>&1
