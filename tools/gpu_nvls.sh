#!/bin/bash
# NVLS setup / fallback on a one-rank communicator; persistent + dist tests; C2 trace.
O=gpurun_out/nvls
mkdir -p $O
FW_DEBUG=1 timeout 600 python -m pytest tests/test_gpu_dist.py -m gpu -q -s -x -k "nvls" > $O/pytest_nvls.log 2>&1; echo "pytest rc=$?" >> $O/pytest_nvls.log
timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_parity.py -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
timeout 300 python tools/ab_options.py --config C2 --sets "persistent=1;persistent=1" --reps 9 > $O/ab_c2.jsonl 2>&1
FW_PERSIST_TRACE=/tmp/tr_c2.bin timeout 120 python tools/solve_once.py --config C2 --reps 3 > $O/solve.log 2>&1
python tools/persist_trace.py /tmp/tr_c2.bin --n 4096 > $O/trace_c2.json 2>&1
cp /tmp/tr_c2.bin $O/
