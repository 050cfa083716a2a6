#!/bin/bash
# small-n phase 2 as two half-width launches on two streams (FW_SPLIT_P2=1) vs one dual launch (0)
mkdir -p gpurun_out/sp
O=gpurun_out/sp
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
for o in 1 0 1 0; do
  FW_SPLIT_P2=$o timeout 300 python bench.py --config C2 --steps 20 --warmup 3 --no-cpu --e2e-steps 3 >> $O/c2_$o.jsonl 2>> $O/err.log
  FW_SPLIT_P2=$o timeout 300 python bench.py --config C3 --steps 10 --warmup 3 --no-cpu --e2e-steps 3 >> $O/c3_$o.jsonl 2>> $O/err.log
done
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e >> $O/c4.jsonl 2>> $O/err.log
