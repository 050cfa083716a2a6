#!/bin/bash
# prio strips on the pivot stream beside the bulk launch (FW_PAIR_ORDER=1) vs before it (0)
mkdir -p gpurun_out/po
timeout 900 python -m pytest tests -m gpu -x -q -k "pair or fuzz or pipeline" > gpurun_out/po/pytest.log 2>&1
for o in 1 0 1 0; do
  FW_PAIR_ORDER=$o timeout 300 python bench.py --steps 5 --warmup 3 >> gpurun_out/po/c4_$o.jsonl 2>> gpurun_out/po/err.log
done
for o in 1 0; do
  FW_PAIR_ORDER=$o timeout 300 python bench.py --config C3 --steps 10 --warmup 3 >> gpurun_out/po/c3_$o.jsonl 2>> gpurun_out/po/err.log
done
