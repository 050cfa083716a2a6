#!/bin/bash
# Round-2 (session 5) evidence: the final tree's bench lines (C5, C3, C2 with e2e, N = 65536, the
# C4 line under torchrun with one rank), the C4 launch list and one ncu --set full capture of a
# mid-solve bulk launch (C4, keys, 256 deep).
O=gpurun_out/ev2e
R=/tmp/ev2e_reps
mkdir -p $O $R
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/gpu.txt 2>&1
timeout 900 python bench.py --config C5 --no-cpu > $O/bench_c5.json 2> $O/bench_c5.err
timeout 600 python bench.py --config C3 --no-cpu --e2e-steps 3 > $O/bench_c3.json 2> $O/bench_c3.err
timeout 600 python bench.py --config C2 --no-cpu --e2e-steps 3 --steps 20 > $O/bench_c2.json 2> $O/bench_c2.err
timeout 1200 python bench.py --n 65536 --steps 1 --warmup 3 --no-e2e --no-cpu --no-isolated > $O/bench_n65536.json 2> $O/bench_n65536.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu --no-e2e > $O/bench_torchrun1.json 2> $O/bench_torchrun1.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $R/launches_c4.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-isolated > $O/ncu_list.log 2>&1
python tools/launch_summary.py $R/launches_c4.csv > $O/launches_c4_summary.txt 2>&1
NCU="ncu --set full --import-source on --clock-control none --kernel-name-base mangled"
timeout 900 $NCU -k regex:'minplus_tile_kernelIfLi128ELi128ELi2ELb0E' --launch-skip 60 --launch-count 1 -f -o $R/p3_c4 python tools/solve_once.py --config C4 > $O/ncu_p3.log 2>&1
python tools/ncu_summary.py $R/p3_c4.ncu-rep > $O/p3_c4_summary.txt 2>&1
for c in c5 c3 c2 n65536 torchrun1; do python - <<PY
import json
try:
    d=json.load(open("$O/bench_$c.json")); print("$c", round(d["value"]), "GFLOPS", round(d["ms_per_step"],2), "ms", "frac", round(d["roofline"]["frac"],3), "e2e", d.get("e2e",{}).get("value"))
except Exception as e: print("$c", "failed", e)
PY
done
head -12 $O/launches_c4_summary.txt
