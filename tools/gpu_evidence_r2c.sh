#!/bin/bash
# Round-2 (session 3) evidence: smoke, bench lines (C4 headline = the driver's default command, C5,
# C3, C2, N=65536), the reference arm, C4 / C2 launch lists, ncu of the four-lane resolve at C5.
O=gpurun_out/ev2c
R=/tmp/ev2c_reps
mkdir -p $O $R
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_c4.json 2> $O/bench_c4.err
timeout 900 python bench.py --config C5 --no-cpu > $O/bench_c5.json 2> $O/bench_c5.err
timeout 600 python bench.py --config C3 --no-cpu --e2e-steps 3 > $O/bench_c3.json 2> $O/bench_c3.err
timeout 600 python bench.py --config C2 --no-cpu --e2e-steps 3 --steps 20 > $O/bench_c2.json 2> $O/bench_c2.err
timeout 1200 python bench.py --n 65536 --steps 1 --warmup 3 --no-e2e --no-cpu --no-isolated > $O/bench_n65536.json 2> $O/bench_n65536.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/reference_arm.json 2> $O/reference_arm.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu --no-e2e > $O/bench_torchrun1.json 2> $O/bench_torchrun1.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $R/launches_c4.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-isolated > $O/ncu_list.log 2>&1
python tools/launch_summary.py $R/launches_c4.csv > $O/launches_c4_summary.txt 2>&1
gzip -c $R/launches_c4.csv > $O/launches_c4.csv.gz
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $R/launches_c2.csv python tools/solve_once.py --config C2 --reps 2 > $O/ncu_list_c2.log 2>&1
python tools/launch_summary.py $R/launches_c2.csv > $O/launches_c2_summary.txt 2>&1
NCU="ncu --set full --import-source on --clock-control none --kernel-name-base mangled"
timeout 900 $NCU -k regex:'resolve_lastk_quad' --launch-count 1 -f -o $R/res_c5 python tools/solve_once.py --config C5 > $O/ncu_res_c5.log 2>&1
python tools/ncu_summary.py $R/res_c5.ncu-rep > $O/res_c5_summary.txt 2>&1
timeout 900 $NCU -k regex:'transpose_panels' --launch-count 1 -f -o $R/tr_c5 python tools/solve_once.py --config C5 > $O/ncu_tr_c5.log 2>&1
python tools/ncu_summary.py $R/tr_c5.ncu-rep > $O/tr_c5_summary.txt 2>&1
