#!/bin/bash
# first-hit resolve: memcheck on a straddling size, TAG-mode tests, C2 / C5 bench lines, C2 resolve ncu
mkdir -p gpurun_out/rs
timeout 600 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/solve_once.py --config C2 --n 640 > gpurun_out/rs/memcheck.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/rs/memcheck.log
timeout 600 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/solve_once.py --config C2 --n 1000 --block 64 > gpurun_out/rs/memcheck64.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/rs/memcheck64.log
timeout 900 python -m pytest tests -m gpu -x -q -k "tag or real or C2 or fuzz or pipeline" > gpurun_out/rs/pytest.log 2>&1
timeout 300 python bench.py --config C2 --no-cpu --e2e-steps 3 > gpurun_out/rs/c2.json 2>> gpurun_out/rs/err.log
timeout 600 python bench.py --config C5 --no-cpu --steps 2 --warmup 3 > gpurun_out/rs/c5.json 2>> gpurun_out/rs/err.log
NCU="ncu --set full --import-source on --clock-control none --kernel-name-base mangled"
timeout 300 $NCU -k regex:resolve_lastk --launch-count 1 -f -o gpurun_out/rs/res_c2 python tools/solve_once.py --config C2 > gpurun_out/rs/ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/rs/res_c2.ncu-rep > gpurun_out/rs/res_c2_summary.txt 2>&1
