#!/bin/bash
# ncu --set full captures (one launch each) of the three solve kernels at C4, mid-solve.
mkdir -p gpurun_out
NCU="ncu --set full --import-source on --clock-control none --kernel-name-base mangled"
timeout 600 $NCU -k regex:'minplus_tile_kernelIfLi128ELi128ELi2ELb0E' --launch-skip 64 --launch-count 1 -f -o gpurun_out/p3b_c4 python tools/solve_once.py --config C4 > gpurun_out/ncu_p3b.log 2>&1
timeout 600 $NCU -k regex:'minplus_tile_kernelIfLi128ELi128ELi2ELb1E' --launch-skip 128 --launch-count 1 -f -o gpurun_out/p2_c4 python tools/solve_once.py --config C4 > gpurun_out/ncu_p2.log 2>&1
timeout 600 $NCU -k regex:'phase1_kernel' --launch-skip 64 --launch-count 1 -f -o gpurun_out/p1_c4 python tools/solve_once.py --config C4 > gpurun_out/ncu_p1.log 2>&1
timeout 600 $NCU -k regex:'resolve_lastk' --launch-count 1 -f -o gpurun_out/resolve_c2 python tools/solve_once.py --config C2 > gpurun_out/ncu_res.log 2>&1
ls -la gpurun_out/*.ncu-rep
for r in p3b_c4 p2_c4 p1_c4 resolve_c2; do
  [ -f gpurun_out/$r.ncu-rep ] && python tools/ncu_summary.py gpurun_out/$r.ncu-rep > gpurun_out/${r}_summary.txt 2>&1
  [ -f gpurun_out/$r.ncu-rep ] && ncu -i gpurun_out/$r.ncu-rep --page raw --csv > gpurun_out/${r}_raw.csv 2>/dev/null
done
rm -f gpurun_out/resolve_c2.ncu-rep gpurun_out/p1_c4.ncu-rep
tail -5 gpurun_out/ncu_p1.log
