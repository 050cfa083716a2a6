#!/bin/bash
# ncu --set full of the register-only operand-pattern probes: the production
# pattern (broadcast scalar + pair), the k-pair pattern (pair + pair) and the L0 mix probe
O=gpurun_out/mixncu
mkdir -p $O
NCU="ncu --set full --import-source on --clock-control none --kernel-name-base mangled"
B=paper_1811_01201_b200/csrc/bench/mix_probe
P=paper_1811_01201_b200/csrc/probe/isa_probe
timeout 300 $NCU -k regex:'_Z5probeILi8ELi2ELi0EEvPfif' --launch-skip 1 --launch-count 1 -f -o $O/prod $B > $O/prod.log 2>&1
timeout 300 $NCU -k regex:'_Z10probe_pairILi8ELi2EEvPfif' --launch-skip 1 --launch-count 1 -f -o $O/pair $B > $O/pair.log 2>&1
timeout 300 $NCU -k regex:'_Z5probeILi4EEvPfPxf' --launch-skip 1 --launch-count 1 -f -o $O/l0mix $P > $O/l0mix.log 2>&1
for r in prod pair l0mix; do python tools/ncu_summary.py $O/$r.ncu-rep > $O/${r}_summary.txt 2>&1; done
ls -la $O
