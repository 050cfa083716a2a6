#!/bin/bash
# Persistent C2: the P2(K+1) placement (persist_gap) against the per-round pivot chain.
O=gpurun_out/gap
mkdir -p $O
timeout 600 python tools/ab_options.py --config C2 --sets "persist_gap=-1;persist_gap=150;persist_gap=300;persist_gap=450;persist_gap=600;persist_gap=-1;persist_gap=900;persist_gap=300,persist_quarters=0;persist_gap=-1,persist_quarters=0" --reps 9 > $O/ab_gap.jsonl 2>&1
for g in 300 450; do
  FW_PERSIST_TRACE=/tmp/tr.bin timeout 120 python -c "
import sys; sys.path.insert(0,'.')
import torch, apsp_inputs as gen, paper_1811_01201_b200 as fw
c=gen.CONFIGS['C2']; W=gen.generate_torch(c['kind'],c['n'],c['seed'],device='cuda')
fw.fw_init(0, fw.FW_TIMING); fw.fw_set_option('persist_gap', $g)
P=torch.empty(W.shape,dtype=torch.int32,device='cuda')
for _ in range(3):
    D=W.clone(); fw.fw_solve_device_f32(D,P,block=128,stream=torch.cuda.current_stream())
fw.fw_free()" > $O/solve_$g.log 2>&1
  python tools/persist_trace.py /tmp/tr.bin --n 4096 > $O/trace_gap$g.json 2>&1
done
