#!/bin/bash
O=gpurun_out/crit2
mkdir -p $O
for q in 0 2; do
FW_PERSIST_TRACE=/tmp/tr.bin timeout 120 python -c "
import sys; sys.path.insert(0,'.')
import torch, apsp_inputs as gen, paper_1811_01201_b200 as fw
c=gen.CONFIGS['C2']; W=gen.generate_torch(c['kind'],c['n'],c['seed'],device='cuda')
fw.fw_init(0, fw.FW_TIMING); fw.fw_set_option('persist_quarters', $q)
P=torch.empty(W.shape,dtype=torch.int32,device='cuda')
for _ in range(3):
    D=W.clone(); fw.fw_solve_device_f32(D,P,block=128,stream=torch.cuda.current_stream())
fw.fw_free()" > $O/solve_$q.log 2>&1
python tools/persist_trace.py /tmp/tr.bin --n 4096 > $O/trace_q$q.json 2>&1
cp /tmp/tr.bin $O/tr_q$q.bin
done
