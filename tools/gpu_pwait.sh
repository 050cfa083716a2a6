#!/bin/bash
# Persistent kernel per-item overhead at C2: relaxed polls, prefetch placement; traces.
O=gpurun_out/pwait
mkdir -p $O
for v in "1 0" "1 1" "0 0" "2 0" "2 1"; do
  set -- $v
  FW_PERSIST_PREFETCH=$1 timeout 300 python tools/ab_options.py --config C2 --sets "persistent=1,persist_relaxed=$2;persistent=1,persist_relaxed=$2" --reps 9 > $O/ab_pf$1_rel$2.jsonl 2>&1
  FW_PERSIST_PREFETCH=$1 FW_PERSIST_RELAXED=$2 FW_PERSIST_TRACE=/tmp/tr.bin timeout 120 python -c "
import sys; sys.path.insert(0,'.')
import torch, apsp_inputs as gen, paper_1811_01201_b200 as fw
c=gen.CONFIGS['C2']; W=gen.generate_torch(c['kind'],c['n'],c['seed'],device='cuda')
fw.fw_init(0, fw.FW_TIMING); fw.fw_set_option('persist_relaxed', $2)
P=torch.empty(W.shape,dtype=torch.int32,device='cuda')
for _ in range(3):
    D=W.clone(); fw.fw_solve_device_f32(D,P,block=128,stream=torch.cuda.current_stream())
fw.fw_free()" > $O/solve_pf$1_rel$2.log 2>&1
  python tools/persist_trace.py /tmp/tr.bin --n 4096 > $O/trace_pf$1_rel$2.json 2>&1
done
