#!/bin/bash
O=gpurun_out/crit
mkdir -p $O
timeout 600 python tools/ab_options.py --config C2 --sets "persist_quarters=0;persist_quarters=2;persist_quarters=1;persist_quarters=0;persist_quarters=2;persist_quarters=2,persist_gap=500;persist_quarters=2,persist_gap=900" --reps 15 > $O/ab_c2.jsonl 2>&1
timeout 600 python tools/ab_options.py --config C2 --n 2048 --sets "persist_quarters=1;persist_quarters=2;persist_quarters=0" --reps 15 > $O/ab_n2048.jsonl 2>&1
timeout 600 python tools/ab_options.py --config C2 --n 3072 --sets "persist_quarters=1;persist_quarters=2;persist_quarters=0" --reps 15 > $O/ab_n3072.jsonl 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -m gpu -q -x -k "persist or C2 or tag or real" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
for q in 2; do
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
done
