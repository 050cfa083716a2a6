#!/bin/bash
O=gpurun_out/lone
mkdir -p $O
timeout 600 python tools/ab_options.py --config C2 --sets "persist_p1_lone=0;persist_p1_lone=1;persist_p1_lone=0;persist_p1_lone=1;persist_p1_lone=1,persist_quarters=1" --reps 15 > $O/ab_c2.jsonl 2>&1
timeout 600 python tools/ab_options.py --config C2 --n 2048 --sets "persist_p1_lone=0;persist_p1_lone=1" --reps 15 > $O/ab_n2048.jsonl 2>&1
timeout 600 python tools/ab_options.py --config C2 --n 3072 --sets "persist_p1_lone=0;persist_p1_lone=1" --reps 15 > $O/ab_n3072.jsonl 2>&1
timeout 600 python tools/ab_options.py --config C3 --sets "persistent=1,persist_p1_lone=0;persistent=1,persist_p1_lone=1;persistent=0" --reps 5 > $O/ab_c3.jsonl 2>&1
python - > $O/check.log 2>&1 <<'PY'
import sys; sys.path.insert(0,'.')
import numpy as np, torch, apsp_inputs as gen, oracle, paper_1811_01201_b200 as fw
for kind, n in [("complete_real", 1000), ("complete_int", 1536), ("er_int", 900)]:
    W = gen.generate(kind, n, 5, p=0.05, lo=1, hi=1000 if kind.startswith("er") else 100)
    fw.fw_init(0, 0); fw.fw_set_option("persistent", 1); fw.fw_set_option("persist_p1_lone", 1)
    dD = torch.from_numpy(W).cuda(); dP = torch.empty(W.shape, dtype=torch.int32, device="cuda")
    (fw.fw_solve_device_i32 if W.dtype == np.int32 else fw.fw_solve_device_f32)(dD, dP, block=128, stream=torch.cuda.current_stream())
    s = fw.fw_last_stats(); fw.fw_free()
    D = dD.cpu().numpy(); P = dP.cpu().numpy(); Dr = oracle.fw(W, None)[0]
    ok = np.array_equal(D, Dr) if W.dtype == np.int32 or kind == "complete_int" else np.allclose(D, Dr, rtol=1e-5)
    print(kind, n, "persistent", s.persistent, "D ok", ok, "bad paths", oracle.check_paths(W, D, P, rtol=1e-5)[0])
PY
