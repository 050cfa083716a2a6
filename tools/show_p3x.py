import json, sys
for l in open(sys.argv[1]):
    try:
        d = json.loads(l)
    except Exception:
        print(l.rstrip()); continue
    print(f"{d['variant']:32s} regs={d['regs']:3d} spill={d['spill']:3d} occ={d['occ']} ms={d['ms']:.3f} relax/clk/SM={d['relax_per_clk_sm_at_max_clock']:.2f}")
