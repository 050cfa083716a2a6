"""Summarise an ncu report (details + per-opcode stall reasons) for profiles/."""
import collections
import csv
import io
import subprocess
import sys

KEYS = ["Duration", "Grid Size", "Block Size", "Registers Per Thread", "SM Frequency", "Issue Slots Busy",
        "Executed Ipc Active", "Eligible Warps Per Scheduler", "Warp Cycles Per Issued Instruction",
        "Achieved Active Warps Per SM", "DRAM Throughput", "L2 Hit Rate", "Memory Throughput",
        "L1/TEX Cache Throughput", "Compute (SM) Throughput"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
       "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
       "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
       "smsp__inst_executed.sum", "sm__cycles_elapsed.avg.per_second",
       "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "launch__grid_size"]


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def main(rep):
    out = []
    det = list(csv.reader(io.StringIO(ncu(rep, "--page", "details", "--csv"))))
    h = det[0]
    name = det[1][h.index("Kernel Name")] if len(det) > 1 else "?"
    out.append(f"kernel: {name}")
    for row in det[1:]:
        mname, unit, val = row[h.index("Metric Name")], row[h.index("Metric Unit")], row[h.index("Metric Value")]
        if mname in KEYS:
            out.append(f"  {mname}: {val} {unit}")
    raw = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    rh, units, rv = raw[0], raw[1], raw[2]
    for k in RAW:
        if k in rh:
            out.append(f"  {k}: {rv[rh.index(k)]} {units[rh.index(k)]}")
    src = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv", "--print-source", "sass"))))
    if len(src) > 2:
        sh = src[1]
        ia = sh.index("Source")
        cols = [c for c in sh if c.startswith("stall_") and "Not Issued" not in c]
        agg = collections.defaultdict(collections.Counter)
        tot = collections.Counter()
        for x in src[2:]:
            toks = x[ia].split()
            if not toks:
                continue
            op = toks[1] if toks[0].startswith("@") else toks[0]
            for c in cols:
                try:
                    v = int(x[sh.index(c)])
                except ValueError:
                    continue
                agg[op][c] += v
                tot[c] += v
        T = sum(tot.values()) or 1
        out.append("  stall samples (all): " + ", ".join(f"{c[6:]} {100*v/T:.1f}%" for c, v in tot.most_common(8)))
        for op in sorted(agg, key=lambda o: -sum(agg[o].values()))[:8]:
            s = sum(agg[op].values())
            out.append(f"    {op:16s} {100*s/T:5.1f}%  " + ", ".join(f"{c[6:]} {v}" for c, v in agg[op].most_common(4)))
    print("\n".join(out))


if __name__ == "__main__":
    for rep in sys.argv[1:]:
        main(rep)
