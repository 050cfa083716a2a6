#!/usr/bin/env python
"""Benchmark of the blocked Floyd–Warshall APSP hot path (arxiv 1811.01201) on B200.

Metric (BASELINE.json): APSP GFLOPS = 2 n^3 / t at n = 16384 FP32 (configs[3]), plus the
phase-3 fraction of the FP32 add+min issue roofline. A "step" is one complete solve
(validate, pad/init, R = n/BS rounds of phases 1-3, next-hop post-pass) of a fresh copy of
the seeded synthetic input already resident in HBM.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference] [--config C4]

Prints ONE JSON line on rank 0. See DESIGN.md "Measurement" for every field.
"""
from __future__ import annotations

import argparse
import datetime
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import apsp_inputs as gen  # noqa: E402

METRIC = "APSP GFLOPS (2n³/s) at n=16384 FP32, 1/2/4/8 B200; % of FP32 add+min roofline"
CONFIG_DESC = {
    "C1": "n=512 complete digraph, FP32 integer weights [1,100], BS=32, next-hop P",
    "C2": "n=4096 complete digraph, FP32 real weights [1,100), BS=128, next-hop P",
    "C3": "n=8192 ER p=0.1 digraph, INT32 weights [1,1000], INF=INT32_MAX/2, BS=128, next-hop P",
    "C4": "n=16384 complete digraph, FP32 integer weights [1,100], BS=128, next-hop P",
    "C5": "n=32768 complete digraph, FP32 real weights [1,100), BS=128, next-hop P",
}
PROFILE_TRAFFIC = os.path.join(ROOT, "profiles", "phase3_traffic.json")


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def window(self, t0: float, t1: float):
        """Keep the samples that arrived while [t0, t1] (the timed region) was running; the
        sampler is started before the warm-up so short timed regions still get samples."""
        self.t0, self.t1 = t0, t1

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        t0, t1 = getattr(self, "t0", None), getattr(self, "t1", None)
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 10:
                continue
            try:   # nvidia-smi's own sample time (local time, "YYYY/MM/DD HH:MM:SS.mmm")
                ts = datetime.datetime.strptime(f[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
            except ValueError:
                ts = None
            if t0 is not None and ts is not None and not (t0 - 0.05 <= ts <= t1 + 0.05):
                continue
            f = f[1:]
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def host_matrix(cfg: dict) -> np.ndarray:
    """The whole n x n input on the host (apsp_inputs.generate)."""
    return gen.generate(cfg["kind"], cfg["n"], cfg["seed"], p=cfg.get("p", 1.0),
                        lo=cfg.get("lo", 1), hi=cfg.get("hi", 100))


def cpu_sample(cfg: dict, seconds_target: float = 15.0, W: np.ndarray | None = None):
    """Time the oracle (as it stands) on the host cores on a bounded sample of the same
    workload: the first k-iterations of the triple loop on the full n x n matrix (each
    k-iteration is n^2 relaxations = 2 n^2 flop), scaled to GFLOPS."""
    import oracle
    n = cfg["n"]
    W = host_matrix(cfg) if W is None else W.copy()
    if W.dtype == np.int32:   # INT32 config: the timing sample uses the FP32 loop on the same values
        W = np.where(W >= gen.INF_I32, np.inf, W).astype(np.float32)
    np.fill_diagonal(W, 0)
    i = np.arange(n)
    P = np.where(np.isinf(W), -1, i[None, :]).astype(np.int32)
    P[i, i] = i
    # calibrate: one step, then enough steps for ~seconds_target
    t0 = time.perf_counter()
    oracle.fw_steps(W, P, 0, 1)
    t1 = time.perf_counter() - t0
    ks = int(max(1, min(n - 1, seconds_target / max(t1, 1e-6))))
    t0 = time.perf_counter()
    oracle.fw_steps(W, P, 1, 1 + ks)
    dt = time.perf_counter() - t0
    gflops = 2.0 * n * n * ks / dt / 1e9
    cores = int(os.environ.get("OMP_NUM_THREADS", len(os.sched_getaffinity(0))))
    return {"value": gflops, "unit": "GFLOPS", "cores": cores, "kind": "oracle",
            "sample": f"PROJECTION from a bounded sample: oracle C triple loop (next-hop), k-iterations "
                      f"1..{ks} of {n} on the full {n}x{n} {cfg['name']} matrix ({ks} x n^2 "
                      f"relaxations, {dt:.1f} s); GFLOPS = 2*n^2*k_steps/t (full solves at the sizes "
                      f"the oracle completes: cpu_ladder)",
            "cpu_model": lscpu_model(), "sample_seconds": dt}


def lscpu_model() -> str:
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name:"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def oracle_full_solve(name: str, threads: int, timeout: float = 240.0) -> dict:
    """One FULL oracle solve (triple loop with next-hop P) of config `name` in a subprocess
    with OMP_NUM_THREADS = threads (SURVEY §8(d) timing protocol: C1 at 1 thread and all
    cores, C2, C3 — the sizes the oracle completes)."""
    code = ("import json, time, sys; sys.path.insert(0, %r)\n"
            "import apsp_inputs as gen, oracle\n"
            "W = gen.config_matrix(%r); oracle.lib()\n"
            "t0 = time.perf_counter(); oracle.fw(W, 'next'); dt = time.perf_counter() - t0\n"
            "print(json.dumps({'s': dt, 'n': int(W.shape[0])}))\n") % (ROOT, name)
    env = dict(os.environ, OMP_NUM_THREADS=str(threads))
    try:
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                           timeout=timeout)
        d = json.loads(r.stdout.strip().splitlines()[-1])
    except Exception as e:   # noqa: BLE001 — a baseline that could not be taken is reported as such
        return {"config": name, "threads": threads, "error": str(e)[:200]}
    n = d["n"]
    return {"config": name, "n": n, "threads": threads, "seconds": d["s"],
            "gflops": 2.0 * n ** 3 / d["s"] / 1e9}


def cpu_ladder() -> dict:
    """Full oracle solves at the sizes the oracle completes, on this host's cores."""
    cores = len(os.sched_getaffinity(0))
    runs = [oracle_full_solve("C1", 1), oracle_full_solve("C1", cores), oracle_full_solve("C2", cores),
            oracle_full_solve("C3", cores)]
    return {"kind": "oracle (plain C triple loop, next-hop P, -O3, OpenMP over i)",
            "cpu_model": lscpu_model(), "cores": cores, "runs": runs,
            "note": "full solves, not projections; GFLOPS = 2 n^3 / t (BASELINE configs[0..2])"}


def config_for(name: str, n: int = 0) -> dict:
    c = dict(gen.CONFIGS[name])
    c["name"] = name
    c["desc"] = CONFIG_DESC[name]
    if n and n != c["n"]:   # the config's recipe at another size (e.g. the paper's N=65536)
        c["desc"] = c["desc"].replace(f"n={c['n']}", f"n={n}")
        c["n"] = n
    return c


L2_BYTES = 126 * 2**20   # B200 L2 (B200_PROFILING.md)


def fits_l2(n: int) -> bool:
    return n * n * 4 <= L2_BYTES


def config_json(cfg: dict, block: int, world: int) -> dict:
    """The JSON `config` object (identical on both arms)."""
    n = cfg["n"]
    desc = cfg["desc"].replace(f"BS={cfg['block']}", f"BS={block}")
    return {"workload": desc, "config": cfg["name"], "n": n, "block": block,
            "seed": cfg["seed"], "path": "next-hop",
            "l2": (f"inputs larger than L2 (D and P {n * n * 4 / 2**30:g} GiB each)" if not fits_l2(n)
                   else f"inputs fit in L2 ({n * n * 4 / 2**20:g} MiB): L2 flushed (a {2 * L2_BYTES >> 20} MiB "
                        "write) before every step, outside the timed spans (steps timed one by one and summed)"),
            "parallelism": "single GPU" if world == 1 else
            f"{world}-way block-row partition, per-round NCCL pivot-strip broadcast"}


def run_reference(args, cfg):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    W = host_matrix(cfg)
    base = cpu_sample(cfg, seconds_target=max(2.0, 20.0 / max(1, args.steps + args.warmup)), W=W)
    # each step is one bounded sample; report the median over steps
    vals, secs = [], []
    for _ in range(args.warmup):
        cpu_sample(cfg, seconds_target=3.0, W=W)
    for _ in range(args.steps):
        r = cpu_sample(cfg, seconds_target=max(2.0, 30.0 / max(1, args.steps)), W=W)
        vals.append(r["value"])
        secs.append(r["sample_seconds"])
    v = statistics.median(vals) if vals else base["value"]
    n = cfg["n"]
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "GFLOPS", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup,
        # a step is one bounded sample (k-slice) of the workload: its measured wall time; the
        # full solve at the sampled rate would take ms_per_full_solve_projected
        "ms_per_step": 1e3 * statistics.mean(secs) if secs else None,
        "ms_per_full_solve_projected": 2.0 * n ** 3 / (v * 1e9) * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic", "config": config_json(cfg, args.block or cfg["block"], args.gpus),
        "cpu_baseline": {**base, "value": v},
        "e2e": {"value": v, "unit": "GFLOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def isolated_pivot_phases(fw, solve, dD, dW, dP, n, n_pad, BS, stream, peak_tflops, mix_tflops):
    """Phases 1 and 2 timed ALONE: one extra solve (after the timed region) with the look-ahead
    and the two-rounds-per-pass schedule switched off (fw_set_option), so phase 1, the dual
    phase-2 strip launch and phase 3 of every round run back to back on one stream and the
    library's per-phase CUDA events bracket each launch on an otherwise idle GPU."""
    fw.fw_set_option("lookahead", 0)
    fw.fw_set_option("pairs", 0)
    fw.fw_set_option("persistent", 0)          # the stream schedule: one launch per phase
    try:
        for _ in range(2):                      # the second solve is reported
            dD.copy_(dW)
            solve(dD, dP, n=n, ld=n, block=BS, stream=stream)
            s = fw.fw_last_stats()
    finally:
        fw.fw_set_option("lookahead", 1)
        fw.fw_set_option("pairs", 1)
        ps = os.environ.get("FW_PERSISTENT", "-1")
        fw.fw_set_option("persistent", int(ps) if ps in ("-1", "0", "1") else -1)
    R = s.rounds
    p1_us, p2_us = 1e3 * s.phase1_ms / R, 1e3 * s.phase2_ms / R
    p2_relax = 2.0 * BS * BS * (n_pad - BS)     # row + column strip through BS k each
    p2_bytes = 2.0 * BS * n_pad * 4             # each strip element read once (changed ones written)
    import json as _j
    peaks = {}
    try:
        peaks = _j.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm = peaks.get("hbm_gbs", 6650.0)
    return {
        "phase1_us_per_round": p1_us,
        "phase1_relax_per_round": float(BS) ** 3,
        "phase2_us_per_round": p2_us,
        "phase2_relax_per_round": p2_relax,
        "phase2_tflops": 2.0 * p2_relax / (p2_us * 1e-6) / 1e12 if p2_us > 0 else None,
        "phase2_frac_stated_alu": (2.0 * p2_relax / (p2_us * 1e-6) / 1e12) / peak_tflops if p2_us > 0 else None,
        "phase2_frac_measured_mix": (2.0 * p2_relax / (p2_us * 1e-6) / 1e12) / mix_tflops if p2_us > 0 else None,
        "phase2_alg_bytes_per_round": p2_bytes,
        "phase2_gbps": p2_bytes / (p2_us * 1e-6) / 1e9 if p2_us > 0 else None,
        "phase2_frac_hbm": (p2_bytes / (p2_us * 1e-6) / 1e9) / hbm if p2_us > 0 else None,
        "hbm_peak_gbs": hbm,
        "solve_ms_serialized": s.solve_ms,
        "note": "one extra solve with fw_set_option(lookahead=0, pairs=0, persistent=0): per-round phase-1 and dual "
                "phase-2 launch times from the library's CUDA events, serialized on one stream. The "
                "strips run BS relaxations per 4-byte element (32 relax/B at BS=128): ALU-bound, not "
                "HBM-bound, so phase2_frac_measured_mix is the fraction that matters",
    }


def run_gpu(args, cfg):
    import torch
    import paper_1811_01201_b200 as fw

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    n, BS = cfg["n"], args.block or cfg["block"]
    is_int = cfg["kind"] == "er_int"
    fw.fw_init(0, fw.FW_TIMING)
    if world > 1:
        from paper_1811_01201_b200 import dist as fwdist
        fwdist.comm_init_from_torch()
    # this rank's block-rows (all rows on one GPU): the partition the library uses
    row0, nrows = fw.fw_dist_partition(n, world, rank)
    dW = gen.generate_torch(cfg["kind"], n, cfg["seed"], device=dev, p=cfg.get("p", 1.0),
                            lo=cfg.get("lo", 1), hi=cfg.get("hi", 100),
                            rows=(row0, row0 + nrows))  # resident input (never modified)
    torch.cuda.synchronize()
    dD = torch.empty_like(dW)
    dP = torch.empty((nrows, n), dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream()
    if world > 1:
        solve = fw.fw_dist_solve_device_i32 if is_int else fw.fw_dist_solve_device_f32
    else:
        solve = fw.fw_solve_device_i32 if is_int else fw.fw_solve_device_f32

    def step():
        dD.copy_(dW)                                         # fresh input, device-resident
        solve(dD, dP, n=n, ld=n, block=BS, stream=stream)
        return fw.fw_last_stats()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item())

    with ClockSampler(local) as clk:   # started before the warm-up: samples from the first step on
        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        stats = []
        t_start = time.time()
        if fits_l2(n):
            # the inputs fit in L2: flush it (write a buffer twice its size) before every step,
            # outside the timed spans; the steps are timed one by one and summed
            flush = torch.empty(2 * L2_BYTES // 4, dtype=torch.int32, device=dev)
            spans = []
            for _ in range(args.steps):
                flush.fill_(1)
                a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a_.record(stream)
                stats.append(step())
                b_.record(stream)
                spans.append((a_, b_))
            torch.cuda.synchronize()
            ms_local = sum(a_.elapsed_time(b_) for a_, b_ in spans)
            del flush
        else:
            e0.record(stream)
            for _ in range(args.steps):
                stats.append(step())
            e1.record(stream)
            torch.cuda.synchronize()
            ms_local = e0.elapsed_time(e1)
        clk.window(t_start, time.time())
    if world > 1:
        torch.distributed.barrier()
    ms_total = max_over_ranks(ms_local)
    ms_per_step = ms_total / args.steps
    flops = 2.0 * float(n) ** 3
    gflops = flops * args.steps / (ms_total * 1e-3) / 1e9      # whole job (strong scaling)

    # roofline of the dominant kernel (phase 3): algorithmic flops per launch / avg duration
    props = torch.cuda.get_device_properties(dev)
    sms = props.multi_processor_count
    max_mhz = 1965.0
    try:
        import pynvml  # nvidia_ml_py
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(local)
        max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
    except Exception:
        pass
    peak_tflops = sms * 128 * max_mhz * 1e6 / 1e12       # SMs x 128 lanes x f (2 flop/relax)
    p3_ms = sum(s.phase3_ms for s in stats)
    p3_launches = sum(s.phase3_launches for s in stats)
    p3_relax = sum(s.phase3_relaxations for s in stats)
    avg_launch_ms = p3_ms / max(1, p3_launches)
    achieved_tflops = 2.0 * p3_relax / (p3_ms * 1e-3) / 1e12 if p3_ms > 0 else None
    traffic = None
    if os.path.exists(PROFILE_TRAFFIC):   # ncu capture of this config's phase-3 launch, if any
        try:
            t = json.load(open(PROFILE_TRAFFIC))
            if t.get("n") == n and t.get("block") == BS and t.get("config") == cfg["name"]:
                traffic = t.get("bytes_per_launch")
        except Exception:
            traffic = None
    s0 = stats[0]
    mode = {0: "PLAIN", 1: "TAG", 2: "KEY"}.get(s0.p_method, "?")
    ctype = "float" if s0.compute_f32 else "int32_t"
    # other ceilings, for context: FADD2 + FMNMX3 issue once per relaxation (2x the stated
    # model), and the L0 probe's measured FADD2+FMNMX3 mix (profiles/r01_isa_probe.jsonl)
    single_issue = sms * 128 * max_mhz * 1e6 * 2 / 1e12
    mix = sms * 95.53 * max_mhz * 1e6 * 2 / 1e12
    # the production operand pattern (FADD2 broadcast scalar + pair, FMNMX3 on two pairs) from
    # registers only: 78.4 relax/clk/SM (profiles/r02e_mix_probe_orders.jsonl)
    pattern = sms * 78.4 * max_mhz * 1e6 * 2 / 1e12
    phase2_ms = sum(s.phase2_ms for s in stats) / len(stats)
    n_pad = (n + 127) // 128 * 128
    roof = {"bound": "alu", "achieved": achieved_tflops, "peak": peak_tflops, "unit": "TFLOP/s",
            "frac": (achieved_tflops / peak_tflops) if achieved_tflops else None,
            "traffic": traffic,
            "kernel": (f"fw_persistent_kernel<{ctype},{mode}> (the whole solve's rounds as ONE persistent "
                       "launch, DESIGN.md 4.10: phase-1/2/3 work items; achieved = all n_pad^3 relaxations "
                       "of the launch / its duration)") if s0.persistent else
                      (f"minplus_tile_kernel<{ctype},128,128,{mode}> (phase 3, rank 0"
                       + (", two rounds per pass: 256-deep bulk launches" if s0.phase3_launches < s0.rounds else "")
                       + ")"),
            "launches_per_step": p3_launches / len(stats),
            "avg_launch_ms": avg_launch_ms,
            "flop_per_launch": 2.0 * p3_relax / max(1, p3_launches),
            "timing": "phase-3 CUDA-event span of the step / bulk launches in it (library FW_TIMING "
                      "events on the launching stream; consecutive bulk launches overlap by PDL, so "
                      "the span is their union)",
            "peak_basis": f"stated FP32 add+min issue roofline: {sms} SMs x 128 lanes x {max_mhz:.0f} MHz "
                          "(2 flop per relaxation, BASELINE north_star)",
            "other_ceilings": {
                "single_issue_tflops": single_issue,
                "frac_single_issue": (achieved_tflops / single_issue) if achieved_tflops else None,
                "measured_mix_tflops": mix,
                "frac_measured_mix": (achieved_tflops / mix) if achieved_tflops else None,
                "operand_pattern_tflops": pattern,
                "frac_operand_pattern": (achieved_tflops / pattern) if achieved_tflops else None,
                "basis_operand_pattern": "register-only probe of the kernel's own FADD2 (broadcast scalar "
                                         "+ pair) / FMNMX3 (two pairs) operand pattern, 16 warps/SM: 78.4 "
                                         "relax/clk/SM; the 95.5 mix probe shares one scalar register between consecutive FADD2s (75.8 without)",
                "basis": "FADD2 (2 adds) + FMNMX3 (2 mins) = one issue slot per relaxation: "
                         "SMs x 128 relax/clk; L0 probe FADD2+FMNMX3 mix 95.5 relax/clk/SM"},
            "phase_ms_per_step": {"phase1": sum(s.phase1_ms for s in stats) / len(stats),
                                  "phase2": phase2_ms,
                                  "phase3": p3_ms / len(stats),
                                  "post": sum(s.post_ms for s in stats) / len(stats)}}
    if world == 1 and BS == 128 and not args.no_isolated:
        roof["pivot_path_isolated"] = isolated_pivot_phases(fw, solve, dD, dW, dP, n, n_pad, BS, stream,
                                                           peak_tflops, mix)
    launches = sum(s.kernel_launches for s in stats)

    # e2e: the same metric through the public API with pinned host buffers, H2D + solve + D2H
    e2e = None
    W = dW.cpu().numpy() if (not args.no_e2e or (rank == 0 and world == 1 and not args.no_cpu)) else None
    if not args.no_e2e:
        host_in = torch.from_numpy(W).pin_memory()
        hD = torch.empty_like(host_in).pin_memory()
        hP = torch.empty((nrows, n), dtype=torch.int32).pin_memory()
        ts, hs = [], []
        for it in range(max(1, args.e2e_steps) + 1):
            hD.copy_(host_in)
            torch.cuda.synchronize()
            if world > 1:
                torch.distributed.barrier()
            t0 = time.perf_counter()
            if world == 1:
                (fw.fw_solve_i32 if is_int else fw.fw_solve)(hD, hP, block=BS, ngpus=1)
            else:
                dD.copy_(hD, non_blocking=True)
                solve(dD, dP, n=n, ld=n, block=BS, stream=stream)
                hD.copy_(dD, non_blocking=True)
                hP.copy_(dP, non_blocking=True)
                torch.cuda.synchronize()
            dt = max_over_ranks(time.perf_counter() - t0)
            if it > 0:       # the first call warms the host-side staging
                ts.append(dt)
                if world == 1:
                    hs.append(fw.fw_last_stats())
        e2e = {"value": flops / statistics.median(ts) / 1e9, "unit": "GFLOPS",
               "h2d_bytes_per_step": int(n * n * 4), "d2h_bytes_per_step": int(2 * n * n * 4),
               "ms_per_step": statistics.median(ts) * 1e3,
               "path": "fw_solve (host buffers)" if world == 1 else
                       "pinned rows H2D + fw_dist_solve_device + D2H, per rank"}
        if hs:
            # host pipeline: chunks whose copies overlapped the solve, and the
            # exposed copy time (before the first chunk landed / after the last one computed)
            e2e["host_chunks"] = hs[-1].host_chunks
            e2e["exposed_h2d_ms"] = statistics.median(s.h2d_ms for s in hs)
            e2e["exposed_d2h_ms"] = statistics.median(s.d2h_ms for s in hs)
            e2e["library_ms"] = statistics.median(s.solve_ms for s in hs)
    if world > 1:
        fw.fw_comm_free()
    fw.fw_free()

    cpu = None
    ladder = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_sample(cfg, W=W)
        if not args.no_cpu_ladder:
            ladder = cpu_ladder()

    if rank == 0:
        line = {
            "metric": METRIC, "value": gflops, "unit": "GFLOPS", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None,
            "dtype": "i32" if is_int else "f32", "data": "synthetic",
            "config": config_json(cfg, BS, world),
            "roofline": roof,
            "cpu_baseline": cpu,
            "cpu_ladder": ladder,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "context": "paper: 338 GFLOPS on a 68-core Xeon Phi 7250 (KNL), PAPER.md P:202 (not a target)",
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C4", choices=sorted(gen.CONFIGS))
    ap.add_argument("--block", type=int, default=0)
    ap.add_argument("--n", type=int, default=0, help="the config's recipe at another n (f3: 65536)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-cpu-ladder", action="store_true", help="skip the full oracle solves at C1-C3")
    ap.add_argument("--no-isolated", action="store_true", help="skip the isolated phase-1/2 solve")
    args = ap.parse_args()
    cfg = config_for(args.config, args.n)
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_gpu(args, cfg)


if __name__ == "__main__":
    main()
