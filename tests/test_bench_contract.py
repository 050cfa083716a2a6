"""bench.py keeps the driver's JSON-line contract: the reference arm (the CPU oracle, no GPU)
on CPU, our arm on the GPU (small config so both finish in seconds)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_bench(*args, timeout=600):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_reference_arm_line():
    d = run_bench("--impl", "reference", "--config", "C1", "--steps", "1", "--warmup", "1")
    assert d["impl"] == "reference" and d["unit"] == "GFLOPS" and d["value"] > 0
    assert d["higher_is_better"] is True and d["n_gpus"] == 1
    assert d["config"]["workload"] and d["config"]["n"] == 512
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


@pytest.mark.gpu
def test_our_arm_line():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    d = run_bench("--config", "C1", "--steps", "3", "--warmup", "3", "--no-cpu")
    assert d["metric"].startswith("APSP GFLOPS") and d["value"] > 0 and d["unit"] == "GFLOPS"
    assert d["steps"] == 3 and d["warmup"] == 3 and d["ms_per_step"] > 0
    assert d["dtype"] == "f32" and d["data"] == "synthetic" and d["config"]["workload"]
    roof = d["roofline"]
    assert roof["bound"] == "alu" and roof["achieved"] > 0 and roof["peak"] > 0
    assert abs(roof["frac"] - roof["achieved"] / roof["peak"]) < 1e-9
    e2e = d["e2e"]
    assert e2e["value"] > 0 and e2e["h2d_bytes_per_step"] == 512 * 512 * 4
    assert e2e["d2h_bytes_per_step"] == 2 * 512 * 512 * 4
    assert d["gpu_launches"] > 0 and "clocks" in d and "reasons" in d["clocks"]
