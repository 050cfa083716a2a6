import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run via gpurun)")
    config.addinivalue_line("markers", "slow: long-running")


GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load_golden(name):
    """Parse a tests/golden/*.txt fixture: 'n N' then sections W, D, LASTK, NEXT."""
    import numpy as np
    sections = {}
    n = None
    cur = None
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            if line.startswith("n "):
                n = int(line.split()[1])
                continue
            if line in ("W", "D", "LASTK", "NEXT"):
                cur = line
                sections[cur] = []
                continue
            sections[cur].append([float(x) for x in line.split()])
    out = {"n": n}
    for k, rows in sections.items():
        a = np.array(rows, dtype=np.float64)
        assert a.shape == (n, n), (name, k, a.shape)
        out[k] = a.astype(np.int32) if k in ("LASTK", "NEXT") else a
    return out


def golden_names():
    return sorted(f for f in os.listdir(GOLDEN) if f.endswith(".txt"))
