"""One-off fuzz run (development): many seeded cases of tests/test_gpu_fuzz.py's generator."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import test_gpu_fuzz as tf


class MP:
    def setenv(self, k, v):
        os.environ[k] = v


seed = int(sys.argv[1]) if len(sys.argv) > 1 else 1
count = int(sys.argv[2]) if len(sys.argv) > 2 else 100
rng = np.random.default_rng(seed)
fails = 0
for step in range(count):
    try:
        tf.one_case(rng, step, MP())
    except Exception as e:   # report and continue
        fails += 1
        print("FAIL", step, repr(e)[:400], flush=True)
print("done", count, "fails", fails, flush=True)
