"""Probe: cost of cudaHostRegister / Unregister on pageable numpy buffers (1-3 GiB), and the
H2D bandwidth from registered vs pinned vs pageable memory."""
import time
import numpy as np
import torch

cudart = torch.cuda.cudart()
torch.cuda.init()
for gib in (1, 2):
    a = np.ones((gib << 28,), dtype=np.float32)           # touched (page-faulted in)
    t0 = time.perf_counter()
    r = cudart.cudaHostRegister(a.ctypes.data, a.nbytes, 0)
    t1 = time.perf_counter()
    d = torch.empty(a.shape, dtype=torch.float32, device="cuda")
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    d.copy_(torch.from_numpy(a), non_blocking=True)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    r2 = cudart.cudaHostUnregister(a.ctypes.data)
    t4 = time.perf_counter()
    b = np.ones((gib << 28,), dtype=np.float32)
    torch.cuda.synchronize()
    t5 = time.perf_counter()
    d.copy_(torch.from_numpy(b))
    torch.cuda.synchronize()
    t6 = time.perf_counter()
    print(f"{gib} GiB: register {1e3*(t1-t0):.1f} ms (rc {r}), H2D registered {1e3*(t3-t2):.1f} ms, "
          f"unregister {1e3*(t4-t3):.1f} ms (rc {r2}), H2D pageable {1e3*(t6-t5):.1f} ms", flush=True)
