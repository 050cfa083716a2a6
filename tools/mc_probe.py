"""Probe: does this GPU support switch multicast (NVLS) / fabric handles? (dev tool)"""
import ctypes
cu = ctypes.CDLL("libcuda.so.1")
assert cu.cuInit(0) == 0
dev = ctypes.c_int()
cu.cuDeviceGet(ctypes.byref(dev), 0)
for name, attr in [("MULTICAST_SUPPORTED", 132), ("HANDLE_TYPE_FABRIC_SUPPORTED", 128),
                   ("IPC_EVENT_SUPPORTED", 125)]:
    v = ctypes.c_int(-1)
    rc = cu.cuDeviceGetAttribute(ctypes.byref(v), attr, dev)
    print(name, rc, v.value)
