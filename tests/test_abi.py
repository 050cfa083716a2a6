"""CPU-side checks of the C ABI boundary: the library loads, exports every symbol that
include/fw.h declares, and the host-side error contract that needs no GPU."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "fw.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fw_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for f in ("fw_init", "fw_free", "fw_solve", "fw_solve_i32", "fw_solve_device_f32",
              "fw_solve_device_i32", "fw_last_error", "fw_last_stats"):
        assert f in names


def test_library_exports_every_declared_symbol():
    import paper_1811_01201_b200 as fw
    lib = ctypes.CDLL(fw.library_path())
    missing = [f for f in declared_functions() if not hasattr(lib, f)]
    assert not missing, missing


def test_binding_has_same_names():
    import paper_1811_01201_b200 as fw
    for f in declared_functions():
        assert hasattr(fw, f), f


def test_no_oracle_in_product():
    """The product package never imports or links the oracle (task rule ③)."""
    pkg = os.path.join(ROOT, "paper_1811_01201_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "liboracle" not in txt and "fw_oracle" not in txt, f


def test_state_errors_without_init():
    import paper_1811_01201_b200 as fw
    with pytest.raises(fw.FwError) as e:
        fw.fw_solve(np.zeros((3, 3), np.float32))
    assert e.value.code == fw.FW_ESTATE
    with pytest.raises(fw.FwError) as e:
        fw.fw_last_stats()
    assert e.value.code == fw.FW_ESTATE
    fw.fw_free()   # idempotent
    assert fw.fw_version().startswith("fwb200")


def test_init_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_1811_01201_b200 as fw
    with pytest.raises(fw.FwError) as e:
        fw.fw_init()
    assert e.value.code == fw.FW_ECUDA


def test_binding_marshalling_errors():
    import paper_1811_01201_b200 as fw
    with pytest.raises(TypeError):
        fw.fw_solve(np.zeros((3, 3), np.float64))
    with pytest.raises(ValueError):
        fw.fw_solve(np.zeros((3, 4), np.float32))
    with pytest.raises(ValueError):
        fw.fw_solve(np.zeros((4, 4), np.float32)[:, ::2].T)


def test_binding_shape_and_device_checks():
    """the binding rejects mismatched shapes and host/device mix-ups before any
    pointer reaches the library (an overrun or a device pointer dereferenced on the host)."""
    import torch
    import paper_1811_01201_b200 as fw
    D = np.zeros((4, 4), np.float32)
    with pytest.raises(ValueError):
        fw.fw_solve(D, np.zeros((3, 3), np.int32))           # next smaller than dist
    with pytest.raises(ValueError):
        fw.fw_solve(D, None, n=8)                            # explicit n beyond the array
    with pytest.raises(ValueError):
        fw.fw_solve_i32(np.zeros((4, 4), np.int32), np.zeros((4, 5), np.int32))
    with pytest.raises(ValueError):                          # host tensor on a device entry
        fw.fw_solve_device_f32(torch.zeros((4, 4)), None)
    with pytest.raises(ValueError):
        fw.fw_dist_loopback_solve_device_i32(torch.zeros((4, 4), dtype=torch.int32), None)
    with pytest.raises(ValueError):
        fw.fw_dist_solve_device_f32(torch.zeros((4, 4)), None, n=4)
    with pytest.raises(ValueError):                          # fw_path: D and P shapes differ
        fw.fw_path(np.zeros((4, 4), np.int32), 0, 1, dist=np.zeros((3, 3), np.float32))
