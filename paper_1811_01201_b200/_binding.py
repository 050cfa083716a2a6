"""ctypes binding for libfwb200.so: same names as include/fw.h, argument marshalling only.

Arrays may be numpy arrays (host entry points) or torch tensors (host or CUDA); raw
integer addresses are accepted too. Non-zero status codes raise FwError carrying the
code and fw_last_error().
"""
from __future__ import annotations

import ctypes
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_PKG, "libfwb200.so")

FW_INF_I32 = 0x3FFFFFFF
FW_OK, FW_EINVAL, FW_ENOMEM, FW_ECUDA, FW_ENCCL, FW_ESTATE, FW_ERANGE = range(7)
FW_PATH_NEXT_HOP, FW_PATH_LAST_K, FW_TIMING = 0, 1, 2
_NAMES = {0: "FW_OK", 1: "FW_EINVAL", 2: "FW_ENOMEM", 3: "FW_ECUDA", 4: "FW_ENCCL",
          5: "FW_ESTATE", 6: "FW_ERANGE"}


class FwError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{_NAMES.get(code, code)}: {msg}")
        self.code = code


class FwStats(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int64), ("n_pad", ctypes.c_int64), ("block", ctypes.c_int32),
        ("rounds", ctypes.c_int32), ("is_int", ctypes.c_int32), ("path_mode", ctypes.c_int32),
        ("p_method", ctypes.c_int32),
        ("solve_ms", ctypes.c_double), ("phase1_ms", ctypes.c_double),
        ("phase2_ms", ctypes.c_double), ("phase3_ms", ctypes.c_double),
        ("post_ms", ctypes.c_double), ("h2d_ms", ctypes.c_double), ("d2h_ms", ctypes.c_double),
        ("phase3_launches", ctypes.c_int64), ("phase3_relaxations", ctypes.c_double),
        ("kernel_launches", ctypes.c_int64), ("compute_f32", ctypes.c_int32),
        ("host_chunks", ctypes.c_int32), ("broadcasts", ctypes.c_int64), ("bcast_bytes", ctypes.c_double),
        ("persistent", ctypes.c_int32),
    ]

    def as_dict(self) -> dict:
        return {f: getattr(self, f) for f, _ in self._fields_}


def library_path() -> str:
    return _LIB_PATH


if not os.path.exists(_LIB_PATH):
    raise ImportError(f"{_LIB_PATH} is missing: build the CUDA extension first "
                      "(python -c 'import __graft_entry__ as g; g.build()')")

_lib = ctypes.CDLL(_LIB_PATH)
_P, _I64, _I = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
_lib.fw_init.argtypes = [_I, ctypes.c_uint]
_lib.fw_free.argtypes = []
_lib.fw_solve.argtypes = [_P, _P, _I64, _I, _I]
_lib.fw_solve_i32.argtypes = [_P, _P, _I64, _I, _I]
_lib.fw_set_host_pipeline.argtypes = [_I]
_lib.fw_set_option.argtypes = [ctypes.c_char_p, _I]
_lib.fw_host_pipeline_bounds.argtypes = [_I64, _I, _I, ctypes.POINTER(ctypes.c_int32), _I]
_lib.fw_path.argtypes = [_P, _P, _I, _I64, _I64, _I64, _I, _P, _I64]
_lib.fw_path.restype = ctypes.c_int64
_lib.fw_solve_device_f32.argtypes = [_P, _P, _I64, _I64, _I, _P]
_lib.fw_solve_device_i32.argtypes = [_P, _P, _I64, _I64, _I, _P]
_lib.fw_dist_partition.argtypes = [_I64, _I, _I, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64)]
_lib.fw_dist_owner.argtypes = [_I64, _I, _I64]
_lib.fw_comm_unique_id.argtypes = [ctypes.c_char_p]
_lib.fw_comm_init.argtypes = [ctypes.c_char_p, _I, _I]
_lib.fw_comm_free.argtypes = []
_lib.fw_dist_solve_device_f32.argtypes = [_P, _P, _I64, _I64, _I, _P]
_lib.fw_dist_solve_device_i32.argtypes = [_P, _P, _I64, _I64, _I, _P]
_lib.fw_dist_loopback_solve_device_f32.argtypes = [_P, _P, _I64, _I64, _I, _I, _P]
_lib.fw_dist_loopback_solve_device_i32.argtypes = [_P, _P, _I64, _I64, _I, _I, _P]
_lib.fw_persist_schedule.argtypes = [_I64, _I, _I, _I, _P, _I64]
_lib.fw_persist_schedule.restype = ctypes.c_int64
_lib.fw_last_error.restype = ctypes.c_char_p
_lib.fw_last_stats.argtypes = [ctypes.POINTER(FwStats)]
_lib.fw_version.restype = ctypes.c_char_p


def _check(rc: int):
    if rc != FW_OK:
        raise FwError(rc, _lib.fw_last_error().decode())


def _addr(x, dtype_name: str | None = None):
    """Address of a numpy array / torch tensor / int; None -> NULL."""
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if hasattr(x, "data_ptr"):          # torch.Tensor
        if not x.is_contiguous():
            raise ValueError("tensor must be contiguous")
        if dtype_name and str(x.dtype) != f"torch.{dtype_name}":
            raise TypeError(f"expected torch.{dtype_name}, got {x.dtype}")
        return x.data_ptr()
    if hasattr(x, "ctypes"):            # numpy.ndarray
        if not x.flags["C_CONTIGUOUS"] or not x.flags["WRITEABLE"]:
            raise ValueError("array must be C-contiguous and writeable")
        if dtype_name and x.dtype.name != dtype_name:
            raise TypeError(f"expected {dtype_name}, got {x.dtype}")
        return x.ctypes.data
    raise TypeError(f"cannot take the address of {type(x)}")


def _n_of(dist, n):
    shape = tuple(dist.shape) if hasattr(dist, "shape") else None
    if shape is not None and (len(shape) != 2 or shape[0] != shape[1]):
        raise ValueError(f"dist must be n x n, got {shape}")
    if n is None:
        if shape is None:
            raise ValueError("n is required with a raw address")
        return shape[0]
    n = int(n)
    if shape is not None and n != shape[0]:
        raise ValueError(f"n = {n} but dist is {shape[0]} x {shape[1]}")
    return n


def _is_cuda(x) -> bool:
    return bool(getattr(x, "is_cuda", False))


def _host_matrix(x, n: int, dtype_name: str, what: str):
    """Address of an n x n host matrix (numpy array or CPU tensor) of dtype_name; None -> NULL.
    Raw integer addresses are passed through unchecked (the caller vouches for them)."""
    if x is None or isinstance(x, int):
        return x
    if _is_cuda(x):
        raise ValueError(f"{what}: a CUDA tensor was passed to a host entry point "
                         "(use fw_solve_device_*)")
    if tuple(x.shape) != (n, n):
        raise ValueError(f"{what} must be {n} x {n}, got {tuple(x.shape)}")
    return _addr(x, dtype_name)


def _device_matrix(x, n: int, ld: int, dtype_name: str, what: str):
    """Address of n rows of pitch ld on the CURRENT CUDA device (torch tensor); None -> NULL.
    The tensor must hold at least n rows of ld elements (2-D: shape (>= n, ld))."""
    if x is None or isinstance(x, int):
        return x
    if not _is_cuda(x):
        raise ValueError(f"{what}: device entry points need a CUDA tensor (got a host array)")
    import torch
    if x.device.index != torch.cuda.current_device():
        raise ValueError(f"{what} is on {x.device}, the current device is cuda:{torch.cuda.current_device()}")
    shape = tuple(x.shape)
    if len(shape) != 2 or shape[1] != ld or shape[0] < n:
        raise ValueError(f"{what} must have shape (>= {n}, {ld}) for n = {n}, ld = {ld}; got {shape}")
    return _addr(x, dtype_name)


def _ld_of(x, n: int, ld):
    if ld is not None:
        ld = int(ld)
    elif hasattr(x, "shape") and len(tuple(x.shape)) == 2:
        ld = int(tuple(x.shape)[1])
    else:
        ld = n
    if ld < n:
        raise ValueError(f"ld = {ld} < n = {n}")
    return ld


def fw_init(ngpus_max: int = 0, flags: int = 0) -> None:
    _check(_lib.fw_init(ngpus_max, flags))


def fw_free() -> None:
    _check(_lib.fw_free())


def fw_solve(dist, next=None, n=None, block: int = 0, ngpus: int = 1) -> None:
    """FP32 host solve in place (dist: n x n float32; next: n x n int32 or None).
    ngpus: 1 = current device (default here), G > 1 = devices 0..G-1, 0 = fw_init's ngpus_max."""
    n = _n_of(dist, n)
    _check(_lib.fw_solve(_host_matrix(dist, n, "float32", "dist"), _host_matrix(next, n, "int32", "next"), n,
                         block, ngpus))


def fw_set_option(name: str, value: int) -> None:
    """Schedule switch of the live context: lookahead, pairs, pdl, pair_order (0/1),
    pipe_pair_rows, pipe_first (see include/fw.h)."""
    _check(_lib.fw_set_option(name.encode(), int(value)))


def fw_set_host_pipeline(chunk_tiles: int = -1) -> None:
    """Host-entry copy/solve pipeline: -1 auto, 0 off, k = chunks of k x 128 rows."""
    _check(_lib.fw_set_host_pipeline(chunk_tiles))


def fw_host_pipeline_bounds(n: int, chunk_tiles: int = -1, first_tiles: int = 8) -> list[int]:
    """Chunk boundaries (tile-rows) of the host pipeline for n (host-only); [] = not pipelined."""
    buf = (ctypes.c_int32 * 1024)()
    r = _lib.fw_host_pipeline_bounds(n, chunk_tiles, first_tiles, buf, 1024)
    if r < 0:
        _check(-r)
    return list(buf[:r])


def fw_path(P, i: int, j: int, mode: int = FW_PATH_NEXT_HOP, dist=None) -> list[int]:
    """Vertices of the shortest i -> j path encoded by P (host array from a solve; host-only).
    [] if j is unreachable from i. dist (the solve's D) is required in LAST_K mode."""
    n = _n_of(P, None)
    if _is_cuda(P) or _is_cuda(dist):
        raise ValueError("fw_path is host-only: pass host arrays")
    if dist is not None and tuple(dist.shape) != tuple(P.shape):
        raise ValueError(f"dist {tuple(dist.shape)} and P {tuple(P.shape)} differ in shape")
    d_addr = _addr(dist) if dist is not None else None
    is_int = 1 if (dist is not None and str(getattr(dist, "dtype", "")).endswith("int32")) else 0
    p_addr = _addr(P, "int32")
    r = _lib.fw_path(p_addr, d_addr, is_int, n, i, j, mode, None, 0)
    if r < 0:
        _check(int(-r))
    if r == 0:
        return []
    buf = (ctypes.c_int32 * int(r))()
    r2 = _lib.fw_path(p_addr, d_addr, is_int, n, i, j, mode, ctypes.addressof(buf), int(r))
    if r2 < 0:
        _check(int(-r2))
    return list(buf[:r2])


def fw_solve_i32(dist, next=None, n=None, block: int = 0, ngpus: int = 1) -> None:
    """INT32 host solve in place (no-edge = FW_INF_I32)."""
    n = _n_of(dist, n)
    _check(_lib.fw_solve_i32(_host_matrix(dist, n, "int32", "dist"), _host_matrix(next, n, "int32", "next"), n,
                             block, ngpus))


def _stream_handle(stream):
    if stream is None:
        return None
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream   # torch.cuda.Stream


def fw_solve_device_f32(d_dist, d_next=None, n=None, ld=None, block: int = 0, stream=None) -> None:
    """FP32 device solve in place; d_dist/d_next CUDA tensors (or device addresses)."""
    n = int(n) if n is not None else _n_of(d_dist, None)
    ld = _ld_of(d_dist, n, ld)
    _check(_lib.fw_solve_device_f32(_device_matrix(d_dist, n, ld, "float32", "d_dist"),
                                    _device_matrix(d_next, n, ld, "int32", "d_next"), n, ld, block,
                                    _stream_handle(stream)))


def fw_solve_device_i32(d_dist, d_next=None, n=None, ld=None, block: int = 0, stream=None) -> None:
    n = int(n) if n is not None else _n_of(d_dist, None)
    ld = _ld_of(d_dist, n, ld)
    _check(_lib.fw_solve_device_i32(_device_matrix(d_dist, n, ld, "int32", "d_dist"),
                                    _device_matrix(d_next, n, ld, "int32", "d_next"), n, ld, block,
                                    _stream_handle(stream)))


def fw_dist_partition(n: int, world: int, rank: int) -> tuple[int, int]:
    """(row0, nrows): the rows of the n x n matrix rank `rank` of `world` holds (host-only)."""
    r0, nr = ctypes.c_int64(), ctypes.c_int64()
    _check(_lib.fw_dist_partition(n, world, rank, ctypes.byref(r0), ctypes.byref(nr)))
    return r0.value, nr.value


def fw_dist_owner(n: int, world: int, row: int) -> int:
    return _lib.fw_dist_owner(n, world, row)


def fw_comm_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(_lib.fw_comm_unique_id(buf))
    return buf.raw


def fw_comm_init(uid: bytes, rank: int, world: int) -> None:
    if len(uid) != 128:
        raise ValueError("NCCL unique id must be 128 bytes")
    _check(_lib.fw_comm_init(uid, rank, world))


def fw_comm_free() -> None:
    _check(_lib.fw_comm_free())


def fw_dist_solve_device_f32(d_rows, d_next_rows=None, n=None, ld=None, block: int = 0, stream=None) -> None:
    """Collective FP32 solve of this rank's rows (see fw_dist_partition)."""
    if n is None:
        raise ValueError("n (global vertex count) is required")
    n = int(n)
    ld = _ld_of(d_rows, n, ld)
    rows = d_rows.shape[0] if hasattr(d_rows, "shape") else 0
    if d_next_rows is not None and hasattr(d_next_rows, "shape") and hasattr(d_rows, "shape") \
            and tuple(d_next_rows.shape) != tuple(d_rows.shape):
        raise ValueError(f"d_next_rows {tuple(d_next_rows.shape)} != d_rows {tuple(d_rows.shape)}")
    _check(_lib.fw_dist_solve_device_f32(_device_matrix(d_rows, rows, ld, "float32", "d_rows"),
                                         _device_matrix(d_next_rows, rows, ld, "int32", "d_next_rows"), n, ld,
                                         block, _stream_handle(stream)))


def fw_dist_solve_device_i32(d_rows, d_next_rows=None, n=None, ld=None, block: int = 0, stream=None) -> None:
    if n is None:
        raise ValueError("n (global vertex count) is required")
    n = int(n)
    ld = _ld_of(d_rows, n, ld)
    rows = d_rows.shape[0] if hasattr(d_rows, "shape") else 0
    if d_next_rows is not None and hasattr(d_next_rows, "shape") and hasattr(d_rows, "shape") \
            and tuple(d_next_rows.shape) != tuple(d_rows.shape):
        raise ValueError(f"d_next_rows {tuple(d_next_rows.shape)} != d_rows {tuple(d_rows.shape)}")
    _check(_lib.fw_dist_solve_device_i32(_device_matrix(d_rows, rows, ld, "int32", "d_rows"),
                                         _device_matrix(d_next_rows, rows, ld, "int32", "d_next_rows"), n, ld,
                                         block, _stream_handle(stream)))


def fw_dist_loopback_solve_device_f32(d_dist, d_next=None, n=None, ld=None, block: int = 0, world: int = 2,
                                      stream=None) -> None:
    """Every rank of a `world`-way partition emulated on this GPU (testing transport)."""
    n = int(n) if n is not None else _n_of(d_dist, None)
    ld = _ld_of(d_dist, n, ld)
    _check(_lib.fw_dist_loopback_solve_device_f32(_device_matrix(d_dist, n, ld, "float32", "d_dist"),
                                                  _device_matrix(d_next, n, ld, "int32", "d_next"), n, ld,
                                                  block, world, _stream_handle(stream)))


def fw_dist_loopback_solve_device_i32(d_dist, d_next=None, n=None, ld=None, block: int = 0, world: int = 2,
                                      stream=None) -> None:
    n = int(n) if n is not None else _n_of(d_dist, None)
    ld = _ld_of(d_dist, n, ld)
    _check(_lib.fw_dist_loopback_solve_device_i32(_device_matrix(d_dist, n, ld, "int32", "d_dist"),
                                                  _device_matrix(d_next, n, ld, "int32", "d_next"), n, ld,
                                                  block, world, _stream_handle(stream)))


def fw_persist_schedule(n: int, world: int = 1, rank: int = -1, gap: int = 0):
    """Work-item order of the persistent solve (host-only): a numpy uint32 array of packed
    items (rank << 29 | type << 27 | K << 18 | I << 9 | J)."""
    import numpy as np
    cnt = _lib.fw_persist_schedule(n, world, rank, gap, None, 0)
    if cnt < 0:
        _check(int(-cnt))
    out = np.empty(int(cnt), dtype=np.uint32)
    r = _lib.fw_persist_schedule(n, world, rank, gap, out.ctypes.data, int(cnt))
    if r < 0:
        _check(int(-r))
    return out


def fw_last_error() -> str:
    return _lib.fw_last_error().decode()


def fw_last_stats() -> FwStats:
    s = FwStats()
    _check(_lib.fw_last_stats(ctypes.byref(s)))
    return s


def fw_version() -> str:
    return _lib.fw_version().decode()
