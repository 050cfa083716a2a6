"""B200-native blocked Floyd–Warshall APSP (arxiv 1811.01201), Python binding.

Thin ctypes marshalling over ``libfwb200.so`` whose C ABI is ``include/fw.h``; every
step of the solve runs in the library's CUDA kernels. There is no CPU fallback: if the
extension is missing, importing this package raises.
"""
from ._binding import (  # noqa: F401
    FW_INF_I32,
    FW_OK, FW_EINVAL, FW_ENOMEM, FW_ECUDA, FW_ENCCL, FW_ESTATE, FW_ERANGE,
    FW_PATH_NEXT_HOP, FW_PATH_LAST_K, FW_TIMING,
    FwError,
    FwStats,
    fw_init,
    fw_free,
    fw_solve,
    fw_solve_i32,
    fw_set_host_pipeline,
    fw_set_option,
    fw_host_pipeline_bounds,
    fw_path,
    fw_solve_device_f32,
    fw_solve_device_i32,
    fw_last_error,
    fw_dist_partition,
    fw_dist_owner,
    fw_comm_unique_id,
    fw_comm_init,
    fw_comm_free,
    fw_dist_solve_device_f32,
    fw_dist_solve_device_i32,
    fw_dist_loopback_solve_device_f32,
    fw_dist_loopback_solve_device_i32,
    fw_last_stats,
    fw_persist_schedule,
    fw_version,
    library_path,
)

__all__ = [n for n in dir() if n.startswith("fw") or n.startswith("FW") or n in ("FwError", "FwStats")]
