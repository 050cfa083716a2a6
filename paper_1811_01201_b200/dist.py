"""Multi-GPU plumbing: one process per GPU, torch.distributed for rendezvous only.

The round loop, the pivot-strip broadcast (NCCL) and every kernel run inside libfwb200
(``fw_dist_solve_device_*``); torch.distributed only ships the 128-byte NCCL unique id from
rank 0 to the other ranks (SURVEY §8 e, BASELINE north_star "block-row partition ... NCCL
broadcast").
"""
from __future__ import annotations

from . import _binding as fw


def comm_init_from_torch(group=None) -> tuple[int, int]:
    """Create the library's NCCL communicator over the ranks of a torch process group."""
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    obj = [fw.fw_comm_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    fw.fw_comm_init(obj[0], rank, world)
    return rank, world


def local_rows(n: int, rank: int, world: int) -> tuple[int, int]:
    """Rows [row0, row0 + nrows) of the n x n problem held by `rank` (same as the C partition)."""
    return fw.fw_dist_partition(n, world, rank)
