"""Bootstrap of the row-block distributed plan (§3.1) over torch.distributed.

One process per GPU.  torch.distributed only carries the 128-byte NCCL unique id; the per-sweep
exchange (allgather of x + max-allreduce of d_k) runs inside libjacobi.so's CUDA graphs on NCCL.
"""
from __future__ import annotations

from . import Plan, nccl_unique_id, partition


def bootstrap(n: int):
    """Returns (uid, rank, world, row0, rows).  Every rank raises the same JacobiError
    (EINDIVISIBLE) when the world size does not divide n, before any NCCL/CUDA work."""
    import torch.distributed as dist
    rank, world = dist.get_rank(), dist.get_world_size()
    row0, rows = partition(n, world, rank)
    obj = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0], rank, world, row0, rows


def dist_plan(A_rows, n: int, stream=None) -> Plan:
    """Distributed plan over this rank's row block A_rows (torch CUDA tensor, borrowed, or numpy)."""
    uid, rank, world, row0, rows = bootstrap(n)
    if A_rows.shape[0] != rows:
        raise ValueError(f"rank {rank} must pass rows [{row0}, {row0 + rows}) ({rows} rows), got {A_rows.shape[0]}")
    return Plan(A_rows, n=n, stream=stream, dist=(uid, rank, world))
