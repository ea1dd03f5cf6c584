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


def dist_plan(A_block, n: int, stream=None, layout: str = "rows", p2p: bool = False) -> Plan:
    """Distributed plan over this rank's block (torch CUDA tensor, borrowed, or numpy): its row block
    (layout="rows", §3.1) or its n x m column slab (layout="cols", §3.2).  p2p=True switches
    a row-wise plan to the fused NVLink exchange (NEXT-1): the CUDA IPC handles of every rank's x
    buffers, slots and counters are all-gathered through torch.distributed and mapped."""
    import torch.distributed as dist
    uid, rank, world, row0, rows = bootstrap(n)
    want = rows if layout == "rows" else n
    if A_block.shape[0] != want:
        raise ValueError(f"rank {rank}: expected {want} rows in its {layout} block, got {A_block.shape[0]}")
    plan = Plan(A_block, n=n, stream=stream, dist=(uid, rank, world), layout=layout)
    if p2p:
        mine = plan.ipc_export()
        allh = [None] * world
        dist.all_gather_object(allh, mine)
        plan.ipc_attach(b"".join(allh))
    return plan
