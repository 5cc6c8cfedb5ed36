"""Process-group plumbing for the sharded path (S9/S10): torch.distributed only carries the
NCCL unique id and the per-rank row ranges; every data-path collective runs inside libcsk
(NCCL).  Works with either torch backend (gloo on CPU for tests, nccl on GPUs)."""
from __future__ import annotations

import torch
import torch.distributed as dist


def broadcast_uid(uid: bytes | None, group=None, device="cpu") -> bytes:
    """Broadcast rank 0's 128-byte NCCL unique id to every rank of `group`."""
    buf = torch.zeros(128, dtype=torch.uint8, device=device)
    if dist.get_rank(group) == 0:
        buf.copy_(torch.frombuffer(bytearray(uid), dtype=torch.uint8))
    dist.broadcast(buf, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
    return bytes(buf.cpu().tolist())


def row_shard(m: int, nranks: int, rank: int) -> tuple[int, int]:
    """Contiguous input-row shard [lo, hi) of A for `rank` (balanced; any split is valid since
    rows are hashed with their global index)."""
    return m * rank // nranks, m * (rank + 1) // nranks


def init_comm(ctx=None, group=None):
    """Create the library's NCCL communicator on every rank of `group` (call collectively)."""
    import paper_2004_02480_b200 as csk
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    uid = csk.comm_unique_id() if rank == 0 else None
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else "cpu"
    uid = broadcast_uid(uid, group, dev)
    csk.comm_create(uid, world, rank, ctx)
    return rank, world
