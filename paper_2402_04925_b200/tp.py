"""torch.distributed plumbing for the TP path (one process per GPU): exchange the NCCL
unique id over the launcher's process group, then build the library-owned communicator.

The collectives themselves (AllReduce PAPER.md:L142, AllGather L117) run inside libtpq.so
on that communicator; torch.distributed is only the bootstrap channel (gloo or nccl).
"""
from __future__ import annotations

from . import _lib


def exchange_unique_id(group=None) -> bytes:
    """Rank 0 draws an ncclUniqueId (tpq_comm_unique_id); every rank returns the same 128 B."""
    import torch
    import torch.distributed as dist

    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    buf = torch.zeros(128, dtype=torch.uint8, device=dev)
    if dist.get_rank(group) == 0:
        buf.copy_(torch.frombuffer(bytearray(_lib.comm_unique_id()), dtype=torch.uint8))
    dist.broadcast(buf, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
    return bytes(buf.cpu().numpy().tobytes())


def make_comm(device: int, group=None) -> "_lib.Comm":
    """Collective: the TP communicator of this rank (tp = world size of `group`)."""
    import torch.distributed as dist

    uid = exchange_unique_id(group)
    return _lib.Comm(uid, dist.get_world_size(group), dist.get_rank(group), device)
