"""Multi-process (one rank per GPU) set-up of the d >= 2 slab path.

torch.distributed is plumbing only: it carries the 128-byte NCCL unique id from rank 0 to
every rank; the library then owns the NCCL communicator and exchanges halo rows with
ncclSend/ncclRecv inside bsde_step.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from .bsde import Solver, nccl_unique_id


def broadcast_id(id_bytes: bytes | None, rank: int, src: int = 0) -> bytes:
    """Broadcast 128 bytes from `src` with torch.distributed (any backend)."""
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.zeros(128, dtype=torch.uint8, device=dev)
    if rank == src:
        t.copy_(torch.frombuffer(bytearray(id_bytes), dtype=torch.uint8))
    dist.broadcast(t, src)
    return bytes(t.cpu().tolist())


def make_slab_solver(spec: dict, device: int | None = None, **kw) -> Solver:
    """The calling rank's slab of a d >= 2 problem over all ranks of the default group."""
    rank, world = dist.get_rank(), dist.get_world_size()
    if device is None:
        device = torch.cuda.current_device()
    nid = broadcast_id(nccl_unique_id() if rank == 0 else None, rank)
    return Solver(spec, device=device, nranks=world, rank=rank, nccl_id=nid, **kw)
