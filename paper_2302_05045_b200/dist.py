"""Data-parallel plumbing: communicator rendezvous over torch.distributed.

The gradient exchange itself runs inside libsamo_cuda.so (NCCL on the
compressed fp32 gradient arena, bucketed and overlapped with the step
kernels).  torch.distributed only carries the 128-byte NCCL unique id from
rank 0 to the other ranks (gloo or nccl process groups both work) and the
barrier / max-over-ranks timing of the bench.

Data-parallel semantics: every rank holds the full compressed
state; rank r's dense gradients come from its own batch shard; the step sums
the compressed fp32 gradients of all ranks with 1/G folded into the unscale
(exact for power-of-two G) and skips — on every rank — when any rank saw a
non-finite gradient.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from .samo import Communicator


def broadcast_unique_id(group=None) -> bytes:
    """Rank 0 creates the NCCL unique id; every rank returns the same bytes."""
    rank = dist.get_rank(group)
    backend = dist.get_backend(group)
    device = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    buf = torch.zeros(128, dtype=torch.uint8, device=device)
    if rank == 0:
        buf.copy_(torch.tensor(list(Communicator.unique_id()), dtype=torch.uint8))
    dist.broadcast(buf, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
    return bytes(buf.cpu().tolist())


def make_communicator(group=None) -> Communicator:
    """Collective: one NCCL communicator per rank for the gradient exchange."""
    uid = broadcast_unique_id(group)
    return Communicator(uid, dist.get_world_size(group), dist.get_rank(group))


def rank_seed(seed: int, rank: int) -> int:
    """Seed of rank r's synthetic gradient stream (distinct batch shards)."""
    return seed + 1 + rank
