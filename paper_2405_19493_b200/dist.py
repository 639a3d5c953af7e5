"""Multi-GPU plumbing: streams shard by id across ranks; the generation path
has no collective.  Only the final witnesses of config 4 are exchanged:
per-rank central moments (n, mean, M2, M3, M4) and the per-rank xor of the
per-stream checksums, gathered with one all_gather each (NCCL over NVLink on
the GPU box, gloo in the CPU tests) and merged in rank order, so the result
does not depend on arrival order.  XOR is not an NCCL reduction op, hence the
gather-and-fold.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from .streams import merge_central

MASK64 = (1 << 64) - 1


def shard(total: int, world: int, rank: int):
    """Contiguous block of stream ids [first, first + count) owned by `rank`."""
    base, extra = divmod(total, world)
    first = rank * base + min(rank, extra)
    return first, base + (1 if rank < extra else 0)


def _device():
    return torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" else torch.device("cpu")


def gather_moments(central5) -> tuple:
    """Merge every rank's (n, mean, M2, M3, M4) (Pebay/Chan, in rank order)."""
    world = dist.get_world_size()
    t = torch.as_tensor(list(central5) if not torch.is_tensor(central5) else central5.tolist(),
                        dtype=torch.float64, device=_device())
    parts = [torch.zeros(5, dtype=torch.float64, device=t.device) for _ in range(world)]
    dist.all_gather(parts, t)
    return merge_central([tuple(p.cpu().tolist()) for p in parts])


def gather_xor(x: int) -> int:
    """xor of one 64-bit value per rank."""
    world = dist.get_world_size()
    v = x & MASK64
    t = torch.tensor([v - (1 << 64) if v >= (1 << 63) else v], dtype=torch.int64, device=_device())
    parts = [torch.zeros(1, dtype=torch.int64, device=t.device) for _ in range(world)]
    dist.all_gather(parts, t)
    acc = 0
    for p in parts:
        acc ^= int(p.item()) & MASK64
    return acc
