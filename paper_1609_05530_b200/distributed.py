"""Multi-GPU plumbing for fit_parallel.

The paper's method is communication-free across subsets (PAPER.md:118-128,
SPEC.md:307): GPU g owns the contiguous block range shard_blocks(K, G, g),
samples / ranks / fits / computes variances for it with no exchange, and the
ONLY collective is one all-gather of the fixed-size per-block records
(pcb_fit_result, 48 B each) before the combine, which every rank then runs
in block order on device — so theta_combined is bitwise identical for any G.
One process per GPU; torch.distributed (NCCL on GPUs, gloo in CPU tests) is
the transport.
"""
from __future__ import annotations

from typing import Tuple

RECORD_WORDS = 6  # sizeof(pcb_fit_result) / 8


def shard_blocks(k_total: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous block range [first, last) of `rank` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    q, r = divmod(k_total, world)
    first = rank * q + min(rank, r)
    return first, first + q + (1 if rank < r else 0)


def gather_records(local, k_total: int, group=None):
    """All-gather the per-block records of every rank, in block order.

    `local`: int64 tensor [k_local, 6] holding the raw bytes of k_local
    pcb_fit_result records (bit-preserving view). Returns [k_total, 6] on
    the same device. Ranks hold contiguous block ranges (shard_blocks), so
    concatenation in rank order is block order.
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    kmax = -(-k_total // world)
    pad = torch.zeros((kmax, RECORD_WORDS), dtype=torch.int64, device=local.device)
    pad[: local.shape[0]] = local
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    out = []
    for r in range(world):
        a, b = shard_blocks(k_total, world, r)
        out.append(parts[r][: b - a])
    return torch.cat(out, 0)
