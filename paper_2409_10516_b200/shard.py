"""Multi-GPU sharding of the decode step (SURVEY §8 e).

Unit of work = one KV group: its K/V plus the graphs and queries of its
query heads (engine.cpp runs heads independently, :105-115; PAPER.md: one
index per query head). Ranks own contiguous ranges of groups, so search and
attention need no exchange. The only collective is gathering the per-head
outputs after each step (an all_gather over NCCL on GPUs, gloo on CPU in
tests); uneven shards are padded to the largest shard.
"""
from __future__ import annotations

from typing import List

import torch


def groups_for_rank(n_groups: int, world: int, rank: int) -> List[int]:
    """Contiguous, balanced split of KV groups over ranks (sizes differ by <= 1)."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    return list(range(rank * n_groups // world, (rank + 1) * n_groups // world))


def heads_for_groups(groups: List[int], heads_per_group: int) -> List[int]:
    """Query heads of the given groups (head h belongs to group h // hpg)."""
    return [g * heads_per_group + m for g in groups for m in range(heads_per_group)]


def max_local_heads(n_groups: int, world: int, heads_per_group: int) -> int:
    return max(len(groups_for_rank(n_groups, world, r)) for r in range(world)) * heads_per_group


class OutputGather:
    """all_gather of per-head decode outputs [H_local, d] -> [H, d] in global
    head order on every rank. Buffers are allocated once (no per-step
    allocation on the hot path)."""

    def __init__(self, n_groups: int, heads_per_group: int, d: int, world: int, rank: int,
                 device, dtype=torch.float64):
        self.world, self.rank = world, rank
        self.hpg, self.G, self.d = heads_per_group, n_groups, d
        self.width = max_local_heads(n_groups, world, heads_per_group)
        self.send = torch.zeros((self.width, d), dtype=dtype, device=device)
        self.recv = [torch.zeros((self.width, d), dtype=dtype, device=device)
                     for _ in range(world)]
        self.counts = [len(groups_for_rank(n_groups, world, r)) * heads_per_group
                       for r in range(world)]
        self.out = torch.zeros((n_groups * heads_per_group, d), dtype=dtype, device=device)

    def __call__(self, local: torch.Tensor, dist) -> torch.Tensor:
        n = local.shape[0]
        self.send[:n].copy_(local)
        if self.world == 1:
            self.out.copy_(self.send[:n])
            return self.out
        dist.all_gather(self.recv, self.send)
        off = 0
        for r in range(self.world):
            c = self.counts[r]
            self.out[off:off + c].copy_(self.recv[r][:c])
            off += c
        return self.out
