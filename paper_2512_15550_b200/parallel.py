"""Multi-GPU partition of the decode path.

Every stage is independent per (b, kv head) unit once a KV head's gs query
heads, its centroid rows and its lists are co-located (ck/retrieval.py:144-
145, ck/index.py:46, ck/retrieval.py:181-186), so units are partitioned
over ranks as kv-head shards x batch shards and the only data exchanged is
one all-gather of the head-sharded attention outputs per layer (north_star).
The FIFO cursor (per batch element, ck/index.py:121,133) is replicated on
every rank that holds a shard of that batch element; it advances
deterministically (total recall > 0), so replicas never diverge in
non-error runs.  Index and KV never move.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import torch


@dataclass(frozen=True)
class ShardPlan:
    world: int
    rank: int
    batch: int        # global batch B
    kv_heads: int     # global G
    query_heads: int  # global H

    def __post_init__(self):
        if self.world < 1 or not 0 <= self.rank < self.world:
            raise ValueError(f"bad rank {self.rank} of {self.world}")
        if self.batch % self.batch_shards or self.kv_heads % self.head_shards:
            raise ValueError(f"batch {self.batch} x kv_heads {self.kv_heads} cannot be split "
                             f"{self.batch_shards} x {self.head_shards} ways")

    @property
    def head_shards(self) -> int:
        """kv heads split as evenly as the world allows (gcd), batch takes the rest."""
        return math.gcd(self.world, self.kv_heads)

    @property
    def batch_shards(self) -> int:
        return self.world // self.head_shards

    @property
    def head_rank(self) -> int:
        return self.rank % self.head_shards

    @property
    def batch_rank(self) -> int:
        return self.rank // self.head_shards

    @property
    def b_loc(self) -> int:
        return self.batch // self.batch_shards

    @property
    def g_loc(self) -> int:
        return self.kv_heads // self.head_shards

    @property
    def h_loc(self) -> int:
        return self.g_loc * (self.query_heads // self.kv_heads)

    def batch_range(self, rank: int | None = None) -> tuple[int, int]:
        r = self.rank if rank is None else rank
        b0 = (r // self.head_shards) * self.b_loc
        return b0, b0 + self.b_loc

    def kv_range(self, rank: int | None = None) -> tuple[int, int]:
        r = self.rank if rank is None else rank
        g0 = (r % self.head_shards) * self.g_loc
        return g0, g0 + self.g_loc

    def q_range(self, rank: int | None = None) -> tuple[int, int]:
        g0, g1 = self.kv_range(rank)
        gs = self.query_heads // self.kv_heads
        return g0 * gs, g1 * gs

    def assemble(self, gathered: torch.Tensor) -> torch.Tensor:
        """[world, b_loc, h_loc, d] (rank-major all-gather) -> [B, H, d]."""
        w, bl, hl, d = gathered.shape
        out = gathered.new_empty((self.batch, self.query_heads, d))
        for r in range(w):
            b0, b1 = self.batch_range(r)
            h0, h1 = self.q_range(r)
            out[b0:b1, h0:h1] = gathered[r]
        return out


def all_gather_outputs(plan: ShardPlan, local: torch.Tensor, group=None,
                       buf: torch.Tensor | None = None) -> torch.Tensor:
    """One collective per layer: all-gather the local [b_loc, h_loc, d]
    attention output and reassemble [B, H, d] on every rank."""
    import torch.distributed as dist
    if plan.world == 1:
        return local
    if buf is None:
        buf = local.new_empty((plan.world,) + tuple(local.shape))
    # output passed as [world * b_loc, h_loc, d] (rank-major concat): the
    # form both NCCL and gloo accept
    dist.all_gather_into_tensor(buf.view((-1,) + tuple(local.shape[1:])), local.contiguous(),
                                group=group)
    return plan.assemble(buf)


def gather_lane_outputs(plan: ShardPlan, local: torch.Tensor, buf: torch.Tensor,
                        out: torch.Tensor, lane_b0: int, group=None) -> None:
    """The engine's per-(layer, lane) collective: all-gather one lane's
    local output slice `local` [bl, h_loc, d] (sequences lane_b0 ..
    lane_b0+bl of every rank's batch shard) through `buf` [world, bl, h_loc,
    d] and place each rank's part into the global `out` [B, H, d] view.
    Every rank issues it with the same (layer, lane) order, so the
    collectives match."""
    import torch.distributed as dist
    bl = local.shape[0]
    dist.all_gather_into_tensor(buf.view((-1,) + tuple(local.shape[1:])), local, group=group)
    for r in range(plan.world):
        b0 = plan.batch_range(r)[0] + lane_b0
        h0, h1 = plan.q_range(r)
        out[b0:b0 + bl, h0:h1].copy_(buf[r])
