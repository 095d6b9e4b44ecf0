"""Multi-GPU sharding of the decode path by (sequence, KV head) units.

Every (sequence b, KV head g) pair is an independent unit of work: its
G = Hq/Hkv query-head sessions read only that KV head's K/V rows and their
own proxy rows, B factors and fast-tier sets (ref: SPEC.md:222,
PAPER.md:309, README.md:140-142 -- sessions are independent per head).  A
rank therefore owns a rectangle of units -- a block of whole sequences, or
a block of KV heads of one sequence when there are more ranks than
sequences -- and runs the unchanged single-GPU engine on it.  Nothing is
exchanged inside the step; the only collectives are

  * one all-gather of the per-head attention outputs at the end of a step
    (`gather_outputs`), and
  * one all-reduce of the int64 hit/miss counters when they are read
    (`reduce_counters`, ref: cache.py:63-81 summed over sessions).

Both go through `torch.distributed` (NCCL over NVLink on the B200 box, gloo
in the CPU tests).
"""

from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist


@dataclass(frozen=True)
class Shard:
    """Rank-local block of units: sequences [b0, b1) x KV heads [g0, g1)."""

    rank: int
    b0: int
    b1: int
    g0: int
    g1: int
    group: int  # query heads per KV head

    @property
    def batch(self) -> int:
        return self.b1 - self.b0

    @property
    def n_kv_heads(self) -> int:
        return self.g1 - self.g0

    @property
    def n_q_heads(self) -> int:
        return self.n_kv_heads * self.group

    @property
    def q0(self) -> int:
        return self.g0 * self.group

    @property
    def q1(self) -> int:
        return self.g1 * self.group

    def units(self):
        return [(b, g) for b in range(self.b0, self.b1) for g in range(self.g0, self.g1)]


def plan_shards(batch: int, n_q_heads: int, n_kv_heads: int, world: int) -> list[Shard]:
    """Batch-major contiguous equal blocks of the B x Hkv unit grid.

    Whole sequences per rank when world divides batch; otherwise each
    sequence is split over world/batch ranks by contiguous KV-head blocks
    (SURVEY.md §8e).  Equal blocks keep the all-gather a single
    fixed-shape collective.  Raises ValueError for grids that cannot be
    split into equal rectangles.
    """
    if world < 1 or batch < 1 or n_kv_heads < 1 or n_q_heads % n_kv_heads:
        raise ValueError(f"bad shape: batch={batch} Hq={n_q_heads} Hkv={n_kv_heads} world={world}")
    G = n_q_heads // n_kv_heads
    if batch % world == 0:
        per = batch // world
        return [Shard(r, r * per, (r + 1) * per, 0, n_kv_heads, G) for r in range(world)]
    if world % batch == 0 and n_kv_heads % (world // batch) == 0:
        split = world // batch
        gk = n_kv_heads // split
        return [Shard(r, r // split, r // split + 1, (r % split) * gk, (r % split + 1) * gk, G)
                for r in range(world)]
    raise ValueError(f"cannot split {batch} sequences x {n_kv_heads} KV heads into {world} equal blocks")


def local_slice(x: torch.Tensor, shard: Shard, *, heads: str, batch_dim: int = -3) -> torch.Tensor:
    """This rank's block of a [..., B, H, d] tensor (heads='q' or 'kv')."""
    bd = batch_dim % x.dim()
    h0, h1 = (shard.q0, shard.q1) if heads == "q" else (shard.g0, shard.g1)
    return x.narrow(bd, shard.b0, shard.batch).narrow(bd + 1, h0, h1 - h0)


def gather_outputs(local_out: torch.Tensor, plan: list[Shard], out: torch.Tensor | None = None,
                   group=None) -> torch.Tensor:
    """All-gather per-head outputs [..., b_loc, hq_loc, d] from every rank
    and assemble the full [..., B, Hq, d] tensor on every rank."""
    world = len(plan)
    lead = local_out.shape[:-3]
    src = local_out.contiguous().view(-1)
    buf = torch.empty(world * src.numel(), dtype=local_out.dtype, device=local_out.device)
    dist.all_gather_into_tensor(buf, src, group=group)
    buf = buf.view((world,) + tuple(local_out.shape))
    B = max(s.b1 for s in plan)
    Hq = max(s.q1 for s in plan)
    if out is None:
        out = torch.empty(tuple(lead) + (B, Hq, local_out.shape[-1]), dtype=local_out.dtype,
                          device=local_out.device)
    nd = local_out.dim()
    for s in plan:
        dst = out.narrow(nd - 3, s.b0, s.batch).narrow(nd - 2, s.q0, s.n_q_heads)
        dst.copy_(buf[s.rank])
    return out


def reduce_counters(c_miss: torch.Tensor, c_total: torch.Tensor, group=None) -> tuple[int, int]:
    """Job-wide (misses, selected) totals: local sums all-reduced (int64)."""
    v = torch.stack([c_miss.sum().to(torch.int64), c_total.sum().to(torch.int64)])
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(v, op=dist.ReduceOp.SUM, group=group)
    return int(v[0]), int(v[1])


class ShardedEngine:
    """The single-GPU `Engine` run on this rank's shard of a batch x KV-head
    grid.  Inputs are the job's full per-layer q/k/v rows (each rank reads
    its block); `step` returns the job's full outputs after one all-gather.
    """

    def __init__(self, n_layers: int, batch: int, n_q_heads: int, n_kv_heads: int, rank: int, world: int,
                 device, **shape_kw):
        from .engine import Engine, LayerShape

        self.plan = plan_shards(batch, n_q_heads, n_kv_heads, world)
        self.shard = self.plan[rank]
        s = self.shard
        self.shape = LayerShape(batch=s.batch, n_q_heads=s.n_q_heads, n_kv_heads=s.n_kv_heads, **shape_kw)
        self.engine = Engine(n_layers, self.shape, device=device)
        self.world = world

    def load_inputs(self, q, k, v):
        """q [L, B, Hq, d], k/v [L, B, Hkv, d] (full job) -> this rank's buffers."""
        e, s = self.engine, self.shard
        d = q.shape[-1]
        e.q_buf[..., :d].copy_(local_slice(q, s, heads="q"), non_blocking=True)
        e.k_buf[..., :d].copy_(local_slice(k, s, heads="kv"), non_blocking=True)
        e.v_buf[..., :d].copy_(local_slice(v, s, heads="kv"), non_blocking=True)

    def gather(self, out=None, last_layer_only=False):
        local = self.engine.out_buf[-1] if last_layer_only else self.engine.out_buf
        if self.world == 1:
            return local
        return gather_outputs(local, self.plan, out)

    def counters(self):
        cm, ct = self.engine.counters()
        return reduce_counters(cm, ct)
