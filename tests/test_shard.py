"""Sharding of (sequence, KV head) units across ranks:
partition plans, and the two collectives (output all-gather, counter
all-reduce) run with world_size 2 over gloo on CPU."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2510_23649_b200.shard import gather_outputs, local_slice, plan_shards, reduce_counters


def test_plan_whole_sequences():
    plan = plan_shards(8, 32, 8, 4)
    assert [(s.b0, s.b1, s.g0, s.g1) for s in plan] == [(0, 2, 0, 8), (2, 4, 0, 8), (4, 6, 0, 8), (6, 8, 0, 8)]
    assert all(s.n_q_heads == 32 for s in plan)


def test_plan_split_kv_heads_when_fewer_sequences():
    plan = plan_shards(1, 32, 8, 8)
    assert [(s.b0, s.g0, s.g1, s.q0, s.q1) for s in plan] == [(0, g, g + 1, 4 * g, 4 * g + 4) for g in range(8)]
    plan = plan_shards(2, 28, 4, 4)  # Qwen2.5-7B: 7 q heads per KV head
    assert [(s.b0, s.g0, s.g1, s.q0, s.q1) for s in plan] == [(0, 0, 2, 0, 14), (0, 2, 4, 14, 28),
                                                            (1, 0, 2, 0, 14), (1, 2, 4, 14, 28)]


@pytest.mark.parametrize("B,Hq,Hkv,W", [(8, 32, 8, 1), (8, 32, 8, 2), (8, 32, 8, 8), (1, 32, 8, 4), (4, 28, 4, 8)])
def test_plan_covers_every_unit_once(B, Hq, Hkv, W):
    plan = plan_shards(B, Hq, Hkv, W)
    units = [u for s in plan for u in s.units()]
    assert sorted(units) == [(b, g) for b in range(B) for g in range(Hkv)]
    assert len({(s.batch, s.n_kv_heads) for s in plan}) == 1  # equal blocks


def test_plan_rejects_unequal_split():
    with pytest.raises(ValueError):
        plan_shards(3, 32, 8, 2)
    with pytest.raises(ValueError):
        plan_shards(1, 28, 4, 8)


def test_local_slice_views():
    plan = plan_shards(2, 8, 2, 4)
    q = torch.arange(3 * 2 * 8 * 5).view(3, 2, 8, 5)
    k = torch.arange(3 * 2 * 2 * 5).view(3, 2, 2, 5)
    s = plan[3]  # sequence 1, KV head 1 -> q heads 4..7
    assert torch.equal(local_slice(q, s, heads="q"), q[:, 1:2, 4:8])
    assert torch.equal(local_slice(k, s, heads="kv"), k[:, 1:2, 1:2])


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, B, Hq, Hkv, outdir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        plan = plan_shards(B, Hq, Hkv, world)
        s = plan[rank]
        L, d = 3, 4
        full = torch.arange(L * B * Hq * d, dtype=torch.float32).view(L, B, Hq, d)
        local = local_slice(full, s, heads="q").contiguous()  # what this rank's engine would produce
        got = gather_outputs(local, plan)
        ok = torch.equal(got, full)
        cm = torch.full((s.batch, s.n_q_heads), rank + 1, dtype=torch.int64)
        ct = torch.full((s.batch, s.n_q_heads), 10, dtype=torch.int64)
        miss, tot = reduce_counters(cm, ct)
        per = s.batch * s.n_q_heads
        ok = ok and miss == per * sum(r + 1 for r in range(world)) and tot == 10 * per * world
        with open(os.path.join(outdir, f"rank{rank}"), "w") as f:
            f.write(str(int(ok)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("B,Hq,Hkv", [(4, 8, 2), (1, 8, 2)])
def test_gather_and_counters_world2_gloo(B, Hq, Hkv, tmp_path):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), B, Hq, Hkv, str(tmp_path)), nprocs=world, join=True)
    assert [open(tmp_path / f"rank{r}").read() for r in range(world)] == ["1", "1"]
