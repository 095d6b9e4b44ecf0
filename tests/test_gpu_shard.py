"""Sharded decode on the GPU.

* KV-head split of one sequence: the two rank-local engines a 2-GPU job
  would run (plan_shards(1, Hq, Hkv, 2): KV heads [0, Hkv/2) and
  [Hkv/2, Hkv)), stepped in one process on one GPU, must give the full
  engine's selections and outputs for their heads -- the units are
  independent, only the grid partition (and so the order of
  floating-point partial sums) differs.
* With two or more GPUs, the real 2-rank NCCL run of bench.py (batch
  sharding and KV-head split), so SCALE has a tested path.
"""

import json
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_kv_head_split_engines_match_full_engine():
    from paper_2510_23649_b200.engine import Engine, LayerShape
    from paper_2510_23649_b200.shard import local_slice, plan_shards

    torch.manual_seed(5)
    nL, B, Hq, Hkv, d, r, kb, lb, l = 2, 1, 8, 4, 128, 32, 128, 16, 6000
    kw = dict(head_dim=d, rank=r, k_budget=kb, lite_budget=lb, t_max=l + 16, dtype="bf16")
    full = Engine(nL, LayerShape(batch=B, n_q_heads=Hq, n_kv_heads=Hkv, **kw), device="cuda")
    plan = plan_shards(B, Hq, Hkv, 2)
    parts = [Engine(nL, LayerShape(batch=s.batch, n_q_heads=s.n_q_heads, n_kv_heads=s.n_kv_heads, **kw),
                    device="cuda") for s in plan]
    for i in range(nL):
        AK = torch.randn(B, Hq, l, r, device="cuda")
        BQ = torch.randn(B, Hq, r, d, device="cuda") / d ** 0.5
        BK = torch.randn(B, Hq, r, d, device="cuda") / d ** 0.5
        K = torch.randn(B, Hkv, l, d, device="cuda").bfloat16()
        V = torch.randn(B, Hkv, l, d, device="cuda").bfloat16()
        full.layers[i].load_prompt(AK, BQ, BK, K, V)
        for s, e in zip(plan, parts):
            e.layers[i].load_prompt(AK[:, s.q0:s.q1].contiguous(), BQ[:, s.q0:s.q1].contiguous(),
                                    BK[:, s.q0:s.q1].contiguous(), K[:, s.g0:s.g1].contiguous(),
                                    V[:, s.g0:s.g1].contiguous())
    for step in range(5):
        q = torch.randn(nL, B, Hq, d, device="cuda").bfloat16()
        k = torch.randn(nL, B, Hkv, d, device="cuda").bfloat16()
        v = torch.randn(nL, B, Hkv, d, device="cuda").bfloat16()
        full.q_buf[..., :d].copy_(q)
        full.k_buf[..., :d].copy_(k)
        full.v_buf[..., :d].copy_(v)
        full.decode_step()
        for s, e in zip(plan, parts):
            e.q_buf[..., :d].copy_(local_slice(q, s, heads="q"))
            e.k_buf[..., :d].copy_(local_slice(k, s, heads="kv"))
            e.v_buf[..., :d].copy_(local_slice(v, s, heads="kv"))
            e.decode_step()
        torch.cuda.synchronize()
        full.raise_status()
        for s, e in zip(plan, parts):
            e.raise_status()
            for i in range(nL):
                ref = full.out_buf[i, :, s.q0:s.q1, :d]
                got = e.out_buf[i, :, :, :d]
                assert torch.allclose(got, ref, rtol=1e-4, atol=1e-5), (step, i, s.rank)
                fi, pi = full.layers[i], e.layers[i]
                assert torch.equal(pi.view("res_cnt"), fi.view("res_cnt")[:, s.q0:s.q1])
                for h in range(s.n_q_heads):
                    n = int(pi.view("res_cnt")[0, h])
                    a = torch.sort(pi.view("res_idx")[0, h, :n]).values
                    b = torch.sort(fi.view("res_idx")[0, s.q0 + h, :n]).values
                    assert torch.equal(a, b), (step, i, s.rank, h)
                assert torch.equal(pi.view("c_miss"), fi.view("c_miss")[:, s.q0:s.q1])


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs 2 GPUs")
@pytest.mark.parametrize("extra", [[], ["--global-batch", "1"]])
def test_two_rank_nccl_bench(extra):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", "29531", os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "3",
           "--warmup", "3", "--ctx", "8192", "--layers", "2", "--no-cpu-baseline"] + extra
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and line["value"] > 0
    assert line["scaling"] == ("strong" if extra else "weak")
