"""The fused kernel's shared stream tail (StreamPool, score_common.cuh):
which block streams which tile of a head must not change anything the
selection or the attention sees -- keys, candidate bits and the merged
window histogram are per row, the classification and the attention keep
the static part ranges.  The same decode run with the pool off, at the
default 10 % and with every tile taken from the pool (LRQK_SA_POOL, read
once per process) must give bit-identical selections, counters, outputs
and B factors."""

import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[2])
from paper_2510_23649_b200.engine import Engine, LayerShape
nL, B, Hq, Hkv, d, r, kb, lb, l = 2, 1, 8, 2, 128, 32, 256, 16, 20000
sh = LayerShape(batch=B, n_q_heads=Hq, n_kv_heads=Hkv, head_dim=d, rank=r, k_budget=kb, lite_budget=lb,
                t_max=l + 16, dtype="bf16")
eng = Engine(nL, sh, device="cuda")
g = torch.Generator(device="cuda"); g.manual_seed(1)
for layer in eng.layers:
    AK = torch.randn(B, Hq, l, r, device="cuda", generator=g)
    BQ = torch.randn(B, Hq, r, d, device="cuda", generator=g) / d ** 0.5
    BK = torch.randn(B, Hq, r, d, device="cuda", generator=g) / d ** 0.5
    K = torch.randn(B, Hkv, l, d, device="cuda", generator=g).bfloat16()
    V = torch.randn(B, Hkv, l, d, device="cuda", generator=g).bfloat16()
    layer.load_prompt(AK, BQ, BK, K, V)
outs, idx = [], []
for step in range(5):
    eng.q_buf[..., :d].copy_(torch.randn(nL, B, Hq, d, device="cuda", generator=g))
    eng.k_buf[..., :d].copy_(torch.randn(nL, B, Hkv, d, device="cuda", generator=g))
    eng.v_buf[..., :d].copy_(torch.randn(nL, B, Hkv, d, device="cuda", generator=g))
    eng.decode_step()
    torch.cuda.synchronize()
    eng.raise_status()
    outs.append(eng.out_buf[..., :d].cpu().numpy())
    idx.append(np.stack([lay.view("res_idx").cpu().numpy() for lay in eng.layers]))
assert eng.fused
fused_heads = sum(int(lay.buf["sel_meta"].view(torch.int32)[: B * Hq * 48].view(B * Hq, 48)[:, 38].sum())
                  for lay in eng.layers)
np.savez(sys.argv[1], out=np.stack(outs), idx=np.stack(idx),
         cnt=np.stack([lay.view("res_cnt").cpu().numpy() for lay in eng.layers]),
         miss=np.stack([lay.view("c_miss").cpu().numpy() for lay in eng.layers]),
         bq=np.stack([lay.view("B_Q").cpu().numpy() for lay in eng.layers]),
         bk=np.stack([lay.view("B_K").cpu().numpy() for lay in eng.layers]),
         fused_heads=np.array(fused_heads))
"""


def _run(tmp_path, pool):
    out = tmp_path / f"pool{pool}.npz"
    env = dict(os.environ, LRQK_SA_POOL=str(pool))
    r = subprocess.run([sys.executable, "-c", _SCRIPT, str(out), ROOT], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    return np.load(out)


def test_stream_pool_share_changes_nothing(tmp_path):
    ref = _run(tmp_path, 0)
    # the fused path ran for most head-steps (meta M_STAT + 5 counts them)
    assert int(ref["fused_heads"]) >= 2 * 8 * 3
    for pool in (10, 100):
        got = _run(tmp_path, pool)
        for name in ("idx", "cnt", "miss", "out", "bq", "bk", "fused_heads"):
            assert np.array_equal(got[name], ref[name]), (pool, name)
