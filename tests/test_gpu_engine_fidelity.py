"""Engine.fidelity: recall of every (layer, sequence,
q-head) selection against the exact top-k over the full key history, and
the relative output error against full-history attention, computed on the
device -- checked against float64 numpy of the reference's _fidelity
(session.py:119-131: exact_topk -> selection_recall, exact_attention) on the
same stored keys, values, queries, selections and outputs."""

import math

import numpy as np
import pytest
import torch

from oracle import lrqk_oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_engine_fidelity_matches_float64_reference(dtype):
    from paper_2510_23649_b200.engine import Engine, LayerShape

    torch.manual_seed(3)
    nL, B, Hq, Hkv, d, r, kb, lb, l = 2, 2, 4, 2, 128, 32, 64, 16, 1500
    sh = LayerShape(batch=B, n_q_heads=Hq, n_kv_heads=Hkv, head_dim=d, rank=r, k_budget=kb, lite_budget=lb,
                    t_max=l + 16, dtype=dtype)
    eng = Engine(nL, sh, device="cuda")
    sdt = torch.float32 if dtype == "f32" else torch.bfloat16
    for layer in eng.layers:
        AK = torch.randn(B, Hq, l, r, device="cuda")
        BQ = torch.randn(B, Hq, r, d, device="cuda") / d ** 0.5
        BK = torch.randn(B, Hq, r, d, device="cuda") / d ** 0.5
        K = torch.randn(B, Hkv, l, d, device="cuda").to(sdt)
        V = torch.randn(B, Hkv, l, d, device="cuda").to(sdt)
        layer.load_prompt(AK, BQ, BK, K, V)
    for _ in range(3):
        eng.q_buf[..., :d].copy_(torch.randn(nL, B, Hq, d, device="cuda"))
        eng.k_buf[..., :d].copy_(torch.randn(nL, B, Hkv, d, device="cuda"))
        eng.v_buf[..., :d].copy_(torch.randn(nL, B, Hkv, d, device="cuda"))
        eng.decode_step()
    torch.cuda.synchronize()
    eng.raise_status()
    recall, err = eng.fidelity()
    recall, err = recall.cpu().numpy(), err.cpu().numpy()
    n = int(eng.ctx[0].item())
    G = Hq // Hkv
    k_eff = min(kb, n)
    for i, layer in enumerate(eng.layers):
        Ks = layer.view("slow_k")[:, :, :n, :d].double().cpu().numpy()
        Vs = layer.view("slow_v")[:, :, :n, :d].double().cpu().numpy()
        idx = layer.view("res_idx").cpu().numpy()
        cnt = layer.view("res_cnt").cpu().numpy()
        q = eng.q_buf[i, :, :, :d].double().cpu().numpy()
        out = eng.out_buf[i, :, :, :d].double().cpu().numpy()
        for b in range(B):
            for h in range(Hq):
                Kg, Vg = Ks[b, h // G], Vs[b, h // G]
                s = Kg @ q[b, h]
                exact = set(O.largest_k(s, k_eff).tolist())
                sel = set(idx[b, h, : cnt[b, h]].tolist())
                rec = len(sel & exact) / k_eff
                w = np.exp((s - s.max()) / math.sqrt(d))
                full = (w / w.sum()) @ Vg
                e = np.linalg.norm(out[b, h] - full) / np.linalg.norm(full)
                # one top-k boundary row may flip between the fp32 device and
                # fp64 host products of the same q and K
                assert abs(recall[i, b, h] - rec) <= 1.0 / k_eff + 1e-6, (i, b, h, recall[i, b, h], rec)
                assert abs(err[i, b, h] - e) <= 1e-4 + 1e-3 * e, (i, b, h, err[i, b, h], e)
    assert np.all((recall >= 0) & (recall <= 1)) and np.all(np.isfinite(err))
