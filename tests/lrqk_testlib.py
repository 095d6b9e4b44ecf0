"""Helpers shared by the GPU parity tests: build a one-layer device state
from oracle-side arrays and run step-locked comparisons against the CPU
oracle (oracle/lrqk_oracle.py)."""

from __future__ import annotations

import numpy as np
import torch

from oracle import lrqk_oracle as O


def make_layer(B, Hq, Hkv, d, r, kb, lb, t_max, dtype="f32", policy="hbm", **kw):
    from paper_2510_23649_b200.engine import LayerShape, LayerState

    shape = LayerShape(batch=B, n_q_heads=Hq, n_kv_heads=Hkv, head_dim=d, rank=r, k_budget=kb,
                       lite_budget=lb, t_max=t_max, dtype=dtype, policy=policy)
    return LayerState(shape, **kw)


def to_dev(x, dtype=torch.float32):
    return torch.as_tensor(np.asarray(x), dtype=dtype, device="cuda")


def seed_layer(layer, A_K, B_Q, B_K, K, V):
    """A_K [B,Hq,l,r], B_* [B,Hq,r,d], K/V [B,Hkv,l,d] numpy float64."""
    layer.load_prompt(to_dev(A_K), to_dev(B_Q), to_dev(B_K), to_dev(K), to_dev(V))


def quantize(x, dtype):
    """Round float64 values to the storage dtype and back (what the GPU sees)."""
    t = torch.as_tensor(np.asarray(x), dtype=torch.float64)
    if dtype == "bf16":
        return t.to(torch.bfloat16).to(torch.float64).numpy()
    return t.to(torch.float32).to(torch.float64).numpy()


def rows_dev(x, layer):
    """[.., d] float64 -> padded device rows in the layer's storage dtype."""
    from paper_2510_23649_b200.engine import pad_last

    t = torch.as_tensor(np.asarray(x), dtype=torch.float32, device="cuda")
    return pad_last(t, layer.shape.dim_stride).to(layer.sdt).contiguous()


def near_tie_ok(scores, got, want, k_eff, eps):
    """Indices in the symmetric difference must be near-ties of the k-th score."""
    diff = set(got) ^ set(want)
    if not diff:
        return True, 0
    s = np.asarray(scores)
    kth = np.sort(s)[::-1][k_eff - 1] if k_eff > 0 else 0.0
    for i in diff:
        if abs(s[i] - kth) > eps:
            return False, len(diff)
    return True, len(diff)
