"""Step-locked oracle parity at the BASELINE.json configurations.

  * C1 exactly: one LLaMA-3-8B attention layer (32 q / 8 kv heads, d=128),
    4K prompt, r=32, top-k 256, 16 recent, fp32, 32 decode steps -- once
    through lrqk_decode_step and once through the Engine (CUDA-graph replay).
  * C4 shape, bf16: one KV group (4 q heads sharing one K/V head) at a 128K
    prompt, r=32, top-k 2048, 16 recent, through the first (sampled-radix)
    step and the fused threshold-window steps after it.

Every head-step is compared with the CPU oracle run from the GPU's previous
state (tests/lrqk_testlib.StepLocked): q_hat/k_hat, the appended proxy row,
the post-step B_Q/B_K (the line search, including the bf16 deferred update
the bench runs), the scores against fp64 products on the same q_hat, the
selection against the reference rule modulo the documented near-tie bound
(every excused index logged), bit-exact hit/miss counters, and attention
outputs (fp32 1e-4 / bf16 2e-2 relative).
"""

import numpy as np
import pytest
import torch

from tests.lrqk_testlib import ParityLog, StepLocked, make_layer, quantize, rows_dev

pytestmark = pytest.mark.gpu


def _c1_inputs(T, Hq=32, Hkv=8, d=128):
    """SURVEY §8(d) synthetic inputs: Q per q-head from default_rng(100+h),
    K then V per KV head from default_rng(200+g), fp32."""
    Q = np.stack([np.random.default_rng(100 + h).standard_normal((T, d), dtype=np.float32) for h in range(Hq)])
    KV = [np.random.default_rng(200 + g) for g in range(Hkv)]
    K = np.stack([g.standard_normal((T, d), dtype=np.float32) for g in KV])
    V = np.stack([g.standard_normal((T, d), dtype=np.float32) for g in KV])
    return Q[None].astype(np.float64), K[None].astype(np.float64), V[None].astype(np.float64)


def _prefill_into(layer, Q, K, V, prompt, dtype):
    from paper_2510_23649_b200.engine import prefill_factorize_device

    sh = layer.shape
    B, Hq, Hkv, d, r = sh.batch, sh.n_q_heads, sh.n_kv_heads, sh.head_dim, sh.rank
    sdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    Qp = torch.as_tensor(Q[:, :, :prompt], dtype=torch.float32, device="cuda").reshape(B * Hq, prompt, d).to(sdt)
    Kp = torch.as_tensor(K[:, :, :prompt], dtype=torch.float32, device="cuda").reshape(B * Hkv, prompt, d).to(sdt)
    Vp = torch.as_tensor(V[:, :, :prompt], dtype=torch.float32, device="cuda").reshape(B * Hkv, prompt, d).to(sdt)
    res = prefill_factorize_device(Qp, Kp, r, dtype=dtype, group=Hq // Hkv)
    layer.load_prompt(res["A_K"].reshape(B, Hq, prompt, r), res["B_Q"].reshape(B, Hq, r, d),
                      res["B_K"].reshape(B, Hq, r, d), Kp.view(B, Hkv, prompt, d), Vp.view(B, Hkv, prompt, d))


@pytest.mark.parametrize("driver", ["decode_step", "engine"])
def test_c1_step_locked(driver, select_path):
    from paper_2510_23649_b200.engine import Engine, LayerShape

    prompt, steps = 4096, 32
    Hq, Hkv, d, r, kb, lb = 32, 8, 128, 32, 256, 16
    Q, K, V = _c1_inputs(prompt + steps)
    shape = LayerShape(batch=1, n_q_heads=Hq, n_kv_heads=Hkv, head_dim=d, rank=r, k_budget=kb, lite_budget=lb,
                       t_max=prompt + steps + 8, dtype="f32")
    if driver == "engine":
        eng = Engine(1, shape, device="cuda")
        layer = eng.layers[0]
        out = eng.out_buf[0]
    else:
        layer = make_layer(1, Hq, Hkv, d, r, kb, lb, t_max=prompt + steps + 8, dtype="f32")
        out = torch.zeros(1, Hq, layer.shape.dim_stride, device="cuda")
    _prefill_into(layer, Q, K, V, prompt, "f32")
    lock = StepLocked(layer, Q, K, V, prompt)
    log = ParityLog(f"c1_{driver}")
    for i, t in enumerate(range(prompt, prompt + steps)):
        q, k, v = rows_dev(Q[:, :, t], layer), rows_dev(K[:, :, t], layer), rows_dev(V[:, :, t], layer)
        if driver == "engine":
            eng.q_buf[0].copy_(q)
            eng.k_buf[0].copy_(k)
            eng.v_buf[0].copy_(v)
            if i < 2:
                eng.decode_step()
            else:
                eng.replay()
        else:
            layer.step(q, k, v, out)
        torch.cuda.synchronize()
        layer.raise_status()
        lock.check_step(out, log, "f32", rtol_hat=2e-3)
    log.write()
    assert log.rec["head_steps"] == steps * Hq
    # near-ties are rare at fp32: the selection equals the fp64 one on the same q_hat almost always
    assert log.rec["selections_identical"] >= 0.95 * steps * Hq


def test_c4_shape_kv_group_128k_bf16(select_path):
    torch.manual_seed(0)
    prompt, steps = 131072, 6
    Hq, Hkv, d, r, kb, lb = 4, 1, 128, 32, 2048, 16
    rng = np.random.default_rng(41)
    T = prompt + steps
    Q = quantize(rng.standard_normal((1, Hq, T, d), dtype=np.float32), "bf16")
    K = quantize(rng.standard_normal((1, Hkv, T, d), dtype=np.float32), "bf16")
    V = quantize(rng.standard_normal((1, Hkv, T, d), dtype=np.float32), "bf16")
    layer = make_layer(1, Hq, Hkv, d, r, kb, lb, t_max=T + 32, dtype="bf16")
    _prefill_into(layer, Q, K, V, prompt, "bf16")
    lock = StepLocked(layer, Q, K, V, prompt)
    log = ParityLog("c4_kv_group_128k_bf16")
    out = torch.zeros(1, Hq, layer.shape.dim_stride, device="cuda")
    for t in range(prompt, T):
        layer.step(rows_dev(Q[:, :, t], layer), rows_dev(K[:, :, t], layer), rows_dev(V[:, :, t], layer), out)
        torch.cuda.synchronize()
        layer.raise_status()
        lock.check_step(out, log, "bf16", rtol_hat=5e-2)
    log.write()
    # the first step runs the sampled radix select, the rest the fused window path
    stat = layer.view("sel_meta")[0, :, 33:40].sum(0).cpu().numpy()
    assert stat[0] == Hq and stat[5] == Hq * (steps - 1), stat
