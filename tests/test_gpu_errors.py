"""Error and recovery paths of the fused decode step on the GPU (SURVEY §5
failure detection): the device status word raises the reference's exception
classes (errors.py:4-9), a failed session step leaves the session as it was
(the reference raises before mutating anything, session.py:94-101), and the
singular-system path (jittered direct solves, linalg.py:80-91) completes and
stays consistent with the oracle on the GPU's own q_hat."""

import numpy as np
import pytest
import torch

import paper_2510_23649_b200 as lrqk
from paper_2510_23649_b200 import _lib
from tests.lrqk_testlib import ParityLog, StepLocked, make_layer, quantize, rows_dev, seed_layer

pytestmark = pytest.mark.gpu


def _layer_with_prompt(dtype="f32", zero_b=False, seed=0):
    rng = np.random.default_rng(seed)
    B, Hq, Hkv, d, r, kb, lb, l = 1, 4, 2, 64, 16, 24, 8, 200
    T = l + 8
    Q = quantize(rng.standard_normal((B, Hq, T, d)), dtype)
    K = quantize(rng.standard_normal((B, Hkv, T, d)), dtype)
    V = quantize(rng.standard_normal((B, Hkv, T, d)), dtype)
    A = quantize(rng.standard_normal((B, Hq, l, r)), dtype)
    BQ = np.zeros((B, Hq, r, d)) if zero_b else rng.standard_normal((B, Hq, r, d)) / 8
    BK = np.zeros((B, Hq, r, d)) if zero_b else rng.standard_normal((B, Hq, r, d)) / 8
    layer = make_layer(B, Hq, Hkv, d, r, kb, lb, t_max=T + 8, dtype=dtype)
    seed_layer(layer, A, BQ, BK, K[:, :, :l], V[:, :, :l])
    return layer, Q, K, V, l


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("where", ["q", "k", "v"])
def test_non_finite_input_raises(dtype, where):
    layer, Q, K, V, l = _layer_with_prompt(dtype)
    q, k, v = rows_dev(Q[:, :, l], layer), rows_dev(K[:, :, l], layer), rows_dev(V[:, :, l], layer)
    {"q": q, "k": k, "v": v}[where][0, 1, 3] = float("nan")
    out = torch.zeros(1, 4, layer.shape.dim_stride, device="cuda")
    layer.step(q, k, v, out)
    torch.cuda.synchronize()
    with pytest.raises(lrqk.NonFiniteError):
        layer.raise_status()


def test_session_step_is_atomic_on_device_errors():
    """1e39 is finite in float64 (it passes the as_row gate, linalg.py:37-45)
    but overflows the fp32 device rows: the step raises NonFiniteError and the
    session is left exactly as before, so it continues like a twin session
    that never saw the bad token."""
    from tests.conftest import golden

    g = golden("sessions")
    prompt, r, kb, lb = (int(x) for x in g["cfg2"])
    Q, K, V = g["Q2"], g["K2"], g["V2"]
    cfg = lrqk.SessionConfig(prefill=lrqk.PrefillConfig(rank=r), k_budget=kb, lite_budget=lb)
    a, b = lrqk.DecodeSession(cfg), lrqk.DecodeSession(cfg)
    a.prefill(Q[:prompt], K[:prompt], V[:prompt])
    b.prefill(Q[:prompt], K[:prompt], V[:prompt])
    for i in range(prompt, prompt + 3):
        a.decode_step(Q[i], K[i], V[i], compute_metrics=False)
        b.decode_step(Q[i], K[i], V[i], compute_metrics=False)
    bad = Q[prompt + 3].copy()
    bad[0] = 1e39
    with pytest.raises(lrqk.NonFiniteError):
        a.decode_step(bad, K[prompt + 3], V[prompt + 3], compute_metrics=False)
    with pytest.raises(lrqk.NonFiniteError):  # the host gate, as the reference
        a.decode_step(np.full(Q.shape[1], np.nan), K[prompt + 3], V[prompt + 3])
    assert a.cache.size == b.cache.size and a.cache.fast_resident == b.cache.fast_resident
    for i in range(prompt + 3, prompt + 12):
        ra = a.decode_step(Q[i], K[i], V[i])
        rb = b.decode_step(Q[i], K[i], V[i])
        assert (ra.step, ra.miss_count, ra.selected_count, ra.recall_vs_exact) == \
               (rb.step, rb.miss_count, rb.selected_count, rb.recall_vs_exact)
        np.testing.assert_array_equal(a.last_output, b.last_output)
        np.testing.assert_array_equal(a.factors.B_Q, b.factors.B_Q)
    assert (a.stats.c_miss, a.stats.c_total) == (b.stats.c_miss, b.stats.c_total)


def test_capacity_exhaustion_raises():
    layer, Q, K, V, l = _layer_with_prompt("f32")
    out = torch.zeros(1, 4, layer.shape.dim_stride, device="cuda")
    layer.view("ctx_len").fill_(layer.shape.t_max)
    layer.step(rows_dev(Q[:, :, l], layer), rows_dev(K[:, :, l], layer), rows_dev(V[:, :, l], layer), out)
    torch.cuda.synchronize()
    with pytest.raises(RuntimeError, match="capacity"):
        layer.raise_status()


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_singular_systems_take_the_jittered_solve(dtype):
    """B_Q = B_K = 0 with fewer resident rows than the rank makes every
    compression system singular: the kernel falls back to the direct solves
    with the reference's jitter retry (LRQK_ST_FALLBACK | LRQK_ST_JITTERED;
    linalg.py:80-91) and the step completes.  The jittered solutions of these
    rank-deficient systems are conditioning-limited in fp32,
    so q_hat is only required to be finite, and the rest of the step --
    scores, selection, counters, attention, the B line search -- is judged
    against the oracle on the GPU's own q_hat."""
    layer, Q, K, V, l = _layer_with_prompt(dtype, zero_b=True, seed=3)
    lock = StepLocked(layer, Q, K, V, l)
    log = ParityLog(f"singular_{dtype}")
    out = torch.zeros(1, 4, layer.shape.dim_stride, device="cuda")
    seen = 0
    for t in range(l, l + 5):
        layer.step(rows_dev(Q[:, :, t], layer), rows_dev(K[:, :, t], layer), rows_dev(V[:, :, t], layer), out)
        torch.cuda.synchronize()
        seen |= layer.raise_status()
        lock.check_step(out, log, dtype, rtol_hat=2e-3 if dtype == "f32" else 5e-2, strict=False)
        assert np.isfinite(layer.view("q_hat").cpu().numpy()).all()
    assert seen & _lib.ST_FALLBACK and seen & _lib.ST_JITTERED
    log.write()
