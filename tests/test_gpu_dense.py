"""The reference's per-call linear algebra on the float64 device kernels
(dense.cu) against the reference's own outputs (tests/golden/dense.npz,
spd.npz, compress.npz): gram, fro_norm_sq, solve_spd (incl. the jittered
rank-deficient case and both error classes), update_B/AK/AQ,
lagrangian_value, factor_residuals, khat_initial_guess, update_qhat/khat,
decode_compress with its workspace, update_projections, and top-k on float64
scores closer together than float32 can resolve."""

import numpy as np
import pytest

import paper_2510_23649_b200 as lrqk

pytestmark = pytest.mark.gpu

R64 = dict(rtol=1e-9, atol=1e-11)


def _f(g, i):
    return lrqk.LowRankFactors(g[f"A_Q{i}"], g[f"A_K{i}"], g[f"B_Q{i}"], g[f"B_K{i}"])


def test_gram_and_fro_norm(gold):
    np.testing.assert_array_equal(lrqk.gram(np.array([[1.0, 2.0], [3.0, 4.0]])), [[10.0, 14.0], [14.0, 20.0]])
    with pytest.raises(ValueError):
        lrqk.gram(np.zeros((0, 3)))
    g = gold("dense")
    for i in range(int(g["n"])):
        G = lrqk.gram(g[f"A_Q{i}"])
        np.testing.assert_allclose(G, g[f"gram{i}"], rtol=1e-12, atol=1e-12)
        np.testing.assert_array_equal(G, G.T)  # exactly symmetric, as the reference's mirror
        np.testing.assert_allclose(lrqk.gram(g[f"B_K{i}"].T), g[f"gramT{i}"], rtol=1e-12, atol=1e-14)
        assert lrqk.fro_norm_sq(g[f"Q{i}"]) == pytest.approx(float(g[f"fro{i}"]), rel=1e-12)


def test_solve_spd_golden_including_jitter(gold):
    g = gold("spd")
    for i in range(int(g["n"])):
        M = g[f"M{i}"]
        X = lrqk.solve_spd(M, g[f"R{i}"])
        # forward error of a backward-stable solve: cond(M [+ jitter]) * 2^-52
        # (case 9 is rank 8 of 32: the jittered system has cond ~1e11)
        ev = np.linalg.eigvalsh(M)
        lo = ev[0] if ev[0] > 1e-9 * ev[-1] else 1e-10 * (np.trace(M) / M.shape[0] + 1.0)
        rtol = max(1e-12, 50 * (ev[-1] / lo) * 2.0 ** -52)
        np.testing.assert_allclose(X, g[f"X{i}"], rtol=rtol, atol=rtol * np.abs(g[f"X{i}"]).max())


def test_solve_spd_errors():
    with pytest.raises(lrqk.NonFiniteError):
        lrqk.solve_spd(np.array([[np.nan, 0.0], [0.0, 1.0]]), np.ones((1, 2)))
    with pytest.raises(lrqk.NonFiniteError):
        lrqk.solve_spd(np.eye(2), np.array([[1.0, np.inf]]))
    with pytest.raises(lrqk.SolveFailedError):
        lrqk.solve_spd(-np.eye(3), np.ones((1, 3)))
    with pytest.raises(lrqk.SolveFailedError):  # indefinite: the jitter cannot rescue it
        lrqk.solve_spd(np.array([[1.0, 2.0], [2.0, 1.0]]), np.ones((1, 2)))
    with pytest.raises(ValueError, match="square"):
        lrqk.solve_spd(np.ones((2, 3)), np.ones((1, 2)))
    with pytest.raises(ValueError, match="cols"):
        lrqk.solve_spd(np.eye(2), np.ones((1, 3)))
    # the zero matrix is singular: the jittered retry (1e-10 (0 + 1) I) solves it
    X = lrqk.solve_spd(np.zeros((2, 2)), np.array([[1e-10, 2e-10]]))
    np.testing.assert_allclose(X, [[1.0, 2.0]], rtol=1e-12)


def test_prefill_algebra_matches_reference(gold):
    g = gold("dense")
    for i in range(int(g["n"])):
        Q, K = g[f"Q{i}"], g[f"K{i}"]
        f = _f(g, i)
        lq, lk = g[f"lam{i}"]
        cfg = lrqk.PrefillConfig(rank=f.A_Q.shape[1], lambda_q=float(lq), lambda_k=float(lk))
        np.testing.assert_allclose(lrqk.update_B(f.A_Q, Q), g[f"uB{i}"], **R64)
        np.testing.assert_allclose(lrqk.update_AK(Q, K, f, cfg), g[f"uAK{i}"], **R64)
        np.testing.assert_allclose(lrqk.update_AQ(Q, K, f, cfg), g[f"uAQ{i}"], **R64)
        assert lrqk.lagrangian_value(Q, K, f, cfg) == pytest.approx(float(g[f"lag{i}"]), rel=1e-10)
        np.testing.assert_allclose(lrqk.factor_residuals(Q, K, f), g[f"res{i}"], rtol=1e-9)


def test_prefill_golden_residuals_and_objective(gold):
    """factor_residuals / lagrangian_value of the reference's own converged
    factors (tests/golden/prefill.npz)."""
    g = gold("prefill")
    for i in range(int(g["n"])):
        f = lrqk.LowRankFactors(g[f"A_Q{i}"], g[f"A_K{i}"], g[f"B_Q{i}"], g[f"B_K{i}"])
        r = int(g[f"cfg{i}"][0])
        np.testing.assert_allclose(lrqk.factor_residuals(g[f"Q{i}"], g[f"K{i}"], f), g[f"res{i}"], rtol=1e-6,
                                   atol=1e-9)
        val = lrqk.lagrangian_value(g[f"Q{i}"], g[f"K{i}"], f, lrqk.PrefillConfig(rank=r))
        assert val == pytest.approx(float(g[f"obj{i}"][-1]), rel=1e-8, abs=1e-9)


def test_decode_closed_forms_match_reference(gold):
    g = gold("dense")
    for i in range(int(g["n"])):
        f = _f(g, i)
        l1, l2 = g[f"dlam{i}"]
        cfg = lrqk.DecodeConfig(lambda_1=float(l1), lambda_2=float(l2))
        step = lrqk.TokenStep(q=g[f"q{i}"], k=g[f"k{i}"], v=g[f"v{i}"])
        np.testing.assert_allclose(lrqk.khat_initial_guess(step.k, f.B_K), g[f"kh0{i}"], **R64)
        comp = lrqk.CompressedToken(g[f"qh_in{i}"], g[f"kh_in{i}"])
        ws = lrqk.DecodeWorkspace()
        np.testing.assert_allclose(lrqk.update_qhat(step, comp, f, g[f"A_res{i}"], g[f"K_res{i}"], cfg, ws),
                                   g[f"uq{i}"], **R64)
        np.testing.assert_allclose(ws.m_lq, g[f"m_lq{i}"], rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(ws.M_rq, g[f"M_rq{i}"], rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(lrqk.update_khat(step, comp, f, cfg), g[f"uk{i}"], **R64)
        with pytest.raises(ValueError, match="differ"):
            lrqk.update_qhat(step, comp, f, g[f"A_res{i}"], g[f"K_res{i}"][:0] if len(g[f"A_res{i}"]) else
                             np.zeros((1, step.q.shape[1])), cfg, ws)


def test_decode_compress_workspace_and_line_search(gold):
    g = gold("compress")
    for i in range(int(g["n"])):
        lam1, lam2, it, tol = g[f"cfg{i}"]
        cfg = lrqk.DecodeConfig(lambda_1=lam1, lambda_2=lam2, max_iter=int(it), tol=tol)
        step = lrqk.TokenStep(q=g[f"q{i}"], k=g[f"k{i}"], v=g[f"k{i}"])
        r, d = g[f"B_Q{i}"].shape
        f = lrqk.LowRankFactors(np.zeros((1, r)), np.zeros((1, r)), g[f"B_Q{i}"], g[f"B_K{i}"])
        comp, ws = lrqk.decode_compress(step, f, g[f"A_res{i}"], g[f"K_res{i}"], cfg)
        np.testing.assert_allclose(comp.q_hat, g[f"q_hat{i}"], **R64)
        np.testing.assert_allclose(comp.k_hat, g[f"k_hat{i}"], **R64)
        np.testing.assert_allclose(ws.M_rq, g[f"M_rq{i}"], rtol=1e-10, atol=1e-12)
        np.testing.assert_allclose(ws.m_lq, g[f"m_lq{i}"], rtol=1e-10, atol=1e-12)
        ws2 = lrqk.DecodeWorkspace()
        new = lrqk.update_projections(step, lrqk.CompressedToken(g[f"q_hat{i}"], g[f"k_hat{i}"]), f, ws2)
        np.testing.assert_allclose(new.B_Q, g[f"B_Q_new{i}"], **R64)
        np.testing.assert_allclose(new.B_K, g[f"B_K_new{i}"], **R64)
        np.testing.assert_allclose([ws2.eta_Q, ws2.eta_K], g[f"eta{i}"], rtol=1e-10)


def test_topk_float64_order(gold):
    """Scores 1e-12 apart round to the same float32: the float64 device
    select must still order them like the reference's argsort."""
    g = gold("dense")
    np.testing.assert_array_equal(lrqk.topk_indices(g["tk_s"], 37), g["tk_o"])
    s = np.array([1.0, 1.0 + 1e-13, 1.0 - 1e-13, 1.0, -0.0, 0.0])
    np.testing.assert_array_equal(lrqk.topk_indices(s, 2), [0, 1])
    np.testing.assert_array_equal(lrqk.topk_indices(s, 4), [0, 1, 2, 3])
    np.testing.assert_array_equal(lrqk.topk_indices(np.array([-0.0, 0.0, -1.0]), 1), [0])


def test_fp32_select_kernel_matches_reference_rule():
    """lrqk_select_scores (the general K4 select on fp32 scores, with the
    lite window) against the reference rule on the same fp32 values."""
    import torch
    from oracle import lrqk_oracle as O
    from paper_2510_23649_b200.api import _select_device

    rng = np.random.default_rng(9)
    for t, kb, lb, quant in [(40, 5, 3, True), (5000, 256, 16, False), (70000, 2048, 16, True), (9, 20, 4, False)]:
        s = rng.standard_normal(t + 1).astype(np.float32)
        if quant:
            s = np.round(s, 1).astype(np.float32)
        om, cnt = _select_device(torch.as_tensor(s[None], device="cuda"), t, kb, lb)
        got = np.sort(om[0, : int(cnt[0])].cpu().numpy().astype(np.int64))
        _, _, want = O.select(s.astype(np.float64), t, kb, lb)
        np.testing.assert_array_equal(got, want)
