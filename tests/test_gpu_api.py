"""The drop-in API, exercised like the reference's own tests
(pkg/tests/test_cache.py, test_linalg.py, test_attention.py,
test_session.py, test_decode.py), at GPU (fp32) tolerances."""

import numpy as np
import pytest

import paper_2510_23649_b200 as lrqk
from oracle import lrqk_oracle as O

pytestmark = pytest.mark.gpu


def topk_oracle(scores, k):
    pairs = sorted(((-s, i) for i, s in enumerate(scores)))
    return sorted(i for _, i in pairs[: min(k, len(scores))])


def brute_force_selection(scores, t, k_budget, lite_budget):
    lite = list(range(max(0, t + 1 - lite_budget), t + 1))
    rest = [i for i in range(t + 1) if i not in lite]
    rest.sort(key=lambda i: (-scores[i], i))
    return sorted(rest[:k_budget]), lite


def test_topk_golden(gold):
    np.testing.assert_array_equal(lrqk.topk_indices(np.array([0.1, 0.9, 0.5]), 2), [1, 2])
    np.testing.assert_array_equal(lrqk.topk_indices(np.array([3.0, 3.0, 3.0]), 2), [0, 1])
    np.testing.assert_array_equal(lrqk.topk_indices(np.array([7.0]), 5), [0])
    with pytest.raises(ValueError):
        lrqk.topk_indices(np.array([1.0]), 0)
    g = gold("topk")
    for i in range(int(g["n"])):
        np.testing.assert_array_equal(lrqk.topk_indices(g[f"s{i}"], int(g[f"k{i}"])), g[f"o{i}"])


def test_topk_quantized_ties_vs_sort_oracle():
    rng = np.random.default_rng(3)
    for _ in range(30):
        n = int(rng.integers(1, 40))
        scores = np.round(rng.standard_normal(n), 1)
        k = int(rng.integers(1, n + 3))
        np.testing.assert_array_equal(lrqk.topk_indices(scores, k), topk_oracle(scores.tolist(), k))


def test_select_active_golden_and_rules(gold):
    sel = lrqk.select_active(np.zeros(5), t=4, k_budget=3, lite_budget=2)
    np.testing.assert_array_equal(sel.omega, np.arange(5))
    sel = lrqk.select_active(np.ones(6), t=5, k_budget=2, lite_budget=2)
    np.testing.assert_array_equal(sel.omega_l, [4, 5])
    np.testing.assert_array_equal(sel.omega_k, [0, 1])
    with pytest.raises(ValueError, match="cover"):
        lrqk.select_active(np.zeros(4), t=4, k_budget=1, lite_budget=1)
    g = gold("select")
    for i in range(int(g["n"])):
        t, kb, lb = (int(x) for x in g[f"p{i}"])
        sel = lrqk.select_active(g[f"s{i}"], t, kb, lb)
        np.testing.assert_array_equal(sel.omega, g[f"o{i}"])
        np.testing.assert_array_equal(sel.omega_k, g[f"ok{i}"])


def test_select_active_brute_force():
    rng = np.random.default_rng(3)
    for _ in range(30):
        t = int(rng.integers(0, 40))
        scores = np.round(rng.standard_normal(t + 1), 1)
        kb, lb = int(rng.integers(1, 6)), int(rng.integers(1, 6))
        sel = lrqk.select_active(scores, t, kb, lb)
        want_k, want_l = brute_force_selection(scores, t, kb, lb)
        assert sel.omega_k.tolist() == want_k and sel.omega_l.tolist() == want_l


def test_proxy_scores():
    np.testing.assert_array_equal(lrqk.proxy_scores(np.array([[0.0, 0.0, 1.0, 0.0]]), np.eye(4)), [0, 0, 1, 0])
    rng = np.random.default_rng(1)
    store = rng.standard_normal((16, 4))
    q = rng.standard_normal((1, 4))
    np.testing.assert_allclose(lrqk.proxy_scores(q, store), store @ q.ravel(), rtol=1e-6, atol=1e-6)


def test_exact_attention(gold):
    res = lrqk.exact_attention(np.ones((1, 3)), np.ones((1, 3)), np.full((1, 3), 2.0))
    np.testing.assert_allclose(res.weights, [1.0])
    np.testing.assert_allclose(res.output, np.full((1, 3), 2.0))
    with pytest.raises(ValueError, match="at least one key"):
        lrqk.exact_attention(np.ones((1, 2)), np.zeros((0, 2)), np.zeros((0, 2)))
    q = np.full((1, 2), 500.0)
    K = np.array([[1000.0, 0.0], [0.0, 1000.0], [-1000.0, -1000.0]])
    res = lrqk.exact_attention(q, K, np.eye(3, 2))
    assert np.isfinite(res.weights).all() and np.isfinite(res.output).all()
    g = gold("scores_attention")
    for i in range(int(g["n"])):
        r = lrqk.exact_attention(g[f"q{i}"], g[f"K{i}"], g[f"V{i}"])
        np.testing.assert_allclose(r.output, g[f"out{i}"], rtol=1e-4, atol=1e-5)
        np.testing.assert_allclose(r.weights, g[f"w{i}"], rtol=1e-4, atol=1e-6)


def test_cache_accounting_replay():
    rng = np.random.default_rng(8)
    dim, rank, kb, lb = 3, 2, 3, 2
    cache = lrqk.TieredKVCache(dim=dim, rank=rank, k_budget=kb, lite_budget=lb)
    stats = lrqk.CacheStats()
    selections = []
    for t in range(40):
        lrqk.append_token(cache, rng.standard_normal((1, dim)), rng.standard_normal((1, dim)),
                          rng.standard_normal((1, rank)))
        scores = lrqk.proxy_scores(rng.standard_normal((1, rank)), cache.proxy_store)
        sel = lrqk.select_active(scores, t, kb, lb)
        lrqk.fetch_and_merge(cache, sel, stats)
        selections.append([int(i) for i in sel.omega])
    resident, c_miss, c_total = set(), 0, 0
    for t, omega in enumerate(selections):
        resident.add(t)
        c_miss += len(set(omega) - resident)
        c_total += len(omega)
        resident = set(omega)
    assert (stats.c_miss, stats.c_total) == (c_miss, c_total)


def test_fetch_and_merge_partial_overlap_and_range():
    rng = np.random.default_rng(0)
    cache = lrqk.TieredKVCache(dim=3, rank=2, k_budget=4, lite_budget=2)
    for _ in range(6):
        lrqk.append_token(cache, rng.standard_normal((1, 3)), rng.standard_normal((1, 3)), rng.standard_normal((1, 2)))
    cache.fast_resident = {0, 1, 2, 3}
    stats = lrqk.CacheStats()
    omega = np.array([2, 3, 4, 5])
    K, V = lrqk.fetch_and_merge(cache, lrqk.SelectionSet(omega[:2], omega[2:], omega), stats)
    assert stats.c_miss == 2 and stats.c_total == 4 and cache.fast_resident == {2, 3, 4, 5}
    with pytest.raises(IndexError):
        bad = np.array([1, 9])
        lrqk.fetch_and_merge(cache, lrqk.SelectionSet(bad[:1], bad[1:], bad), lrqk.CacheStats())
    assert lrqk.miss_rate(lrqk.CacheStats(c_miss=2, c_total=5)) == pytest.approx(0.4)


def test_decode_compress_and_update_projections_match_golden(gold):
    g = gold("compress")
    for i in range(int(g["n"])):
        lam1, lam2, it, tol = g[f"cfg{i}"]
        cfg = lrqk.DecodeConfig(lambda_1=lam1, lambda_2=lam2, max_iter=int(it), tol=tol)
        step = lrqk.TokenStep(q=g[f"q{i}"], k=g[f"k{i}"], v=g[f"k{i}"])
        r, d = g[f"B_Q{i}"].shape
        f = lrqk.LowRankFactors(np.zeros((1, r)), np.zeros((1, r)), g[f"B_Q{i}"], g[f"B_K{i}"])
        comp, ws = lrqk.decode_compress(step, f, g[f"A_res{i}"], g[f"K_res{i}"], cfg)
        np.testing.assert_allclose(comp.q_hat, g[f"q_hat{i}"], rtol=2e-3, atol=2e-3 * np.abs(g[f"q_hat{i}"]).max())
        np.testing.assert_allclose(comp.k_hat, g[f"k_hat{i}"], rtol=2e-3, atol=2e-3 * np.abs(g[f"k_hat{i}"]).max())
        # line search on the reference's own compressed rows
        ref_comp = lrqk.CompressedToken(g[f"q_hat{i}"], g[f"k_hat{i}"])
        ws2 = lrqk.DecodeWorkspace()
        new = lrqk.update_projections(step, ref_comp, f, ws2)
        np.testing.assert_allclose(new.B_Q, g[f"B_Q_new{i}"], rtol=1e-4, atol=1e-5)
        np.testing.assert_allclose(new.B_K, g[f"B_K_new{i}"], rtol=1e-4, atol=1e-5)
        np.testing.assert_allclose([ws2.eta_Q, ws2.eta_K], g[f"eta{i}"], rtol=1e-4)


def test_prefill_run_matches_golden(gold):
    g = gold("prefill")
    for i in (0, 1):
        r, it, tol = g[f"cfg{i}"]
        cfg = lrqk.PrefillConfig(rank=int(r), max_iter=int(it), tol=float(tol),
                                 init=lrqk.InitStrategy(str(g[f"init{i}"]), 0))
        run = lrqk.prefill_run(g[f"Q{i}"], g[f"K{i}"], cfg)
        assert run.sweeps == int(g[f"sweeps{i}"]) and run.converged == bool(g[f"conv{i}"])
        np.testing.assert_allclose(run.objective, g[f"obj{i}"], rtol=2e-3)


def test_session_and_run_simulation():
    from tests.conftest import golden

    g = golden("sessions")
    prompt, r, kb, lb = (int(x) for x in g["cfg1"])
    Q, K, V = g["Q1"], g["K1"], g["V1"]
    cfg = lrqk.SessionConfig(prefill=lrqk.PrefillConfig(rank=r), decode=lrqk.DecodeConfig(), k_budget=kb,
                             lite_budget=lb)
    sess = lrqk.DecodeSession(cfg)
    with pytest.raises(RuntimeError, match="prefill"):
        sess.decode_step(np.ones(Q.shape[1]), np.ones(Q.shape[1]), np.ones(Q.shape[1]))
    sess.prefill(Q[:prompt], K[:prompt], V[:prompt])
    assert sess.cache.size == prompt
    assert sess.cache.fast_resident == set(range(prompt - lb, prompt))
    for i in range(prompt, prompt + 15):
        rep = sess.decode_step(Q[i], K[i], V[i])
        idx = sess.last_selection.omega
        ref = O.attend(Q[i : i + 1], K[idx], V[idx])[0]
        np.testing.assert_allclose(sess.last_output, ref, rtol=1e-4, atol=1e-4 * np.abs(ref).max())
        assert rep.step == i and rep.selected_count == len(idx) and 0.0 <= rep.recall_vs_exact <= 1.0
    res = lrqk.run_simulation(Q[:80], K[:80], V[:80], prompt_len=40,
                              cfg=lrqk.SessionConfig(prefill=lrqk.PrefillConfig(rank=r), k_budget=200, lite_budget=8))
    assert all(abs(x.output_err) < 1e-5 for x in res.reports)  # full coverage -> exact attention
    assert res.stats.c_total == sum(x.selected_count for x in res.reports)
