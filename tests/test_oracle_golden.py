"""Pin the CPU oracle to the reference: replay every golden fixture produced
by tests/golden/make_golden.py (which imported the reference package) through
oracle/lrqk_oracle.py.  Index sets and counters must match exactly; float
results to 1e-9 relative (BLAS summation order differs)."""

import numpy as np
import pytest

from oracle import lrqk_oracle as O


def test_topk_matches_reference(gold):
    g = gold("topk")
    for i in range(int(g["n"])):
        got = O.largest_k(g[f"s{i}"], int(g[f"k{i}"]))
        np.testing.assert_array_equal(got, g[f"o{i}"])


def test_select_matches_reference(gold):
    g = gold("select")
    for i in range(int(g["n"])):
        t, kb, lb = (int(x) for x in g[f"p{i}"])
        ok, ol, om = O.select(g[f"s{i}"], t, kb, lb)
        np.testing.assert_array_equal(ok, g[f"ok{i}"])
        np.testing.assert_array_equal(ol, g[f"ol{i}"])
        np.testing.assert_array_equal(om, g[f"o{i}"])


def test_scores_and_attention_match_reference(gold):
    g = gold("scores_attention")
    for i in range(int(g["n"])):
        np.testing.assert_allclose(O.proxy_scores(g[f"qh{i}"], g[f"store{i}"]), g[f"sc{i}"],
                                   rtol=1e-12, atol=1e-12)
        out, w = O.attend(g[f"q{i}"], g[f"K{i}"], g[f"V{i}"])
        np.testing.assert_allclose(out, g[f"out{i}"], rtol=1e-10, atol=1e-12)
        np.testing.assert_allclose(w, g[f"w{i}"], rtol=1e-10, atol=1e-14)


def test_spd_matches_reference(gold):
    g = gold("spd")
    for i in range(int(g["n"])):
        X = O.spd_right_solve(g[f"M{i}"], g[f"R{i}"])
        np.testing.assert_allclose(X, g[f"X{i}"], rtol=1e-7, atol=1e-9)


def test_spd_errors():
    with pytest.raises(O.NonFiniteError):
        O.spd_right_solve(np.array([[np.nan, 0.0], [0.0, 1.0]]), np.ones((1, 2)))
    with pytest.raises(O.SolveFailedError):
        O.spd_right_solve(-np.eye(3), np.ones((1, 3)))


def test_compression_matches_reference(gold):
    g = gold("compress")
    for i in range(int(g["n"])):
        lam1, lam2, it, tol = g[f"cfg{i}"]
        c = O.compress_token(g[f"q{i}"], g[f"k{i}"], g[f"B_Q{i}"], g[f"B_K{i}"], g[f"A_res{i}"],
                             g[f"K_res{i}"], lam1, lam2, int(it), tol)
        np.testing.assert_allclose(c.q_hat, g[f"q_hat{i}"], rtol=1e-9, atol=1e-10)
        np.testing.assert_allclose(c.k_hat, g[f"k_hat{i}"], rtol=1e-9, atol=1e-10)
        np.testing.assert_allclose(c.M_rq, g[f"M_rq{i}"], rtol=1e-12, atol=1e-10)
        BQ, BK, eq, ek = O.refresh_projections(g[f"q{i}"], g[f"k{i}"], c, g[f"B_Q{i}"], g[f"B_K{i}"])
        np.testing.assert_allclose(BQ, g[f"B_Q_new{i}"], rtol=1e-9, atol=1e-10)
        np.testing.assert_allclose(BK, g[f"B_K_new{i}"], rtol=1e-9, atol=1e-10)
        np.testing.assert_allclose([eq, ek], g[f"eta{i}"], rtol=1e-9)


def test_prefill_matches_reference(gold):
    g = gold("prefill")
    for i in range(int(g["n"])):
        r, it, tol = g[f"cfg{i}"]
        run = O.factorize(g[f"Q{i}"], g[f"K{i}"], rank=int(r), max_iter=int(it), tol=float(tol),
                          init=str(g[f"init{i}"]))
        assert run.sweeps == int(g[f"sweeps{i}"])
        assert run.converged == bool(g[f"conv{i}"])
        obj = np.array(run.objective)
        np.testing.assert_allclose(obj, g[f"obj{i}"], rtol=1e-7, atol=1e-9 * abs(g[f"obj{i}"][0]))
        for nm in ("A_Q", "A_K", "B_Q", "B_K"):
            want = g[f"{nm}{i}"]
            np.testing.assert_allclose(getattr(run.factors, nm), want, rtol=1e-6,
                                       atol=1e-7 * (1 + np.abs(want).max()))


def test_sessions_match_reference(gold):
    """Free-running fp64 replay of full decode sessions: selections and
    counters bit-exact, outputs and B factors to 1e-8."""
    g = gold("sessions")
    for i in range(int(g["n"])):
        prompt, r, kb, lb = (int(x) for x in g[f"cfg{i}"])
        Q, K, V = g[f"Q{i}"], g[f"K{i}"], g[f"V{i}"]
        f0 = O.Factors(g[f"A_Q0_{i}"], g[f"A_K0_{i}"], g[f"B_Q0_{i}"], g[f"B_K0_{i}"])
        # the oracle's own prefill must land on the same factors
        run = O.factorize(Q[:prompt], K[:prompt], rank=r)
        np.testing.assert_allclose(run.factors.A_K, f0.A_K, rtol=1e-6, atol=1e-8)
        st = O.seed_head(K[:prompt], V[:prompt], f0, kb, lb)
        om = g[f"omega{i}"]
        outs = g[f"out{i}"]
        for j, t in enumerate(range(prompt, Q.shape[0])):
            res = O.head_step(st, Q[t], K[t], V[t])
            want = om[j][om[j] >= 0]
            np.testing.assert_array_equal(res.omega, want)
            assert res.miss == int(g[f"miss{i}"][j])
            assert res.total == int(g[f"total{i}"][j])
            np.testing.assert_allclose(res.output.ravel(), outs[j], rtol=1e-8, atol=1e-10)
            np.testing.assert_allclose(res.k_hat.ravel(), g[f"khat{i}"][j], rtol=1e-6, atol=1e-8)
        assert (st.c_miss, st.c_total) == (int(g[f"c_miss{i}"]), int(g[f"c_total{i}"]))
        np.testing.assert_allclose(st.B_Q, g[f"BQ{i}"][-1], rtol=1e-6, atol=1e-8)


def test_dense_algebra_matches_reference(gold):
    """gram, fro_norm_sq, update_B/AK/AQ, lagrangian_value, factor_residuals,
    khat_initial_guess, update_qhat/khat (tests/golden/dense.npz)."""
    g = gold("dense")
    for i in range(int(g["n"])):
        Q, K = g[f"Q{i}"], g[f"K{i}"]
        f = O.Factors(g[f"A_Q{i}"], g[f"A_K{i}"], g[f"B_Q{i}"], g[f"B_K{i}"])
        lq, lk = g[f"lam{i}"]
        np.testing.assert_allclose(O.sym_gram(f.A_Q), g[f"gram{i}"], rtol=1e-12)
        np.testing.assert_allclose(O.sym_gram(f.B_K.T), g[f"gramT{i}"], rtol=1e-12)
        assert O.sq_norm(Q) == pytest.approx(float(g[f"fro{i}"]), rel=1e-12)
        np.testing.assert_allclose(O.fit_B(f.A_Q, Q), g[f"uB{i}"], rtol=1e-9, atol=1e-12)
        np.testing.assert_allclose(O.fit_A_K(Q, K, f, lk), g[f"uAK{i}"], rtol=1e-9, atol=1e-12)
        np.testing.assert_allclose(O.fit_A_Q(Q, K, f, lq), g[f"uAQ{i}"], rtol=1e-9, atol=1e-12)
        assert O.objective(Q, K, f, lq, lk) == pytest.approx(float(g[f"lag{i}"]), rel=1e-10)
        np.testing.assert_allclose(O.relative_residuals(Q, K, f), g[f"res{i}"], rtol=1e-9)
        q, k = g[f"q{i}"], g[f"k{i}"]
        l1, l2 = g[f"dlam{i}"]
        np.testing.assert_allclose(O.khat_seed(k, f.B_K), g[f"kh0{i}"], rtol=1e-9, atol=1e-12)
        qh, M, m = O.solve_qhat(q, k, g[f"kh_in{i}"], f.B_Q, g[f"A_res{i}"], g[f"K_res{i}"], l1, l2)
        np.testing.assert_allclose(qh, g[f"uq{i}"], rtol=1e-9, atol=1e-12)
        np.testing.assert_allclose(M, g[f"M_rq{i}"], rtol=1e-12)
        np.testing.assert_allclose(m, g[f"m_lq{i}"], rtol=1e-12)
        np.testing.assert_allclose(O.solve_khat(q, k, g[f"qh_in{i}"], f.B_K, l1), g[f"uk{i}"], rtol=1e-9,
                                   atol=1e-12)
    np.testing.assert_array_equal(O.largest_k(g["tk_s"], 37), g["tk_o"])
