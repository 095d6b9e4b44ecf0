"""CPU check of the algebra behind the K1 prefill (csrc/prefill.cu): the
reference sweep (prefill.py:197-223) restated in Gram space -- X enters only
through GX = X^T X and C0 = X^T A0 -- reproduces the reference's golden
objective trajectory, sweep count, convergence flag and factors.  This pins
the re-association itself, independently of the GPU kernels."""
import numpy as np
import pytest


def _inv_spd(M):
    # the kernel's Gauss-Jordan with the reference's single jitter retry
    r = M.shape[0]
    for jit in (0.0, 1e-10 * (np.trace(M) / r + 1.0)):
        W = M + jit * np.eye(r)
        try:
            np.linalg.cholesky(W)
        except np.linalg.LinAlgError:
            continue
        return np.linalg.inv(W)
    raise np.linalg.LinAlgError("solve failed")


def gram_space_run(Q, K, A_Q0, A_K0, lq, lk, max_iter, tol):
    l, d = Q.shape
    r = A_Q0.shape[1]
    GQ, GK = Q.T @ Q, K.T @ K
    Cq, Ck = Q.T @ A_Q0, K.T @ A_K0
    Cq0, Ck0 = Cq.copy(), Ck.copy()
    GAQ, GAK = A_Q0.T @ A_Q0, A_K0.T @ A_K0
    trq0, trk0 = np.trace(GAQ), np.trace(GAK)
    Bq, Bk = np.zeros((r, d)), np.zeros((r, d))
    Wq = Wk = None

    def objective():
        fit = max(np.sum(GQ * GK) - 2 * np.sum(Cq * Ck) + np.sum(GAQ * GAK), 0.0)
        rq = np.trace(GQ) - 2 * np.sum(Bq.T * Cq) + np.sum(GAQ * (Bq @ Bq.T))
        rk = np.trace(GK) - 2 * np.sum(Bk.T * Ck) + np.sum(GAK * (Bk @ Bk.T))
        return 0.5 * fit + 0.5 * lq * rq + 0.5 * lk * rk

    obj = [objective()]
    sweeps, conv = 0, False
    for s in range(max_iter):
        Boq, Bok = Bq, Bk
        Bq = _inv_spd(GAQ) @ Cq.T
        Bk = _inv_spd(GAK) @ Ck.T
        Wn = (Cq + lk * Bk.T) @ _inv_spd(GAQ + lk * Bk @ Bk.T)
        if s == 0:
            Ck = GK @ Wn
            dak = np.sum(Wn * (Ck - 2 * Ck0)) + trk0
        else:
            dW = Wn - Wk
            Dt = GK @ dW
            dak, Ck = np.sum(dW * Dt), Ck + Dt
        Wk = Wn
        GAK = Wk.T @ Ck
        Wn = (Ck + lq * Bq.T) @ _inv_spd(GAK + lq * Bq @ Bq.T)
        if s == 0:
            Cq = GQ @ Wn
            daq = np.sum(Wn * (Cq - 2 * Cq0)) + trq0
        else:
            dW = Wn - Wq
            Dt = GQ @ dW
            daq, Cq = np.sum(dW * Dt), Cq + Dt
        Wq = Wn
        GAQ = Wq.T @ Cq
        sweeps += 1
        obj.append(objective())
        delta = (daq / (l * r) + dak / (l * r) + np.sum((Bq - Boq) ** 2) / (r * d) +
                 np.sum((Bk - Bok) ** 2) / (r * d)) / 4
        if delta <= tol:
            conv = True
            break
    return dict(obj=np.array(obj), sweeps=sweeps, conv=conv, A_Q=Q @ Wq, A_K=K @ Wk, B_Q=Bq, B_K=Bk)


@pytest.mark.parametrize("case", [0, 1, 2, 3])
def test_gram_space_sweep_matches_reference_golden(gold, case):
    from oracle import lrqk_oracle as O

    g = gold("prefill")
    r, it, tol = g[f"cfg{case}"]
    Q, K = g[f"Q{case}"], g[f"K{case}"]
    f0 = O.initial_factors(Q, K, int(r), str(g[f"init{case}"]), 0)
    res = gram_space_run(Q, K, f0.A_Q, f0.A_K, 1.0, 1.0, int(it), float(tol))
    assert res["sweeps"] == int(g[f"sweeps{case}"])
    assert res["conv"] == bool(g[f"conv{case}"])
    np.testing.assert_allclose(res["obj"], g[f"obj{case}"], rtol=1e-7)
    for nm in ("A_Q", "A_K", "B_Q", "B_K"):
        np.testing.assert_allclose(res[nm], g[f"{nm}{case}"], rtol=1e-6, atol=1e-8 * np.abs(g[f"{nm}{case}"]).max())
