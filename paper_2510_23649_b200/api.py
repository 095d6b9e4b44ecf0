"""Drop-in mirror of the reference package's public API for the decode-time
sparse-attention path (ref: pkg/src/lrqk/__init__.py:10-82).

Same names, dataclasses, argument meaning and errors as the reference
(`NonFiniteError`, `SolveFailedError`, `ValueError`, `IndexError`,
`RuntimeError`); every numeric result is computed by the sm_100a kernels
behind include/lrqk_b200.h (fp32 storage, fp32 arithmetic), and returned as
float64 numpy arrays like the reference's.  Without the CUDA library or a
device every call raises LibraryUnavailable -- there is no CPU fallback.

Implemented entry points and the kernels behind them:
  gram, fro_norm_sq, solve_spd      -> float64 dense kernels (dense.cu)     (linalg.py:48-93)
  topk_indices, select_active       -> lrqk_topk_f64 (exact float64 order) (linalg.py:96-110, cache.py:149-171)
  update_B, update_AK, update_AQ,
  lagrangian_value, factor_residuals -> float64 dense kernels               (prefill.py:142-181, 239-253)
  prefill_run / prefill_factorize  -> float64 dense kernels, reference order (prefill.py:197-230);
                                      the engine's batched prefill is K1 (lrqk_prefill_factorize)
  init_factors, importance_scores  -> host initialisation, as the reference (prefill.py:108-139)
  khat_initial_guess, update_qhat,
  update_khat, decode_compress,
  update_projections               -> float64 dense kernels               (decode.py:79-184)
  proxy_scores                     -> lrqk_proxy_scores_f32 (K3 arithmetic) (cache.py:141-146)
  fetch_and_merge                  -> lrqk_count_misses                    (cache.py:174-196)
  exact_attention, exact_topk      -> lrqk_attention_rows / gemm + topk     (attention.py:23-41)
  DecodeSession, run_simulation    -> the fused per-layer decode step (K2-K6) (session.py:62-165)
"""

from __future__ import annotations

import csv
import ctypes as C
import math
from dataclasses import asdict, dataclass, field

import numpy as np
import torch

from . import _lib
from .engine import LayerShape, LayerState, pad_last, pow2_at_least, prefill_factorize_device
from . import dense as D
from .errors import NonFiniteError, SolveFailedError

INIT_KINDS = ("randn", "top", "topcol")
JITTER_EPS = 1e-10     # ref: linalg.py:19
ETA_DENOM_FLOOR = 1e-14  # ref: decode.py:26


def _dev():
    _lib.lib()  # raises LibraryUnavailable without a device / library
    return torch.device("cuda")


def _f32(x, dev=None):
    return torch.as_tensor(np.ascontiguousarray(x, dtype=np.float32), device=dev or _dev())


def _np64(t):
    return t.detach().double().cpu().numpy()


# ---------------------------------------------------------------------------
# validation gate (ref: linalg.py:22-45)
# ---------------------------------------------------------------------------
def as_matrix(a, name: str = "matrix") -> np.ndarray:
    out = np.ascontiguousarray(a, dtype=np.float64)
    if out.ndim != 2:
        raise ValueError(f"{name} must be 2-D, got shape {out.shape}")
    if not np.isfinite(out).all():
        raise NonFiniteError(f"{name} contains non-finite entries")
    return out


def as_row(a, name: str = "row") -> np.ndarray:
    arr = np.asarray(a, dtype=np.float64)
    if arr.ndim == 1:
        arr = arr[None, :]
    out = as_matrix(arr, name)
    if out.shape[0] != 1:
        raise ValueError(f"{name} must be a single row, got shape {out.shape}")
    return out


# ---------------------------------------------------------------------------
# dense kernels (ref: linalg.py:48-93), float64 on the device (dense.cu)
# ---------------------------------------------------------------------------
def gram(A) -> np.ndarray:
    """A^T A, exactly symmetric (ref: linalg.py:48-55)."""
    A = np.asarray(A, dtype=np.float64)
    if A.size == 0:
        raise ValueError("gram requires a nonempty matrix")
    return D.np64(D.gram(D.t64(A)))


def fro_norm_sq(A) -> float:
    """Sum of squared entries (ref: linalg.py:58-60)."""
    a = D.t64(np.asarray(A, dtype=np.float64).ravel())
    if a.numel() == 0:
        return 0.0
    return float(D.dot(a, a).item())


def solve_spd(M, RHS) -> np.ndarray:
    """X with X M = RHS, Cholesky with one jittered retry (ref: linalg.py:63-93)."""
    M = np.asarray(M, dtype=np.float64)
    RHS = np.asarray(RHS, dtype=np.float64)
    r = M.shape[0]
    if M.ndim != 2 or M.shape[1] != r or RHS.ndim != 2 or RHS.shape[1] != r:
        # the reference validates finiteness before shapes (linalg.py:71-78)
        if not np.isfinite(M).all():
            raise NonFiniteError("solve_spd: M contains non-finite entries")
        if not np.isfinite(RHS).all():
            raise NonFiniteError("solve_spd: RHS contains non-finite entries")
        if M.ndim != 2 or M.shape[1] != r:
            raise ValueError(f"M must be square, got {M.shape}")
        raise ValueError(f"RHS has {RHS.shape[1] if RHS.ndim == 2 else RHS.shape} cols, expected {r}")
    return D.np64(D.solve_spd(D.t64(M), D.t64(RHS)))


# ---------------------------------------------------------------------------
# selection (ref: linalg.py:96-110, cache.py:149-171)
# ---------------------------------------------------------------------------
def _select_device(scores_2d: torch.Tensor, t: int, k_budget: int, lite_budget: int):
    """scores_2d [H, t+1] f32 on device -> (omega [H, s_cap] int32, counts [H])."""
    lib = _lib.lib()
    H = scores_2d.shape[0]
    ws_bytes = lib.lrqk_select_scores_workspace(H, t, k_budget, lite_budget)
    ws = torch.empty(max(256, ws_bytes), dtype=torch.uint8, device=scores_2d.device)
    omega = torch.empty(H, k_budget + lite_budget, dtype=torch.int32, device=scores_2d.device)
    cnt = torch.empty(H, dtype=torch.int32, device=scores_2d.device)
    _lib.check(lib.lrqk_select_scores(scores_2d.data_ptr(), H, t, k_budget, lite_budget, omega.data_ptr(),
                                      cnt.data_ptr(), ws.data_ptr(), ws_bytes, _lib.stream_ptr()),
               "lrqk_select_scores")
    return omega, cnt


def topk_indices(scores, k: int) -> np.ndarray:
    """Indices of the k largest scores, ascending; ties toward the lower index
    (ref: linalg.py:96-110).  Selected on the device over order-preserving
    64-bit keys of the float64 scores, so the order is the reference's."""
    if k < 1:
        raise ValueError(f"k must be >= 1, got {k}")
    s = np.asarray(scores, dtype=np.float64).ravel()
    n = s.shape[0]
    if k >= n:
        return np.arange(n)
    return D.topk(D.t64(s), k).cpu().numpy().astype(np.int64)


@dataclass
class SelectionSet:
    omega_k: np.ndarray
    omega_l: np.ndarray
    omega: np.ndarray


def select_active(scores, t: int, k_budget: int, lite_budget: int) -> SelectionSet:
    """ref: cache.py:149-171 -- lite window [max(0, t+1-lite), t] plus the
    top-k (float64 order, device select) of the scores before it."""
    s = np.asarray(scores, dtype=np.float64).ravel()
    if s.shape[0] != t + 1:
        raise ValueError(f"scores must cover tokens 0..{t}, got {s.shape[0]}")
    lite_start = max(0, t + 1 - lite_budget)
    omega_l = np.arange(lite_start, t + 1)
    if lite_start == 0:
        omega_k = np.arange(0)
    else:
        omega_k = topk_indices(s[:lite_start], min(k_budget, lite_start))
    return SelectionSet(omega_k=omega_k.astype(np.intp), omega_l=omega_l,
                        omega=np.concatenate([omega_k, omega_l]).astype(np.intp))


# ---------------------------------------------------------------------------
# proxy scores (ref: cache.py:141-146)
# ---------------------------------------------------------------------------
def proxy_scores(q_hat, proxy_store) -> np.ndarray:
    store = np.asarray(proxy_store, dtype=np.float64)
    qh = np.asarray(q_hat, dtype=np.float64).reshape(1, -1)
    t, r = store.shape
    if t == 0:
        return np.zeros(0)
    dev = _dev()
    rs = pow2_at_least(r)
    st = pad_last(_f32(store, dev), rs).contiguous()
    q = pad_last(_f32(qh, dev), rs).contiguous()
    out = torch.empty(t, dtype=torch.float32, device=dev)
    _lib.check(_lib.lib().lrqk_proxy_scores_f32(st.data_ptr(), _lib.F32, q.data_ptr(), out.data_ptr(), 1, t, rs,
                                                 _lib.stream_ptr()), "lrqk_proxy_scores_f32")
    return _np64(out)


# ---------------------------------------------------------------------------
# attention (ref: attention.py:23-50)
# ---------------------------------------------------------------------------
@dataclass
class AttentionResult:
    output: np.ndarray
    weights: np.ndarray


def _attention_device(q: torch.Tensor, K: torch.Tensor, V: torch.Tensor, d: int, want_weights=True):
    H, n, ld = K.shape
    out = torch.empty(H, ld, dtype=torch.float32, device=K.device)
    w = torch.empty(H, n, dtype=torch.float32, device=K.device) if want_weights else None
    _lib.check(_lib.lib().lrqk_attention_rows(q.data_ptr(), K.data_ptr(), V.data_ptr(), H, n, d, ld, out.data_ptr(),
                                               w.data_ptr() if w is not None else None, _lib.stream_ptr()),
               "lrqk_attention_rows")
    return out, w


def exact_attention(q, K, V) -> AttentionResult:
    K = np.asarray(K, dtype=np.float64)
    V = np.asarray(V, dtype=np.float64)
    n, d = K.shape
    if n == 0:
        raise ValueError("exact_attention requires at least one key")
    if V.shape[0] != n:
        raise ValueError(f"K has {n} rows but V has {V.shape[0]}")
    dev = _dev()
    out, w = _attention_device(_f32(np.asarray(q).reshape(1, d), dev), _f32(K[None], dev), _f32(V[None], dev), d)
    return AttentionResult(output=_np64(out[:, :d]), weights=_np64(w[0]))


def _exact_topk_dev(q64: torch.Tensor, K64: torch.Tensor, k: int) -> np.ndarray:
    """Top-k of raw q K^T (float64 GEMM + float64 select on the device)."""
    n = K64.shape[0]
    if k >= n:
        return np.arange(n)
    s = D.gemm(K64, q64, tb=True).reshape(-1)
    return D.topk(s, k).cpu().numpy().astype(np.int64)


def exact_topk(q, K, k: int) -> np.ndarray:
    """ref: attention.py:37-41."""
    K = np.asarray(K, dtype=np.float64)
    if K.shape[0] == 0:
        raise ValueError("exact_topk requires at least one key")
    if k < 1:
        raise ValueError(f"k must be >= 1, got {k}")
    return _exact_topk_dev(D.t64(np.asarray(q).reshape(1, -1)), D.t64(K), k)


def selection_recall(proxy, exact) -> float:
    exact = set(int(i) for i in exact)
    if not exact:
        raise ValueError("selection_recall undefined for an empty exact set")
    proxy = set(int(i) for i in proxy)
    return len(proxy & exact) / len(exact)


# ---------------------------------------------------------------------------
# prefill (ref: prefill.py)
# ---------------------------------------------------------------------------
@dataclass(frozen=True)
class InitStrategy:
    kind: str = "randn"
    seed: int = 0

    def __post_init__(self):
        if self.kind not in INIT_KINDS:
            raise ValueError(f"init kind must be one of {INIT_KINDS}, got {self.kind!r}")


@dataclass(frozen=True)
class PrefillConfig:
    rank: int = 32
    lambda_q: float = 1.0
    lambda_k: float = 1.0
    max_iter: int = 2
    tol: float = 1e-2
    init: InitStrategy = field(default_factory=InitStrategy)

    def __post_init__(self):
        if self.rank < 1:
            raise ValueError(f"rank must be >= 1, got {self.rank}")
        if self.lambda_q < 0 or self.lambda_k < 0:
            raise ValueError("lambda_q and lambda_k must be >= 0")
        if self.max_iter < 1:
            raise ValueError(f"max_iter must be >= 1, got {self.max_iter}")
        if self.tol <= 0:
            raise ValueError(f"tol must be > 0, got {self.tol}")


@dataclass
class LowRankFactors:
    A_Q: np.ndarray
    A_K: np.ndarray
    B_Q: np.ndarray
    B_K: np.ndarray

    @property
    def rank(self) -> int:
        return self.A_Q.shape[1]

    def copy(self) -> "LowRankFactors":
        return LowRankFactors(self.A_Q.copy(), self.A_K.copy(), self.B_Q.copy(), self.B_K.copy())


@dataclass(frozen=True)
class ImportanceScores:
    s_q: np.ndarray
    s_k: np.ndarray
    s_qk: np.ndarray


@dataclass
class PrefillRun:
    factors: LowRankFactors
    objective: list
    sweeps: int
    converged: bool


def importance_scores(Q, K) -> ImportanceScores:
    """ref: prefill.py:108-113 (host-side initialisation helper)."""
    Q, K = np.asarray(Q, dtype=np.float64), np.asarray(K, dtype=np.float64)
    if Q.shape != K.shape:
        raise ValueError(f"Q and K must share a shape, got {Q.shape} vs {K.shape}")
    s_q = np.abs(Q).sum(axis=0)
    s_k = np.abs(K).sum(axis=0)
    return ImportanceScores(s_q=s_q, s_k=s_k, s_qk=s_q + s_k)


def _host_topk(scores, k):
    s = np.asarray(scores, dtype=np.float64)
    if k >= s.size:
        return np.arange(s.size)
    return np.sort(np.lexsort((np.arange(s.size), -s))[:k])


def init_factors(Q, K, cfg: PrefillConfig) -> LowRankFactors:
    """Initial A_Q, A_K (ref: prefill.py:116-139).  Like the reference this
    runs on the host: a PCG64 draw or a column pick, uploaded once."""
    Q, K = np.asarray(Q, dtype=np.float64), np.asarray(K, dtype=np.float64)
    if Q.shape != K.shape:
        raise ValueError(f"Q and K must share a shape, got {Q.shape} vs {K.shape}")
    l, d = Q.shape
    r = cfg.rank
    if r > d:
        raise ValueError(f"rank {r} exceeds head dimension {d}")
    if cfg.init.kind == "randn":
        rng = np.random.default_rng(cfg.init.seed)
        A_Q = rng.standard_normal((l, r))
        A_K = rng.standard_normal((l, r))
    else:
        sc = importance_scores(Q, K)
        if cfg.init.kind == "top":
            A_Q = Q[:, _host_topk(sc.s_q, r)].copy()
            A_K = K[:, _host_topk(sc.s_k, r)].copy()
        else:
            cols = _host_topk(sc.s_qk, r)
            A_Q, A_K = Q[:, cols].copy(), K[:, cols].copy()
    return LowRankFactors(A_Q=A_Q, A_K=A_K, B_Q=np.zeros((r, d)), B_K=np.zeros((r, d)))


def _factor_sweep_f64(Qd, Kd, f, cfg):
    """One BCD sweep B_Q, B_K, A_K, A_Q in the reference's association
    (prefill.py:211-214), float64 device tensors in f (dict)."""
    def update_b(A, X):
        return D.solve_spd(D.gram(A), D.gemm(X, A, ta=True)).t().contiguous()

    def update_a(Xo, Xs, Ao, Bs, lam):
        T = D.gemm(Xo, Ao, ta=True)
        D.axpby(lam, Bs.t().contiguous(), 1.0, T)
        M = D.gram(Ao)
        D.axpby(lam, D.gram(Bs, of_transpose=True), 1.0, M)
        return D.solve_spd(M, D.gemm(Xs, T))

    f["B_Q"] = update_b(f["A_Q"], Qd)
    f["B_K"] = update_b(f["A_K"], Kd)
    f["A_K"] = update_a(Qd, Kd, f["A_Q"], f["B_K"], cfg.lambda_k)
    f["A_Q"] = update_a(Kd, Qd, f["A_K"], f["B_Q"], cfg.lambda_q)


def _objective_f64(Qd, Kd, f, cfg):
    """lagrangian_value on device factors (prefill.py:142-158)."""
    GQ, GK = D.gram(Qd), D.gram(Kd)
    qq = D.dot(GQ, GK)
    cross = D.dot(D.gemm(Qd, f["A_Q"], ta=True), D.gemm(Kd, f["A_K"], ta=True))
    approx = D.dot(D.gram(f["A_Q"]), D.gram(f["A_K"]))
    rq = D.residual_sq(Qd, f["A_Q"], f["B_Q"])
    rk = D.residual_sq(Kd, f["A_K"], f["B_K"])
    qq, cross, approx, rq, rk = (float(x.item()) for x in (qq, cross, approx, rq, rk))
    return 0.5 * max(qq - 2.0 * cross + approx, 0.0) + 0.5 * cfg.lambda_q * rq + 0.5 * cfg.lambda_k * rk


def prefill_run(Q, K, cfg: PrefillConfig) -> PrefillRun:
    """The alternating sweeps with the objective trajectory and the
    mean-squared-change stop (ref: prefill.py:197-223), in float64 on the
    device, so sweeps / converged / objective follow the reference's to
    rounding.  The batched bf16 / fp32 engine prefill is the fused K1 pass
    (engine.prefill_factorize_device)."""
    Q = as_matrix(Q, "Q")
    K = as_matrix(K, "K")
    if Q.shape != K.shape:
        raise ValueError(f"Q and K must share a shape, got {Q.shape} vs {K.shape}")
    f0 = init_factors(Q, K, cfg)
    Qd, Kd = D.t64(Q), D.t64(K)
    f = {nm: D.t64(getattr(f0, nm)) for nm in ("A_Q", "A_K", "B_Q", "B_K")}
    objective = [_objective_f64(Qd, Kd, f, cfg)]
    converged, sweeps = False, 0
    for _ in range(cfg.max_iter):
        prev = {nm: t.clone() for nm, t in f.items()}
        _factor_sweep_f64(Qd, Kd, f, cfg)
        sweeps += 1
        for nm in ("A_Q", "A_K", "B_Q", "B_K"):
            if not math.isfinite(float(D.dot(f[nm], f[nm]).item())):
                raise NonFiniteError(f"factor {nm} diverged at sweep {sweeps}")
        objective.append(_objective_f64(Qd, Kd, f, cfg))
        delta = 0.0
        for nm in ("A_Q", "A_K", "B_Q", "B_K"):
            diff = D.axpby(-1.0, prev[nm], 1.0, f[nm].clone())
            delta += float(D.dot(diff, diff).item()) / diff.numel()
        if delta / 4.0 <= cfg.tol:
            converged = True
            break
    fac = LowRankFactors(**{nm: D.np64(t) for nm, t in f.items()})
    return PrefillRun(factors=fac, objective=objective, sweeps=sweeps, converged=converged)


def prefill_factorize(Q, K, cfg: PrefillConfig) -> LowRankFactors:
    return prefill_run(Q, K, cfg).factors


# The per-call prefill algebra of the reference, float64 on the device.  The
# fused K1 pass (prefill_run above) computes the same quantities re-associated
# in one stream over Q and K per sweep; these are the reference's individual
# entry points with its exact association (prefill.py:142-181, 239-253).
def _lagrangian_terms(Qd, Kd, f):
    """Device scalars: sum(GQ o GK), cross, approx (ref: prefill.py:150-153)."""
    GQ, GK = D.gram(Qd), D.gram(Kd)
    AQ, AK = D.t64(f.A_Q), D.t64(f.A_K)
    CQ, CK = D.gemm(Qd, AQ, ta=True), D.gemm(Kd, AK, ta=True)
    return D.dot(GQ, GK), D.dot(CQ, CK), D.dot(D.gram(AQ), D.gram(AK)), AQ, AK


def lagrangian_value(Q, K, f: LowRankFactors, cfg: PrefillConfig) -> float:
    """Objective through d x d / r x r Gram traces (ref: prefill.py:142-158)."""
    Q, K = np.asarray(Q, dtype=np.float64), np.asarray(K, dtype=np.float64)
    Qd, Kd = D.t64(Q), D.t64(K)
    qq, cross, approx, AQ, AK = _lagrangian_terms(Qd, Kd, f)
    rq = D.residual_sq(Qd, AQ, D.t64(f.B_Q))
    rk = D.residual_sq(Kd, AK, D.t64(f.B_K))
    qq, cross, approx, rq, rk = (float(x.item()) for x in (qq, cross, approx, rq, rk))
    qk_term = max(qq - 2.0 * cross + approx, 0.0)
    return 0.5 * qk_term + 0.5 * cfg.lambda_q * rq + 0.5 * cfg.lambda_k * rk


def update_B(A, X) -> np.ndarray:
    """B = (A^T A)^-1 A^T X (ref: prefill.py:161-163)."""
    Ad, Xd = D.t64(A), D.t64(X)
    return D.np64(D.solve_spd(D.gram(Ad), D.gemm(Xd, Ad, ta=True))).T.copy()


def _update_A(X_other, X_self, A_other, B_self, lam):
    """X_self (X_other^T A_other + lam B_self^T) (gram(A_other) + lam gram(B_self^T))^-1."""
    Xo, Xs, Ao = D.t64(X_other), D.t64(X_self), D.t64(A_other)
    BT = D.t64(np.ascontiguousarray(np.asarray(B_self, dtype=np.float64).T))
    T = D.gemm(Xo, Ao, ta=True)
    D.axpby(lam, BT, 1.0, T)
    rhs = D.gemm(Xs, T)
    M = D.gram(Ao)
    D.axpby(lam, D.gram(BT), 1.0, M)
    return D.np64(D.solve_spd(M, rhs))


def update_AK(Q, K, f: LowRankFactors, cfg: PrefillConfig) -> np.ndarray:
    """Closed-form A_K (ref: prefill.py:166-172)."""
    return _update_A(Q, K, f.A_Q, f.B_K, cfg.lambda_k)


def update_AQ(Q, K, f: LowRankFactors, cfg: PrefillConfig) -> np.ndarray:
    """Closed-form A_Q (ref: prefill.py:175-181)."""
    return _update_A(K, Q, f.A_K, f.B_Q, cfg.lambda_q)


def _rel(num_sq: float, den_sq: float) -> float:
    if den_sq == 0.0:
        return 0.0 if num_sq == 0.0 else float("inf")
    return float(np.sqrt(num_sq / den_sq))


def factor_residuals(Q, K, f: LowRankFactors) -> tuple:
    """Relative reconstruction errors of Q, K and Q K^T (ref: prefill.py:239-253)."""
    Q, K = np.asarray(Q, dtype=np.float64), np.asarray(K, dtype=np.float64)
    Qd, Kd = D.t64(Q), D.t64(K)
    den, cross, approx, AQ, AK = _lagrangian_terms(Qd, Kd, f)
    rq = D.residual_sq(Qd, AQ, D.t64(f.B_Q))
    rk = D.residual_sq(Kd, AK, D.t64(f.B_K))
    q2, k2 = D.dot(Qd, Qd), D.dot(Kd, Kd)
    den, cross, approx, rq, rk, q2, k2 = (float(x.item()) for x in (den, cross, approx, rq, rk, q2, k2))
    return _rel(rq, q2), _rel(rk, k2), _rel(max(den - 2.0 * cross + approx, 0.0), den)


# ---------------------------------------------------------------------------
# decode compression (ref: decode.py)
# ---------------------------------------------------------------------------
@dataclass(frozen=True)
class DecodeConfig:
    lambda_1: float = 1.0
    lambda_2: float = 1.0
    max_iter: int = 2
    tol: float = 1e-2

    def __post_init__(self):
        if self.lambda_1 < 0 or self.lambda_2 < 0:
            raise ValueError("lambda_1 and lambda_2 must be >= 0")
        if self.max_iter < 1:
            raise ValueError(f"max_iter must be >= 1, got {self.max_iter}")
        if self.tol <= 0:
            raise ValueError(f"tol must be > 0, got {self.tol}")


@dataclass(frozen=True)
class TokenStep:
    q: np.ndarray
    k: np.ndarray
    v: np.ndarray

    def __post_init__(self):
        if not (self.q.shape == self.k.shape == self.v.shape):
            raise ValueError("q, k, v must share the same 1 x d shape")


@dataclass
class CompressedToken:
    q_hat: np.ndarray
    k_hat: np.ndarray


@dataclass
class DecodeWorkspace:
    """Intermediates of the last step: the q-side normal system (m_lq, M_rq),
    the B gradients and the line-search step sizes (ref: decode.py:66-76)."""

    m_lq: np.ndarray | None = None
    M_rq: np.ndarray | None = None
    grad_BQ: np.ndarray | None = None
    grad_BK: np.ndarray | None = None
    eta_Q: float = 0.0
    eta_K: float = 0.0


def khat_initial_guess(k, B_K) -> np.ndarray:
    """Least-squares k in the row space of B_K (ref: decode.py:79-81)."""
    B = D.t64(np.ascontiguousarray(np.asarray(B_K, dtype=np.float64)))
    kd = D.t64(np.asarray(k, dtype=np.float64).reshape(1, -1))
    return D.np64(D.solve_spd(D.gram(B, of_transpose=True), D.gemm(kd, B, tb=True)))


def _qk(step: TokenStep):
    qd = D.t64(step.q.reshape(1, -1))
    kd = D.t64(step.k.reshape(1, -1))
    return qd, kd, D.dot(qd, kd)


def update_qhat(step: TokenStep, comp: CompressedToken, f: LowRankFactors, A_K_resident, K_resident,
                cfg: DecodeConfig, ws: DecodeWorkspace) -> np.ndarray:
    """Closed-form q_hat given k_hat (ref: decode.py:84-108); fills ws.m_lq, ws.M_rq."""
    A_res = np.asarray(A_K_resident, dtype=np.float64)
    K_res = np.asarray(K_resident, dtype=np.float64)
    if A_res.shape[0] != K_res.shape[0]:
        raise ValueError(f"resident proxy/key row counts differ: {A_res.shape[0]} vs {K_res.shape[0]}")
    qd, kd, qk = _qk(step)
    BQ = D.t64(f.B_Q)
    kh = D.t64(np.asarray(comp.k_hat, dtype=np.float64).reshape(1, -1))
    m_lq = D.gemm(qd, BQ, tb=True)
    D.axpby(cfg.lambda_1, kh, 1.0, m_lq, scale=qk)
    M_rq = D.gram(BQ, of_transpose=True)
    D.gemm(kh, kh, ta=True, alpha=cfg.lambda_1, beta=1.0, out=M_rq)
    if A_res.shape[0] > 0:
        Ad, Kd = D.t64(A_res), D.t64(K_res)
        w = D.gemm(qd, Kd, tb=True)
        D.gemm(w, Ad, alpha=cfg.lambda_2, beta=1.0, out=m_lq)
        D.axpby(cfg.lambda_2, D.gram(Ad), 1.0, M_rq)
    ws.m_lq, ws.M_rq = D.np64(m_lq), D.np64(M_rq)
    return D.np64(D.solve_spd(M_rq, m_lq))


def update_khat(step: TokenStep, comp: CompressedToken, f: LowRankFactors, cfg: DecodeConfig) -> np.ndarray:
    """Closed-form k_hat given q_hat (ref: decode.py:111-119)."""
    qd, kd, qk = _qk(step)
    BK = D.t64(f.B_K)
    qh = D.t64(np.asarray(comp.q_hat, dtype=np.float64).reshape(1, -1))
    rhs = D.gemm(kd, BK, tb=True)
    D.axpby(cfg.lambda_1, qh, 1.0, rhs, scale=qk)
    M = D.gram(BK, of_transpose=True)
    D.gemm(qh, qh, ta=True, alpha=cfg.lambda_1, beta=1.0, out=M)
    return D.np64(D.solve_spd(M, rhs))


def decode_compress(step: TokenStep, f: LowRankFactors, A_K_resident, K_resident, cfg: DecodeConfig):
    """k_hat guess, then alternating q_hat / k_hat solves with the mean
    squared change stop (ref: decode.py:122-147), float64 on the device.
    The fused fp32 compression of the decode step (compress.cu, K2) is what
    DecodeSession / Engine run."""
    ws = DecodeWorkspace()
    r = f.B_Q.shape[0]
    comp = CompressedToken(q_hat=np.zeros((1, r)), k_hat=khat_initial_guess(step.k, f.B_K))
    prev = None
    for _ in range(cfg.max_iter):
        comp.q_hat = update_qhat(step, comp, f, A_K_resident, K_resident, cfg, ws)
        comp.k_hat = update_khat(step, comp, f, cfg)
        cur = np.concatenate([comp.q_hat, comp.k_hat], axis=1)
        if prev is not None and fro_norm_sq(cur - prev) / cur.size <= cfg.tol:
            break
        prev = cur
    return comp, ws


def _line_search_step(row_hat, B, target):
    """Gradient and exact step (ref: decode.py:150-166): grad = x^T (x B - t),
    eta = (resid . s) / (s . s), s = x grad, 0 under the floor."""
    xd = D.t64(np.asarray(row_hat, dtype=np.float64).reshape(1, -1))
    Bd = D.t64(B)
    resid = D.t64(np.asarray(target, dtype=np.float64).reshape(1, -1))
    D.gemm(xd, Bd, beta=-1.0, out=resid)
    grad = D.gemm(xd, resid, ta=True)
    sv = D.gemm(xd, grad)
    denom, numer = float(D.dot(sv, sv).item()), float(D.dot(resid, sv).item())
    if denom <= ETA_DENOM_FLOOR * (1.0 + abs(numer)):
        return grad, Bd, 0.0
    return grad, Bd, numer / denom


def update_projections(step: TokenStep, comp: CompressedToken, f: LowRankFactors, ws: DecodeWorkspace):
    """One exact line-search step on B_Q, B_K (ref: decode.py:169-184); A
    factors pass through."""
    gq, BQ, ws.eta_Q = _line_search_step(comp.q_hat, f.B_Q, step.q)
    gk, BK, ws.eta_K = _line_search_step(comp.k_hat, f.B_K, step.k)
    ws.grad_BQ, ws.grad_BK = D.np64(gq), D.np64(gk)
    D.axpby(-ws.eta_Q, gq, 1.0, BQ)
    D.axpby(-ws.eta_K, gk, 1.0, BK)
    return LowRankFactors(A_Q=f.A_Q, A_K=f.A_K, B_Q=D.np64(BQ), B_K=D.np64(BK))


# ---------------------------------------------------------------------------
# cache manager (ref: cache.py)
# ---------------------------------------------------------------------------
@dataclass
class CacheStats:
    c_miss: int = 0
    c_total: int = 0
    per_step: list = field(default_factory=list)

    def record(self, step: int, miss_count: int, selected_count: int) -> None:
        self.c_miss += miss_count
        self.c_total += selected_count
        self.per_step.append((step, miss_count, selected_count))


def miss_rate(stats: CacheStats) -> float:
    if stats.c_total == 0:
        raise ValueError("miss rate undefined: no selections recorded")
    return stats.c_miss / stats.c_total


class TieredKVCache:
    """One head's tiered cache: slow tier K/V and the proxy store live on the
    device; `fast_resident` is the fast-tier index set (ref: cache.py:84-138)."""

    def __init__(self, dim: int, rank: int, k_budget: int, lite_budget: int):
        if k_budget < 1 or lite_budget < 1:
            raise ValueError("k_budget and lite_budget must be >= 1")
        self.dim, self.rank, self.k_budget, self.lite_budget = dim, rank, k_budget, lite_budget
        self._dev = _dev()
        self._K = torch.zeros(16, dim, dtype=torch.float32, device=self._dev)
        self._V = torch.zeros(16, dim, dtype=torch.float32, device=self._dev)
        self._P = torch.zeros(16, rank, dtype=torch.float32, device=self._dev)
        self._n = 0
        self.fast_resident: set[int] = set()

    def _grow(self, need):
        cap = self._K.shape[0]
        if need <= cap:
            return
        while cap < need:
            cap *= 2
        for nm in ("_K", "_V", "_P"):
            old = getattr(self, nm)
            new = torch.zeros(cap, old.shape[1], dtype=old.dtype, device=old.device)
            new[: self._n] = old[: self._n]
            setattr(self, nm, new)

    def _extend(self, K, V, P):
        n = K.shape[0]
        self._grow(self._n + n)
        self._K[self._n: self._n + n] = _f32(K, self._dev)
        self._V[self._n: self._n + n] = _f32(V, self._dev)
        self._P[self._n: self._n + n] = _f32(P, self._dev)
        self._n += n

    @property
    def size(self) -> int:
        return self._n

    @property
    def proxy_store(self) -> np.ndarray:
        v = _np64(self._P[: self._n])
        v.flags.writeable = False
        return v

    def seed_prompt(self, K, V, A_K) -> None:
        if not (K.shape[0] == V.shape[0] == A_K.shape[0]):
            raise ValueError("prompt K, V, and proxy row counts must match")
        self._extend(np.asarray(K), np.asarray(V), np.asarray(A_K))
        start = max(0, self.size - self.lite_budget)
        self.fast_resident = set(range(start, self.size))

    def resident_rows(self):
        idx = np.array(sorted(self.fast_resident), dtype=np.intp)
        it = torch.as_tensor(idx, dtype=torch.long, device=self._dev)
        return idx, _np64(self._P[it]), _np64(self._K[it])

    def slow_rows(self, indices):
        it = torch.as_tensor(np.asarray(indices, dtype=np.int64), device=self._dev)
        return _np64(self._K[it]), _np64(self._V[it])

    def full_history(self):
        K, V = _np64(self._K[: self._n]), _np64(self._V[: self._n])
        K.flags.writeable = False
        V.flags.writeable = False
        return K, V


def append_token(cache: TieredKVCache, k, v, k_hat) -> int:
    """ref: cache.py:199-214."""
    t = cache.size
    cache._extend(np.asarray(k).reshape(1, -1), np.asarray(v).reshape(1, -1), np.asarray(k_hat).reshape(1, -1))
    cache.fast_resident.add(t)
    return t


def fetch_and_merge(cache: TieredKVCache, sel: SelectionSet, stats: CacheStats):
    """ref: cache.py:174-196 (miss counting by lrqk_count_misses)."""
    dev = cache._dev
    omega = np.unique(np.asarray(sel.omega, dtype=np.int64))
    res = np.array(sorted(cache.fast_resident), dtype=np.int32)
    out = torch.zeros(3, dtype=torch.int32, device=dev)
    om_t = torch.as_tensor(omega.astype(np.int32), device=dev)
    res_t = torch.as_tensor(res, device=dev) if res.size else torch.zeros(1, dtype=torch.int32, device=dev)
    _lib.check(_lib.lib().lrqk_count_misses(res_t.data_ptr(), int(res.size), om_t.data_ptr(), int(omega.size),
                                             cache.size, out.data_ptr(), _lib.stream_ptr()), "lrqk_count_misses")
    miss, total, bad = (int(x) for x in out.cpu())
    if bad:
        lo, hi = int(omega.min()), int(omega.max())
        raise IndexError(f"selection references token {hi if hi >= cache.size else lo}, "
                         f"valid range is 0..{cache.size - 1}")
    stats.record(step=cache.size - 1, miss_count=miss, selected_count=total)
    K, V = cache.slow_rows(np.sort(np.asarray(sel.omega)))
    cache.fast_resident = set(int(i) for i in omega)
    return K, V


def write_stats_csv(path, stats: CacheStats) -> None:
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["step", "selected", "miss", "hit", "miss_rate"])
        for step, miss, selected in stats.per_step:
            w.writerow([step, selected, miss, selected - miss, repr(miss / selected if selected else 0.0)])


# ---------------------------------------------------------------------------
# session (ref: session.py)
# ---------------------------------------------------------------------------
@dataclass(frozen=True)
class SessionConfig:
    prefill: PrefillConfig = field(default_factory=PrefillConfig)
    decode: DecodeConfig = field(default_factory=DecodeConfig)
    k_budget: int = 2048
    lite_budget: int = 64

    def __post_init__(self):
        if self.k_budget < 1 or self.lite_budget < 1:
            raise ValueError("k_budget and lite_budget must be >= 1")


@dataclass
class StepReport:
    step: int
    selected_count: int
    miss_count: int
    recall_vs_exact: float
    output_err: float


@dataclass
class SimulationResult:
    reports: list
    stats: CacheStats
    session: "DecodeSession"


class _SessionCacheView:
    """Read-only view of a session's device cache with the reference's
    TieredKVCache accessors (size, proxy_store, fast_resident, ...)."""

    def __init__(self, session: "DecodeSession"):
        self._s = session

    @property
    def size(self) -> int:
        return self._s._t

    @property
    def proxy_store(self) -> np.ndarray:
        L = self._s._layer
        v = _np64(L.proxy_rows()[0, 0, : self.size, : L.shape.rank])
        v.flags.writeable = False
        return v

    @property
    def fast_resident(self) -> set:
        L = self._s._layer
        n = int(L.view("res_cnt")[0, 0])
        return set(int(i) for i in L.view("res_idx")[0, 0, :n].cpu())

    def resident_rows(self):
        idx = np.array(sorted(self.fast_resident), dtype=np.intp)
        P = self.proxy_store
        K, _ = self.full_history()
        return idx, P[idx], K[idx]

    def slow_rows(self, indices):
        K, V = self.full_history()
        return K[indices], V[indices]

    def full_history(self):
        L = self._s._layer
        d = L.shape.head_dim
        K = _np64(L.view("slow_k")[0, 0, : self.size, :d])
        V = _np64(L.view("slow_v")[0, 0, : self.size, :d])
        return K, V


class DecodeSession:
    """One head's lifecycle on the GPU: prefill once, then step tokens
    (ref: session.py:62-131)."""

    def __init__(self, cfg: SessionConfig):
        self.cfg = cfg
        self.factors: LowRankFactors | None = None
        self.cache = None
        self.stats = CacheStats()
        self.last_selection: SelectionSet | None = None
        self.last_output: np.ndarray | None = None
        self._layer = None
        self._t = 0

    def _alloc(self, t_max):
        c = self.cfg
        d = self._d
        shape = LayerShape(batch=1, n_q_heads=1, n_kv_heads=1, head_dim=d, rank=c.prefill.rank,
                           k_budget=c.k_budget, lite_budget=c.lite_budget, t_max=t_max, dtype="f32")
        return LayerState(shape, lambda_1=c.decode.lambda_1, lambda_2=c.decode.lambda_2,
                          max_iter=c.decode.max_iter, tol=c.decode.tol)

    def prefill(self, Q, K, V) -> LowRankFactors:
        Q = as_matrix(Q, "Q")
        K = as_matrix(K, "K")
        V = as_matrix(V, "V")
        if not (Q.shape == K.shape == V.shape):
            raise ValueError("prompt Q, K, V must share one l x d shape")
        run = prefill_run(Q, K, self.cfg.prefill)
        self.factors = run.factors
        l, self._d = Q.shape
        self._layer = self._alloc(max(2 * l, l + 256))
        dev = self._layer.device
        self._layer.load_prompt(_f32(self.factors.A_K[None, None], dev), _f32(self.factors.B_Q[None, None], dev),
                                _f32(self.factors.B_K[None, None], dev), _f32(K[None, None], dev),
                                _f32(V[None, None], dev))
        self._t = l
        self.cache = _SessionCacheView(self)
        return self.factors

    def _regrow(self):
        """Double the store capacity (the reference's _RowStore growth)."""
        old = self._layer
        new = self._alloc(2 * old.shape.t_max)
        t = self._t
        for nm in ("B_Q", "B_K", "res_idx", "res_cnt", "c_miss", "c_total", "ctx_len", "sel_meta"):
            new.view(nm).copy_(old.view(nm))
        # the residency bitmap of Omega_{t-1}: the next step's hit/miss count
        # reads it (compress.cu count_hits_hbm); its per-head stride grows
        ow = old.view("res_bits").shape[-1]
        new.view("res_bits")[..., :ow].copy_(old.view("res_bits"))
        new.view("slow_k")[:, :, :t].copy_(old.view("slow_k")[:, :, :t])
        new.view("slow_v")[:, :, :t].copy_(old.view("slow_v")[:, :, :t])
        tl = (t + 31) // 32
        new.proxy_tiles()[:, :, :tl].copy_(old.proxy_tiles()[:, :, :tl])
        if old.shape.row_mirror:
            new.view("proxy_rowmajor")[:, :, :t].copy_(old.view("proxy_rowmajor")[:, :, :t])
        new.buf["pre"].copy_(old.buf["pre"])
        self._layer = new

    def decode_step(self, q, k, v, compute_metrics: bool = True) -> StepReport:
        if self.factors is None or self._layer is None:
            raise RuntimeError("decode_step called before prefill")
        step = TokenStep(q=as_row(q, "q"), k=as_row(k, "k"), v=as_row(v, "v"))
        if self._t + 1 >= self._layer.shape.t_max:
            self._regrow()
        L = self._layer
        dev = L.device
        ds = L.shape.dim_stride
        qd = pad_last(_f32(step.q, dev), ds).contiguous()
        kd = pad_last(_f32(step.k, dev), ds).contiguous()
        vd = pad_last(_f32(step.v, dev), ds).contiguous()
        out = torch.zeros(1, 1, ds, dtype=torch.float32, device=dev)
        snap = L.snapshot()
        L.step(qd, kd, vd, out, advance=True)
        torch.cuda.synchronize()
        try:
            L.raise_status()
        except (NonFiniteError, SolveFailedError, IndexError, RuntimeError):
            # a failed step leaves the session as it was, like the reference,
            # which raises before it mutates any state (session.py:94-101)
            L.restore(snap)
            torch.cuda.synchronize()
            raise
        t = self._t
        self._t += 1
        n = int(L.view("res_cnt")[0, 0])
        omega = np.sort(L.view("res_idx")[0, 0, :n].cpu().numpy().astype(np.intp))  # stored unordered
        lite_start = max(0, t + 1 - self.cfg.lite_budget)
        self.last_selection = SelectionSet(omega_k=omega[omega < lite_start], omega_l=omega[omega >= lite_start],
                                           omega=omega)
        self.last_output = _np64(out[0, :, : self._d])
        miss = int(L.view("step_miss")[0, 0])
        total = int(L.view("step_total")[0, 0])
        self.stats.record(t, miss, total)
        r = self.cfg.prefill.rank
        self.factors = LowRankFactors(A_Q=self.factors.A_Q, A_K=self.factors.A_K,
                                      B_Q=_np64(L.view("B_Q")[0, 0, :r, : self._d]),
                                      B_K=_np64(L.view("B_K")[0, 0, :r, : self._d]))
        if compute_metrics:
            recall, err = self._fidelity(step.q, omega, self.last_output, t)
        else:
            recall, err = math.nan, math.nan
        return StepReport(step=t, selected_count=total, miss_count=miss, recall_vs_exact=recall, output_err=err)

    def _fidelity(self, q, omega, output, t):
        """Recall against the exact top-k over the full history and error
        against full-history attention (ref: session.py:119-131).  Both run
        on the device over the stored history: a float64 q K^T GEMM and
        float64 select for the exact set, the attention kernel for the
        full-history output; only k indices and one d-row come back."""
        L = self._layer
        d = self._d
        K = L.view("slow_k")[0, 0, : t + 1, :d]
        V = L.view("slow_v")[0, 0, : t + 1, :d]
        exact = _exact_topk_dev(D.t64(q.reshape(1, -1)), K.double().contiguous(), min(self.cfg.k_budget, t + 1))
        recall = selection_recall(omega, exact)
        full, _ = _attention_device(_f32(q, L.device), K.contiguous()[None], V.contiguous()[None], d,
                                    want_weights=False)
        full = _np64(full[:, :d])
        denom = float(np.linalg.norm(full))
        diff = float(np.linalg.norm(output - full))
        err = diff / denom if denom > 0 else (0.0 if diff == 0.0 else math.inf)
        return recall, err


def run_simulation(Q, K, V, prompt_len: int, cfg: SessionConfig, steps: int | None = None,
                   compute_metrics: bool = True) -> SimulationResult:
    """ref: session.py:134-165."""
    Q = as_matrix(Q, "Q")
    K = as_matrix(K, "K")
    V = as_matrix(V, "V")
    total = Q.shape[0]
    if not 1 <= prompt_len <= total:
        raise ValueError(f"prompt_len must be in [1, {total}], got {prompt_len}")
    available = total - prompt_len
    if steps is None:
        steps = available
    if steps > available:
        raise ValueError(f"{steps} decode steps requested, only {available} available")
    session = DecodeSession(cfg)
    session.prefill(Q[:prompt_len], K[:prompt_len], V[:prompt_len])
    reports = [session.decode_step(Q[i], K[i], V[i], compute_metrics=compute_metrics)
               for i in range(prompt_len, prompt_len + steps)]
    return SimulationResult(reports=reports, stats=session.stats, session=session)


def summarize(result: SimulationResult, cfg: SessionConfig) -> dict:
    errs = [r.output_err for r in result.reports]
    recalls = [r.recall_vs_exact for r in result.reports]
    have = bool(errs) and not any(math.isnan(e) for e in errs)
    return {
        "steps": len(result.reports),
        "mean_miss_rate": (result.stats.c_miss / result.stats.c_total if result.stats.c_total else None),
        "mean_recall": float(np.mean(recalls)) if have else None,
        "p50_output_err": float(np.percentile(errs, 50)) if have else None,
        "p95_output_err": float(np.percentile(errs, 95)) if have else None,
        "config": asdict(cfg),
    }


def write_report_csv(path, reports) -> None:
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["step", "selected", "miss", "recall", "output_err"])
        for r in reports:
            w.writerow([r.step, r.selected_count, r.miss_count, repr(r.recall_vs_exact), repr(r.output_err)])
