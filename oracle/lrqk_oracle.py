"""CPU oracle for the LRQK decode-time sparse-attention path.

TEST INFRASTRUCTURE ONLY.  This module is a float64 numpy restatement of the
reference package (``pkg/src/lrqk`` in arXiv 2510.23649's artefact, read from
``/root/reference`` during development).  It exists so that

  * ``tests/`` can check the CUDA path against it,
  * ``__graft_entry__.smoke()`` can check one small CUDA invocation,
  * ``bench.py`` can time it as the ``cpu_baseline`` / ``--impl reference`` arm.

Nothing in the product package (``paper_2510_23649_b200``) imports it; the
product path fails loudly when the CUDA library is missing instead of falling
back here.

Parity of this restatement is PINNED against the reference itself: the
fixtures in ``tests/golden/`` were produced by importing the reference package
(``tests/golden/make_golden.py``) and ``tests/test_oracle_golden.py`` replays
them through this module.

Every function names the reference lines it restates as
``ref: <file>:<lines>`` (paths relative to ``pkg/src/lrqk``).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import scipy.linalg as sla

# ref: linalg.py:19 -- relative jitter for a singular SPD system
SPD_JITTER = 1e-10
# ref: decode.py:26 -- line-search denominator floor
ETA_FLOOR = 1e-14


class NonFiniteError(ValueError):
    """ref: errors.py:4-5"""


class SolveFailedError(RuntimeError):
    """ref: errors.py:8-9"""


# --------------------------------------------------------------------------
# dense helpers  (ref: linalg.py)
# --------------------------------------------------------------------------

def check_matrix(a, what="matrix"):
    """ref: linalg.py:22-34 -- float64, C-order, 2-D, all finite."""
    m = np.ascontiguousarray(a, dtype=np.float64)
    if m.ndim != 2:
        raise ValueError(f"{what} must be 2-D, got shape {m.shape}")
    if not np.all(np.isfinite(m)):
        raise NonFiniteError(f"{what} contains non-finite entries")
    return m


def check_row(a, what="row"):
    """ref: linalg.py:37-45 -- 1-D input is promoted to a 1 x n row."""
    arr = np.asarray(a, dtype=np.float64)
    m = check_matrix(arr.reshape(1, -1) if arr.ndim == 1 else arr, what)
    if m.shape[0] != 1:
        raise ValueError(f"{what} must be a single row, got shape {m.shape}")
    return m


def sym_gram(A):
    """ref: linalg.py:48-55 -- A^T A with the upper triangle copied down."""
    if A.size == 0:
        raise ValueError("gram requires a nonempty matrix")
    G = A.T @ A
    upper = np.triu(G, 1)
    return np.triu(G) + upper.T


def sq_norm(A):
    """ref: linalg.py:58-60"""
    return float(np.sum(A * A))


def spd_right_solve(M, RHS):
    """Solve X M = RHS (M small, symmetric PSD).  ref: linalg.py:63-93.

    Cholesky; on failure one retry with jitter 1e-10 (tr(M)/r + 1) on the
    diagonal; a second failure raises SolveFailedError.
    """
    if not (np.all(np.isfinite(M)) and np.all(np.isfinite(RHS))):
        raise NonFiniteError("solve_spd: non-finite system")
    r = M.shape[0]
    if M.shape != (r, r):
        raise ValueError(f"M must be square, got {M.shape}")
    if RHS.shape[1] != r:
        raise ValueError(f"RHS has {RHS.shape[1]} cols, expected {r}")
    try:
        fac = sla.cho_factor(M, lower=True, check_finite=False)
    except np.linalg.LinAlgError:
        bump = SPD_JITTER * (np.trace(M) / r + 1.0)
        try:
            fac = sla.cho_factor(M + bump * np.eye(r), lower=True, check_finite=False)
        except np.linalg.LinAlgError as exc:
            raise SolveFailedError(f"SPD solve failed for {r}x{r} even with jitter") from exc
    return sla.cho_solve(fac, RHS.T, check_finite=False).T


def largest_k(scores, k):
    """Indices of the k largest scores, returned ascending; equal scores
    prefer the lower index.  ref: linalg.py:96-110."""
    if k < 1:
        raise ValueError(f"k must be >= 1, got {k}")
    s = np.asarray(scores, dtype=np.float64).ravel()
    if k >= s.size:
        return np.arange(s.size)
    # lexsort: last key is primary -> (-score, index) ascending
    order = np.lexsort((np.arange(s.size), -s))
    return np.sort(order[:k])


# --------------------------------------------------------------------------
# prefill factorisation  (ref: prefill.py)
# --------------------------------------------------------------------------

@dataclass
class Factors:
    """ref: prefill.py:65-81 (A_* l x r, B_* r x d)."""

    A_Q: np.ndarray
    A_K: np.ndarray
    B_Q: np.ndarray
    B_K: np.ndarray

    def clone(self):
        return Factors(self.A_Q.copy(), self.A_K.copy(), self.B_Q.copy(), self.B_K.copy())


def column_mass(Q, K):
    """ref: prefill.py:108-113 -- columnwise L1 mass of Q, of K, and the sum."""
    sq = np.abs(Q).sum(axis=0)
    sk = np.abs(K).sum(axis=0)
    return sq, sk, sq + sk


def initial_factors(Q, K, rank, kind="randn", seed=0):
    """ref: prefill.py:116-139."""
    if Q.shape != K.shape:
        raise ValueError("Q and K must share a shape")
    l, d = Q.shape
    if rank > d:
        raise ValueError(f"rank {rank} exceeds head dimension {d}")
    if kind == "randn":
        gen = np.random.default_rng(seed)
        A_Q = gen.standard_normal((l, rank))
        A_K = gen.standard_normal((l, rank))
    elif kind == "top":
        sq, sk, _ = column_mass(Q, K)
        A_Q = Q[:, largest_k(sq, rank)].copy()
        A_K = K[:, largest_k(sk, rank)].copy()
    elif kind == "topcol":
        _, _, sqk = column_mass(Q, K)
        cols = largest_k(sqk, rank)
        A_Q, A_K = Q[:, cols].copy(), K[:, cols].copy()
    else:
        raise ValueError(f"unknown init kind {kind!r}")
    return Factors(A_Q, A_K, np.zeros((rank, d)), np.zeros((rank, d)))


def objective(Q, K, f, lam_q, lam_k):
    """Prefill Lagrangian through d x d / r x r Gram traces.
    ref: prefill.py:142-158 (incl. the clamp at 0, :155)."""
    gq, gk = sym_gram(Q), sym_gram(K)
    cross = float(np.sum((Q.T @ f.A_Q) * (K.T @ f.A_K)))
    approx = float(np.sum(sym_gram(f.A_Q) * sym_gram(f.A_K)))
    fit = max(float(np.sum(gq * gk)) - 2.0 * cross + approx, 0.0)
    rq = sq_norm(Q - f.A_Q @ f.B_Q)
    rk = sq_norm(K - f.A_K @ f.B_K)
    return 0.5 * fit + 0.5 * lam_q * rq + 0.5 * lam_k * rk


def fit_B(A, X):
    """ref: prefill.py:161-163 -- B = (A^T A)^-1 A^T X."""
    return spd_right_solve(sym_gram(A), X.T @ A).T


def fit_A_K(Q, K, f, lam_k):
    """ref: prefill.py:166-172."""
    M = sym_gram(f.A_Q) + lam_k * sym_gram(f.B_K.T)
    return spd_right_solve(M, K @ (Q.T @ f.A_Q + lam_k * f.B_K.T))


def fit_A_Q(Q, K, f, lam_q):
    """ref: prefill.py:175-181."""
    M = sym_gram(f.A_K) + lam_q * sym_gram(f.B_Q.T)
    return spd_right_solve(M, Q @ (K.T @ f.A_K + lam_q * f.B_Q.T))


def mean_factor_change(new, old):
    """ref: prefill.py:184-194."""
    acc = 0.0
    for a, b in ((new.A_Q, old.A_Q), (new.A_K, old.A_K), (new.B_Q, old.B_Q), (new.B_K, old.B_K)):
        acc += sq_norm(a - b) / a.size
    return acc / 4.0


@dataclass
class PrefillTrace:
    """ref: prefill.py:93-100"""

    factors: Factors
    objective: list
    sweeps: int
    converged: bool


def factorize(Q, K, rank=32, lam_q=1.0, lam_k=1.0, max_iter=2, tol=1e-2,
              init="randn", seed=0, init_factors=None):
    """BCD sweeps B_Q, B_K, A_K, A_Q.  ref: prefill.py:197-223.

    ``init_factors`` (optional) replaces the randn draw -- used by tests that
    hand the GPU and the oracle the very same starting point.
    """
    Q = check_matrix(Q, "Q")
    K = check_matrix(K, "K")
    if Q.shape != K.shape:
        raise ValueError("Q and K must share a shape")
    f = init_factors.clone() if init_factors is not None else initial_factors(Q, K, rank, init, seed)
    obj = [objective(Q, K, f, lam_q, lam_k)]
    done = False
    n = 0
    for _ in range(max_iter):
        before = f.clone()
        f.B_Q = fit_B(f.A_Q, Q)
        f.B_K = fit_B(f.A_K, K)
        f.A_K = fit_A_K(Q, K, f, lam_k)
        f.A_Q = fit_A_Q(Q, K, f, lam_q)
        n += 1
        for nm in ("A_Q", "A_K", "B_Q", "B_K"):
            if not np.all(np.isfinite(getattr(f, nm))):
                raise NonFiniteError(f"factor {nm} diverged at sweep {n}")
        obj.append(objective(Q, K, f, lam_q, lam_k))
        if mean_factor_change(f, before) <= tol:
            done = True
            break
    return PrefillTrace(f, obj, n, done)


def relative_residuals(Q, K, f):
    """ref: prefill.py:239-253 (factor_residuals)."""
    def rel(num, den):
        if den == 0.0:
            return 0.0 if num == 0.0 else math.inf
        return math.sqrt(num / den)

    den = float(np.sum(sym_gram(Q) * sym_gram(K)))
    cross = float(np.sum((Q.T @ f.A_Q) * (K.T @ f.A_K)))
    approx = float(np.sum(sym_gram(f.A_Q) * sym_gram(f.A_K)))
    return (rel(sq_norm(Q - f.A_Q @ f.B_Q), sq_norm(Q)),
            rel(sq_norm(K - f.A_K @ f.B_K), sq_norm(K)),
            rel(max(den - 2.0 * cross + approx, 0.0), den))


# --------------------------------------------------------------------------
# per-token compression  (ref: decode.py)
# --------------------------------------------------------------------------

@dataclass
class Compression:
    """q_hat, k_hat (1 x r) plus the workspace values the reference exposes.
    ref: decode.py:58-76"""

    q_hat: np.ndarray
    k_hat: np.ndarray
    M_rq: np.ndarray = None
    m_lq: np.ndarray = None
    rounds: int = 0


def khat_seed(k, B_K):
    """ref: decode.py:79-81"""
    return spd_right_solve(sym_gram(B_K.T), k @ B_K.T)


def solve_qhat(q, k, k_hat, B_Q, A_res, K_res, lam1, lam2):
    """ref: decode.py:84-108 -- returns (q_hat, M_rq, m_lq)."""
    if A_res.shape[0] != K_res.shape[0]:
        raise ValueError("resident proxy/key row counts differ")
    qk = (q @ k.T).item()
    rhs = q @ B_Q.T + lam1 * qk * k_hat
    M = sym_gram(B_Q.T) + lam1 * (k_hat.T @ k_hat)
    if A_res.shape[0]:
        rhs = rhs + lam2 * (q @ K_res.T) @ A_res
        M = M + lam2 * sym_gram(A_res)
    return spd_right_solve(M, rhs), M, rhs


def solve_khat(q, k, q_hat, B_K, lam1):
    """ref: decode.py:111-119"""
    qk = (q @ k.T).item()
    M = sym_gram(B_K.T) + lam1 * (q_hat.T @ q_hat)
    return spd_right_solve(M, k @ B_K.T + lam1 * qk * q_hat)


def compress_token(q, k, B_Q, B_K, A_res, K_res, lam1=1.0, lam2=1.0, max_iter=2, tol=1e-2):
    """ref: decode.py:122-147 -- k_hat seed, then alternating q_hat/k_hat with
    the mean-squared-change stop (only testable from the second round)."""
    r = B_Q.shape[0]
    c = Compression(q_hat=np.zeros((1, r)), k_hat=khat_seed(k, B_K))
    last = None
    for _ in range(max_iter):
        c.q_hat, c.M_rq, c.m_lq = solve_qhat(q, k, c.k_hat, B_Q, A_res, K_res, lam1, lam2)
        c.k_hat = solve_khat(q, k, c.q_hat, B_K, lam1)
        c.rounds += 1
        now = np.hstack([c.q_hat, c.k_hat])
        if last is not None and sq_norm(now - last) / now.size <= tol:
            break
        last = now
    return c


def line_search(row_hat, B, target):
    """ref: decode.py:150-166 -- rank-1 gradient and exact step size."""
    resid = row_hat @ B - target
    grad = row_hat.T @ resid
    s = row_hat @ grad
    den = (s @ s.T).item()
    num = (resid @ s.T).item()
    if den <= ETA_FLOOR * (1.0 + abs(num)):
        return grad, 0.0
    return grad, num / den


def refresh_projections(q, k, comp, B_Q, B_K):
    """ref: decode.py:169-184 -- returns (B_Q', B_K', eta_Q, eta_K)."""
    gq, eq = line_search(comp.q_hat, B_Q, q)
    gk, ek = line_search(comp.k_hat, B_K, k)
    return B_Q - eq * gq, B_K - ek * gk, eq, ek


# --------------------------------------------------------------------------
# scoring, selection, residency accounting  (ref: cache.py)
# --------------------------------------------------------------------------

def proxy_scores(q_hat, proxy):
    """ref: cache.py:141-146 -- unscaled q_hat . A_K rows."""
    return (proxy @ q_hat.reshape(-1, 1)).ravel()


def select(scores, t, k_budget, lite_budget):
    """ref: cache.py:149-171 -> (omega_k, omega_l, omega)."""
    s = np.asarray(scores, dtype=np.float64).ravel()
    if s.size != t + 1:
        raise ValueError(f"scores must cover tokens 0..{t}, got {s.size}")
    lite_lo = max(0, t + 1 - lite_budget)
    omega_l = np.arange(lite_lo, t + 1)
    if lite_lo == 0:
        omega_k = np.arange(0)
    else:
        omega_k = largest_k(s[:lite_lo], min(k_budget, lite_lo))
    return omega_k, omega_l, np.concatenate([omega_k, omega_l])


def count_misses(omega, resident_before):
    """ref: cache.py:174-196 -- misses are selected rows not resident, where
    resident already includes the appended token (cache.py:213)."""
    sel = set(int(i) for i in omega)
    return len(sel - set(resident_before)), len(sel)


def attend(q, K, V):
    """softmax(q K^T / sqrt(d)) V with max subtraction.  ref: attention.py:23-34."""
    n, d = K.shape
    if n == 0:
        raise ValueError("exact_attention requires at least one key")
    z = (q @ K.T).ravel() / np.sqrt(d)
    z = z - z.max()
    w = np.exp(z)
    w = w / w.sum()
    return (w[None, :] @ V), w


# --------------------------------------------------------------------------
# one head's decode session  (ref: session.py:62-117, cache.py:84-138)
# --------------------------------------------------------------------------

class _Rows:
    """Append-only row store with amortised doubling, as the reference's
    _RowStore (ref: cache.py:21-51): capacity starts at 16 rows and doubles
    when full, so after seeding n rows it is the smallest 16 * 2^j >= n and a
    2^17-row prompt pays its regrowth copy on the first decode append, as in
    the reference."""

    def __init__(self, rows):
        rows = np.asarray(rows, dtype=np.float64)
        cap = 16
        while cap < rows.shape[0]:
            cap *= 2
        self.buf = np.empty((cap, rows.shape[1]))
        self.buf[: rows.shape[0]] = rows
        self.n = rows.shape[0]

    def append(self, row):
        if self.n == self.buf.shape[0]:
            grown = np.empty((2 * self.buf.shape[0], self.buf.shape[1]))
            grown[: self.n] = self.buf[: self.n]
            self.buf = grown
        self.buf[self.n] = np.ravel(row)
        self.n += 1

    @property
    def rows(self):
        return self.buf[: self.n]


@dataclass
class HeadState:
    """All state one (sequence, q-head) session carries between steps.

    K, V, proxy are the full histories (slow tier and proxy store); resident
    is the fast-tier index set (ref: cache.py:84-112)."""

    K: np.ndarray
    V: np.ndarray
    proxy: np.ndarray
    B_Q: np.ndarray
    B_K: np.ndarray
    resident: np.ndarray  # sorted int64
    k_budget: int
    lite_budget: int
    lam1: float = 1.0
    lam2: float = 1.0
    max_iter: int = 2
    tol: float = 1e-2
    c_miss: int = 0
    c_total: int = 0
    per_step: list = field(default_factory=list)

    def __post_init__(self):
        self._K, self._V, self._P = _Rows(self.K), _Rows(self.V), _Rows(self.proxy)

    def append(self, k, v, k_hat):
        self._K.append(k)
        self._V.append(v)
        self._P.append(k_hat)
        self.K, self.V, self.proxy = self._K.rows, self._V.rows, self._P.rows


def seed_head(K, V, factors, k_budget, lite_budget, **decode_kw):
    """ref: cache.py:114-124 + session.py:80-87"""
    l = K.shape[0]
    lo = max(0, l - lite_budget)
    return HeadState(K=np.array(K, dtype=np.float64), V=np.array(V, dtype=np.float64),
                     proxy=np.array(factors.A_K, dtype=np.float64),
                     B_Q=np.array(factors.B_Q, dtype=np.float64),
                     B_K=np.array(factors.B_K, dtype=np.float64),
                     resident=np.arange(lo, l), k_budget=k_budget,
                     lite_budget=lite_budget, **decode_kw)


@dataclass
class StepResult:
    t: int
    q_hat: np.ndarray
    k_hat: np.ndarray
    scores: np.ndarray
    omega: np.ndarray
    miss: int
    total: int
    output: np.ndarray
    B_Q: np.ndarray
    B_K: np.ndarray


def head_step(st: HeadState, q, k, v):
    """One decode step of one head, in the reference order
    (ref: session.py:90-104): compress against the previous resident set,
    refresh B, append, score everything, select, account, attend."""
    q = check_row(q, "q")
    k = check_row(k, "k")
    v = check_row(v, "v")
    res = st.resident
    comp = compress_token(q, k, st.B_Q, st.B_K, st.proxy[res], st.K[res],
                          st.lam1, st.lam2, st.max_iter, st.tol)
    st.B_Q, st.B_K, _, _ = refresh_projections(q, k, comp, st.B_Q, st.B_K)
    t = st.K.shape[0]
    st.append(k, v, comp.k_hat)
    before = np.union1d(res, [t])
    scores = proxy_scores(comp.q_hat, st.proxy)
    _, _, omega = select(scores, t, st.k_budget, st.lite_budget)
    miss, total = count_misses(omega, before)
    st.c_miss += miss
    st.c_total += total
    st.per_step.append((t, miss, total))
    st.resident = np.sort(omega)
    out, _ = attend(q, st.K[st.resident], st.V[st.resident])
    return StepResult(t, comp.q_hat, comp.k_hat, scores, np.array(omega), miss, total,
                      out, st.B_Q.copy(), st.B_K.copy())
