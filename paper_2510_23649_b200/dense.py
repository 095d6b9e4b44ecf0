"""Float64 device linear algebra behind the drop-in entry points of the
reference's linalg / prefill / decode modules (pkg/src/lrqk/linalg.py,
prefill.py:142-253, decode.py:79-184).

Every function takes and returns float64 CUDA tensors and runs on the
dense.cu kernels through the C ABI (include/lrqk_b200.h).  torch only
allocates and copies here; the arithmetic is the library's.  Errors follow
the reference: non-finite systems raise NonFiniteError, a Cholesky that
fails even with jitter raises SolveFailedError.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib
from .errors import NonFiniteError, SolveFailedError


def dev():
    _lib.lib()
    return torch.device("cuda")


def t64(x) -> torch.Tensor:
    """numpy / torch -> contiguous float64 device tensor."""
    if isinstance(x, torch.Tensor):
        return x.to(device=dev(), dtype=torch.float64).contiguous()
    return torch.as_tensor(np.ascontiguousarray(x, dtype=np.float64), device=dev())


def np64(t: torch.Tensor) -> np.ndarray:
    return t.detach().to(torch.float64).cpu().numpy()


def _p(t):
    return t.data_ptr() if t is not None else None


def gemm(A, B, *, ta=False, tb=False, alpha=1.0, beta=0.0, out=None):
    """alpha op(A) op(B) + beta out; A, B 2-D float64 device tensors."""
    lib = _lib.lib()
    m, k = (A.shape[1], A.shape[0]) if ta else (A.shape[0], A.shape[1])
    kb, n = (B.shape[1], B.shape[0]) if tb else (B.shape[0], B.shape[1])
    if k != kb:
        raise ValueError(f"inner dimensions differ: {k} vs {kb}")
    if out is None:
        out = torch.zeros(m, n, dtype=torch.float64, device=A.device)
        beta = 0.0
    wsb = lib.lrqk_gemm_f64_workspace(m, n, k)
    ws = torch.empty(max(1, wsb // 8), dtype=torch.float64, device=A.device) if wsb else None
    _lib.check(lib.lrqk_gemm_f64(int(ta), int(tb), m, n, k, float(alpha), _p(A), A.stride(0), _p(B), B.stride(0),
                                 float(beta), _p(out), out.stride(0), _p(ws), wsb, _lib.stream_ptr()),
               "lrqk_gemm_f64")
    return out


def gram(A, *, of_transpose=False):
    """A^T A (or, with of_transpose, A A^T = gram(A^T)), exactly symmetric."""
    G = gemm(A, A, tb=True) if of_transpose else gemm(A, A, ta=True)
    _lib.check(_lib.lib().lrqk_symmetrize_f64(_p(G), G.shape[0], G.stride(0), _lib.stream_ptr()),
               "lrqk_symmetrize_f64")
    return G


def dot(a, b) -> torch.Tensor:
    """sum(a * b) as a 1-element device tensor."""
    out = torch.zeros(1, dtype=torch.float64, device=a.device)
    work = torch.empty(256, dtype=torch.float64, device=a.device)
    _lib.check(_lib.lib().lrqk_dot_f64(_p(a), _p(b), a.numel(), _p(out), _p(work), _lib.stream_ptr()),
               "lrqk_dot_f64")
    return out


def axpby(alpha, x, beta, y, scale=None):
    """y <- alpha [* scale] x + beta y (in place); returns y."""
    _lib.check(_lib.lib().lrqk_axpby_f64(y.numel(), float(alpha), _p(scale), _p(x), float(beta), _p(y),
                                          _lib.stream_ptr()), "lrqk_axpby_f64")
    return y


class Status:
    """Device status word shared by a chain of solves; check() raises the
    reference's exception for whatever the kernels flagged."""

    def __init__(self):
        self.word = torch.zeros(1, dtype=torch.int32, device=dev())

    def check(self, what="solve_spd"):
        st = int(self.word.item()) & 0xFFFFFFFF
        if st & _lib.ST_NONFINITE:
            raise NonFiniteError(f"{what}: non-finite system")
        if st & _lib.ST_SOLVE_FAILED:
            raise SolveFailedError(f"{what}: SPD solve failed even with jitter")
        return st


def solve_spd(M, RHS, status: Status | None = None):
    """X with X M = RHS (M r x r, RHS n x r); errors are flagged in `status`
    (a fresh one is checked before returning when none is given)."""
    own = status is None
    status = status or Status()
    r = M.shape[0]
    n = RHS.shape[0]
    X = torch.zeros(n, r, dtype=torch.float64, device=M.device)
    work = torch.empty(r * r + 1, dtype=torch.float64, device=M.device)
    _lib.check(_lib.lib().lrqk_solve_spd_f64(_p(M), r, M.stride(0), _p(RHS), n, RHS.stride(0) if n else r, _p(X),
                                              r, _p(work), _p(status.word), _lib.stream_ptr()),
               "lrqk_solve_spd_f64")
    if own:
        status.check()
    return X


def topk(scores, k: int) -> torch.Tensor:
    """Ascending indices of the k largest float64 scores (ties -> lower
    index), int32 device tensor; k < n."""
    n = scores.numel()
    out = torch.empty(k, dtype=torch.int32, device=scores.device)
    _lib.check(_lib.lib().lrqk_topk_f64(_p(scores), n, k, _p(out), _lib.stream_ptr()), "lrqk_topk_f64")
    return out


def residual_sq(X, A, B):
    """||X - A B||_F^2 as a device scalar (the factor residual norms)."""
    R = X.clone()
    gemm(A, B, alpha=-1.0, beta=1.0, out=R)
    return dot(R, R)
