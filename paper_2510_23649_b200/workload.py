"""LRQK trace files and the reference's synthetic workloads.

Trace format (ref: workload.py:145-161): the 4 bytes "LRQK", a little-endian
u16 version (1), then records of [u8 role tag (q=0, k=1, v=2), u32 rows,
u32 cols, rows*cols little-endian float32, row-major].  `load_trace` returns
float64 matrices like the reference; `load_trace_device` parses the same
bytes once into a pinned host buffer and uploads every payload to the GPU
as float32 without a float64 round trip -- the engine's input path.

The generators restate the reference's seeded low-rank / recency-biased
heads (ref: workload.py:70-107) so oracle and engine see identical inputs;
they run on the host like the reference (input preparation, not the hot
path).
"""

from __future__ import annotations

import struct
from dataclasses import dataclass

import numpy as np

from .errors import CorruptTraceError, UnsupportedVersionError

MAGIC = b"LRQK"
VERSION = 1
ROLES = ("q", "k", "v")           # tag = index
_HDR = struct.Struct("<BII")      # role tag, rows, cols
RECENCY_TAPS = 40                 # exp(-40) is below float64 resolution


@dataclass(frozen=True)
class SyntheticSpec:
    """One generated head (ref: workload.py:31-56)."""

    l: int
    d: int
    r_true: int
    decay: float = 0.9
    recency_strength: float = 0.0
    seed: int = 0
    scale: float = 1.0

    def __post_init__(self):
        if min(self.l, self.d) < 1:
            raise ValueError("l and d must be >= 1")
        if not 1 <= self.r_true <= min(self.l, self.d):
            raise ValueError(f"r_true must lie in [1, min(l, d)] = [1, {min(self.l, self.d)}], got {self.r_true}")
        if not 0.0 < self.decay <= 1.0:
            raise ValueError(f"decay must be in (0, 1], got {self.decay}")
        if self.recency_strength < 0:
            raise ValueError("recency_strength must be >= 0")
        if self.scale <= 0:
            raise ValueError(f"scale must be > 0, got {self.scale}")


@dataclass(frozen=True)
class TraceRecord:
    role: str
    data: np.ndarray


def gen_lowrank_qk(spec: SyntheticSpec):
    """Q, K with singular values scale * decay^i (i < r_true) and a N(0,1) V;
    one PCG64 stream per spec, consumed Q (U, W), K (U, W), V
    (ref: workload.py:70-84)."""
    g = np.random.default_rng(spec.seed)
    sv = spec.scale * spec.decay ** np.arange(spec.r_true)

    def factor():
        left = np.linalg.qr(g.standard_normal((spec.l, spec.r_true)))[0]
        right = np.linalg.qr(g.standard_normal((spec.d, spec.r_true)))[0]
        return (left * sv) @ right.T

    Q = factor()
    K = factor()
    return Q, K, g.standard_normal((spec.l, spec.d))


def gen_recency_biased(spec: SyntheticSpec):
    """gen_lowrank_qk plus, for each key i and future query t in a 40-step
    window, strength * e^-(t-i) * sqrt(d) * q_t / |q_t|^2 (ref:
    workload.py:87-107); strength 0 returns the plain heads unchanged."""
    Q, K, V = gen_lowrank_qk(spec)
    if spec.recency_strength == 0.0:
        return Q, K, V
    K = K.copy()
    Qn = Q / (np.einsum("ij,ij->i", Q, Q) + 1e-30)[:, None]
    for lag in range(min(spec.l - 1, RECENCY_TAPS) + 1):
        K[: spec.l - lag] += (spec.recency_strength * np.exp(-float(lag)) * np.sqrt(spec.d)) * Qn[lag:]
    return Q, K, V


def save_trace(path, tensors) -> None:
    """Write (role, matrix) pairs (ref: workload.py:145-161)."""
    from .api import as_matrix

    parts = [MAGIC, struct.pack("<H", VERSION)]
    for role, data in tensors:
        key = str(role).lower()
        if key not in ROLES:
            raise ValueError(f"unknown tensor role {role!r}; expected q/k/v")
        m = as_matrix(data, f"{role} tensor")
        parts.append(_HDR.pack(ROLES.index(key), m.shape[0], m.shape[1]))
        parts.append(m.astype("<f4").tobytes(order="C"))
    with open(path, "wb") as fh:
        fh.write(b"".join(parts))


def _records(blob: bytes):
    """Yield (role, rows, cols, payload offset) with the reference's checks
    and error classes (ref: workload.py:164-195)."""
    if len(blob) < 6 or blob[:4] != MAGIC:
        raise CorruptTraceError("bad magic: not a trace file")
    (ver,) = struct.unpack_from("<H", blob, 4)
    if ver != VERSION:
        raise UnsupportedVersionError(f"trace version {ver} not supported (expected {VERSION})")
    pos = 6
    while pos < len(blob):
        if len(blob) - pos < _HDR.size:
            raise CorruptTraceError("truncated record header")
        tag, rows, cols = _HDR.unpack_from(blob, pos)
        pos += _HDR.size
        if tag >= len(ROLES):
            raise CorruptTraceError(f"unknown role tag {tag}")
        n = rows * cols * 4
        if len(blob) - pos < n:
            raise CorruptTraceError("truncated payload")
        yield ROLES[tag], rows, cols, pos
        pos += n


def load_trace(path) -> list:
    with open(path, "rb") as fh:
        blob = fh.read()
    return [TraceRecord(role, np.frombuffer(blob, "<f4", rows * cols, off).astype(np.float64).reshape(rows, cols))
            for role, rows, cols, off in _records(blob)]


def as_heads(records) -> list:
    """Consecutive q, k, v records of one shape form a head (ref: workload.py:198-216)."""
    if len(records) % 3:
        raise CorruptTraceError(f"expected q/k/v triples, got {len(records)} records")
    heads = []
    for h in range(len(records) // 3):
        trio = records[3 * h: 3 * h + 3]
        roles = [x.role for x in trio]
        if roles != list(ROLES):
            raise CorruptTraceError(f"head {h} has roles {roles}, expected q,k,v")
        shapes = {x.data.shape for x in trio}
        if len(shapes) != 1:
            raise CorruptTraceError(f"head {h} mixes shapes {shapes}")
        heads.append(tuple(x.data for x in trio))
    return heads


def load_trace_device(path, device="cuda"):
    """Trace -> per-head (Q, K, V) float32 device tensors, validated exactly as
    load_trace/as_heads.  The file is read once into pinned host memory and
    each payload is uploaded as its own float32 bytes (no float64 copy).
    Returns ([H, l, d] Q, K, V stacked when every head shares one shape)."""
    import torch

    with open(path, "rb") as fh:
        blob = fh.read()
    recs = list(_records(blob))
    if len(recs) % 3:
        raise CorruptTraceError(f"expected q/k/v triples, got {len(recs)} records")
    host = torch.frombuffer(bytearray(blob), dtype=torch.uint8).pin_memory()
    out = {r: [] for r in ROLES}
    for h in range(len(recs) // 3):
        trio = recs[3 * h: 3 * h + 3]
        if [x[0] for x in trio] != list(ROLES):
            raise CorruptTraceError(f"head {h} has roles {[x[0] for x in trio]}, expected q,k,v")
        if len({(x[1], x[2]) for x in trio}) != 1:
            raise CorruptTraceError(f"head {h} mixes shapes")
        for role, rows, cols, off in trio:
            if off % 4:
                raw = host[off: off + rows * cols * 4].clone()
            else:
                raw = host[off: off + rows * cols * 4]
            out[role].append(raw.view(torch.float32).view(rows, cols).to(device, non_blocking=True))
    torch.cuda.synchronize(device)
    return tuple(torch.stack(out[r]) for r in ROLES)
