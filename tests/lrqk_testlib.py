"""Helpers shared by the GPU parity tests: build a one-layer device state
from oracle-side arrays and run step-locked comparisons against the CPU
oracle (oracle/lrqk_oracle.py).

Near-tie rule.  The GPU scores a row as an fp32 FMA chain
over the r entries of q_hat and the STORED proxy row A_i (fp32 or bf16
storage), then rounds the sum to fp32.  Against the fp64 dot product of the
same q_hat and the same stored row, the error is bounded by

    e_i = r * 2^-24 * sum_j |q_hat_j| |A_ij|  +  2^-24 |s_i|

and two selections made from the two score vectors may differ only at
indices i with |s_i - s_(k)| <= e_i + e_(k), s_(k) the k-th largest fp64
score.  When the oracle also uses its own fp64 q_hat (not the GPU's), the
bound on every row grows by sum_j |dq_j| |A_ij|, dq = q_hat_gpu - q_hat_ref
measured that step.  Every excused index is logged.
"""

from __future__ import annotations

import json
import os

import numpy as np
import torch

from oracle import lrqk_oracle as O

U32 = 2.0 ** -24
RTOL = {"f32": 1e-4, "bf16": 2e-2}


def make_layer(B, Hq, Hkv, d, r, kb, lb, t_max, dtype="f32", policy="hbm", **kw):
    from paper_2510_23649_b200.engine import LayerShape, LayerState

    shape = LayerShape(batch=B, n_q_heads=Hq, n_kv_heads=Hkv, head_dim=d, rank=r, k_budget=kb,
                       lite_budget=lb, t_max=t_max, dtype=dtype, policy=policy)
    return LayerState(shape, **kw)


def to_dev(x, dtype=torch.float32):
    return torch.as_tensor(np.asarray(x), dtype=dtype, device="cuda")


def seed_layer(layer, A_K, B_Q, B_K, K, V):
    """A_K [B,Hq,l,r], B_* [B,Hq,r,d], K/V [B,Hkv,l,d] numpy float64."""
    layer.load_prompt(to_dev(A_K), to_dev(B_Q), to_dev(B_K), to_dev(K), to_dev(V))


def quantize(x, dtype):
    """Round float64 values to the storage dtype and back (what the GPU sees)."""
    t = torch.as_tensor(np.asarray(x), dtype=torch.float64)
    if dtype == "bf16":
        return t.to(torch.bfloat16).to(torch.float64).numpy()
    return t.to(torch.float32).to(torch.float64).numpy()


def rows_dev(x, layer):
    """[.., d] float64 -> padded device rows in the layer's storage dtype."""
    from paper_2510_23649_b200.engine import pad_last

    t = torch.as_tensor(np.asarray(x), dtype=torch.float32, device="cuda")
    return pad_last(t, layer.shape.dim_stride).to(layer.sdt).contiguous()


def keys_to_scores(keys_u32):
    """Invert the order-preserving fp32 key of the score kernel."""
    k = np.asarray(keys_u32).astype(np.uint32)
    u = np.where(k & 0x80000000, k & 0x7FFFFFFF, ~k & 0xFFFFFFFF).astype(np.uint32)
    return u.view(np.float32).astype(np.float64)


def score_error_bound(P, q, r, extra_dq=None):
    """Per-row bound e_i of the module docstring; P [n, r] stored rows
    (float64 copies), q [r] the q_hat the GPU used."""
    P = np.asarray(P)
    s = P @ q
    e = r * U32 * (np.abs(P) @ np.abs(q)) + U32 * np.abs(s)
    if extra_dq is not None:
        e = e + np.abs(P) @ np.abs(extra_dq)
    return s, e


def near_tie_diff(s_ref, e, got, want, k_eff):
    """Indices in got ^ want that are NOT excused near-ties, and the excused
    ones: s_ref fp64 scores of the candidates, e their error bounds."""
    diff = sorted(set(int(i) for i in got) ^ set(int(i) for i in want))
    if not diff:
        return [], []
    order = np.lexsort((np.arange(s_ref.size), -s_ref))
    kth = order[k_eff - 1]
    bad, ok = [], []
    for i in diff:
        gap = abs(s_ref[i] - s_ref[kth])
        (ok if gap <= e[i] + e[kth] else bad).append((i, float(gap), float(e[i] + e[kth])))
    return bad, ok


def near_tie_ok(scores, got, want, k_eff, eps):
    """Legacy scalar-epsilon form (kept for the short-context tests)."""
    diff = set(got) ^ set(want)
    if not diff:
        return True, 0
    s = np.asarray(scores)
    kth = np.sort(s)[::-1][k_eff - 1] if k_eff > 0 else 0.0
    for i in diff:
        if abs(s[i] - kth) > eps:
            return False, len(diff)
    return True, len(diff)


def check_scores_on_device(layer, t, heads=None):
    """Score-kernel parity at any context length: the GPU's order-preserving
    keys for tokens 0..t must equal the fp64 product of the stored proxy rows
    and the GPU's q_hat within the per-row bound e_i (computed on the device
    in fp64).  Returns the largest |err| / e_i seen."""
    sh = layer.shape
    r = sh.rank
    P = layer.proxy_rows()[:, :, : t + 1, :r].double()                       # [B,Hq,n,r]
    qh = layer.view("q_hat")[:, :, :r].double()                              # [B,Hq,r]
    keys = layer.view("keys")[:, :, : t + 1].clone()
    u = keys.view(torch.int32).to(torch.int64) & 0xFFFFFFFF
    neg = (u & 0x80000000) == 0
    bits = torch.where(neg, (~u) & 0xFFFFFFFF, u & 0x7FFFFFFF).to(torch.int64)
    bits = torch.where(bits >= 2 ** 31, bits - 2 ** 32, bits).to(torch.int32)
    s_gpu = bits.view(torch.float32).double()
    s64 = torch.einsum("bhnr,bhr->bhn", P, qh)
    e = r * U32 * torch.einsum("bhnr,bhr->bhn", P.abs(), qh.abs()) + U32 * s64.abs() + 1e-37
    ratio = ((s_gpu - s64).abs() / e)
    if heads is not None:
        ratio = ratio[:, heads]
    worst = float(ratio.max())
    assert worst <= 1.0, f"score kernel outside its fp32 error bound at t={t}: max |err|/bound = {worst:.3g}"
    return worst


class ParityLog:
    """Collects the step-locked parity statistics (excused near-ties etc.)
    and, when LRQK_PARITY_LOG names a directory, writes them as JSON."""

    def __init__(self, name):
        self.name = name
        self.rec = dict(test=name, steps=0, head_steps=0, excused_gpu_qhat=[], excused_ref_qhat=[],
                        max_qhat_rel=0.0, max_khat_rel=0.0, max_B_rel=0.0, max_B_rel_ref=0.0,
                        max_out_rel=0.0, max_score_err_over_bound=0.0, selections_identical=0,
                        selections_identical_ref_qhat=0)

    def write(self):
        d = os.environ.get("LRQK_PARITY_LOG")
        if d:
            os.makedirs(d, exist_ok=True)
            with open(os.path.join(d, f"{self.name}.json"), "w") as f:
                json.dump(self.rec, f, indent=1)


def _rel(a, b):
    n = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / n) if n > 0 else float(np.linalg.norm(a))


class StepLocked:
    """One persistent oracle HeadState per (sequence, q-head), re-synced to the
    GPU after every step: the appended proxy row (the GPU's stored k_hat), the
    B factors and the resident set.  Each GPU step is therefore judged against
    the reference algorithm applied to the GPU's own previous state.

    Q [B,Hq,T,d], K/V [B,Hkv,T,d] float64 (storage-representable); the layer
    must already hold the prompt [0, prompt) and the oracle states are built
    from the layer's stored prompt rows."""

    def __init__(self, layer, Q, K, V, prompt, lam=(1.0, 1.0), max_iter=2, tol=1e-2, heads=None):
        self.layer, self.Q, self.K, self.V = layer, Q, K, V
        sh = layer.shape
        self.sh = sh
        self.heads = heads if heads is not None else [(b, h) for b in range(sh.batch) for h in range(sh.n_q_heads)]
        d, r = sh.head_dim, sh.rank
        P = layer.proxy_rows()[:, :, :prompt, :r].float().cpu().numpy().astype(np.float64)
        BQ = layer.view("B_Q")[:, :, :r, :d].cpu().numpy().astype(np.float64)
        BK = layer.view("B_K")[:, :, :r, :d].cpu().numpy().astype(np.float64)
        self.st = {}
        for b, h in self.heads:
            g = h // sh.group
            f = O.Factors(None, P[b, h], BQ[b, h], BK[b, h])
            self.st[(b, h)] = O.seed_head(K[b, g, :prompt], V[b, g, :prompt], f, sh.k_budget, sh.lite_budget,
                                          lam1=lam[0], lam2=lam[1], max_iter=max_iter, tol=tol)
        self.t = prompt

    def check_step(self, out, log: ParityLog, dtype, rtol_hat, check_b=True, strict=True):
        """Compare the GPU step that just ran (token t = self.t) with the
        oracle, then re-sync.  out: [B, Hq, dim_stride] device outputs.
        strict=False skips the comparisons with the oracle's OWN compression
        (q_hat, k_hat, B and the selection it implies) -- for singular
        compression systems, whose jittered solutions are conditioning-limited
        in fp32 -- and keeps everything judged on the GPU's own q_hat."""
        L, sh, t = self.layer, self.sh, self.t
        d, r, kb, lb = sh.head_dim, sh.rank, sh.k_budget, sh.lite_budget
        res_cnt = L.view("res_cnt").cpu().numpy()
        res_idx = L.view("res_idx").cpu().numpy()
        keys = L.view("keys")[:, :, : t + 1].cpu().numpy().view(np.uint32)
        qh = L.view("q_hat")[:, :, :r].cpu().numpy().astype(np.float64)
        kh = L.view("k_hat")[:, :, :r].cpu().numpy().astype(np.float64)
        BQn = L.view("B_Q")[:, :, :r, :d].cpu().numpy().astype(np.float64)
        BKn = L.view("B_K")[:, :, :r, :d].cpu().numpy().astype(np.float64)
        row_t = L.proxy_rows()[:, :, t, :r].float().cpu().numpy().astype(np.float64)
        miss = L.view("step_miss").cpu().numpy()
        tot = L.view("step_total").cpu().numpy()
        cmiss = L.view("c_miss").cpu().numpy()
        outs = out.float().cpu().numpy().astype(np.float64)
        lite_lo = max(0, t + 1 - lb)
        k_eff = min(kb, lite_lo)
        for b, h in self.heads:
            g = h // sh.group
            st = self.st[(b, h)]
            q, k, v = self.Q[b, h, t], self.K[b, g, t], self.V[b, g, t]
            prev_res = st.resident.copy()
            BQ0, BK0 = st.B_Q.copy(), st.B_K.copy()
            ref = O.head_step(st, q, k, v)           # oracle's own step (its own q_hat / k_hat)
            # ---- compression ---------------------------------------------------
            eq = _rel(qh[b, h], ref.q_hat.ravel())
            ek = _rel(kh[b, h], ref.k_hat.ravel())
            log.rec["max_qhat_rel"] = max(log.rec["max_qhat_rel"], eq)
            log.rec["max_khat_rel"] = max(log.rec["max_khat_rel"], ek)
            if strict:
                assert eq <= rtol_hat and ek <= rtol_hat, f"q_hat/k_hat rel err {eq:.3g}/{ek:.3g} at t={t} (b={b},h={h})"
            # ---- the appended proxy row is the GPU's k_hat in storage precision --
            np.testing.assert_allclose(row_t[b, h], quantize(kh[b, h], dtype), rtol=0, atol=0)
            st.proxy[t] = row_t[b, h]                 # sync the store to the stored row
            # ---- post-step B factors: the line search on the GPU's q_hat/k_hat --
            if check_b:
                bq_ref, bk_ref, _, _ = O.refresh_projections(q[None], k[None], O.Compression(qh[b, h][None],
                                                                                            kh[b, h][None]), BQ0, BK0)
                eb = max(_rel(BQn[b, h], bq_ref), _rel(BKn[b, h], bk_ref))
                log.rec["max_B_rel"] = max(log.rec["max_B_rel"], eb)
                assert eb <= 2e-5, f"B line-search update rel err {eb:.3g} at t={t} (b={b},h={h})"
                ebr = max(_rel(BQn[b, h], ref.B_Q), _rel(BKn[b, h], ref.B_K))
                log.rec["max_B_rel_ref"] = max(log.rec["max_B_rel_ref"], ebr)
                assert ebr <= 20 * rtol_hat or not strict, f"B vs oracle's own update rel err {ebr:.3g} at t={t}"
            st.B_Q, st.B_K = BQn[b, h].copy(), BKn[b, h].copy()
            # ---- scores: GPU keys vs the fp64 product on the same q_hat and rows --
            s_gpu = keys_to_scores(keys[b, h])
            s64, e = score_error_bound(st.proxy[: t + 1], qh[b, h], r)
            worst = float(np.max(np.abs(s_gpu - s64) / (e + 1e-300)))
            log.rec["max_score_err_over_bound"] = max(log.rec["max_score_err_over_bound"], worst)
            assert worst <= 1.0, f"scores outside the fp32 bound at t={t}: {worst:.3g}"
            # ---- selection ------------------------------------------------------
            n = int(res_cnt[b, h])
            got = np.sort(res_idx[b, h, :n].astype(np.int64))
            _, _, exact = O.select(s_gpu, t, kb, lb)      # reference rule on the GPU's own scores
            np.testing.assert_array_equal(got, exact)
            # vs the oracle rule on fp64 scores of the same q_hat: near-ties only
            _, _, sel64 = O.select(s64, t, kb, lb)
            if k_eff > 0:
                bad, ok = near_tie_diff(s64[:lite_lo], e[:lite_lo], got[got < lite_lo], sel64[sel64 < lite_lo],
                                        k_eff)
                assert not bad, f"selection differs beyond near-ties at t={t} (b={b},h={h}): {bad[:5]}"
                log.rec["excused_gpu_qhat"] += [(t, b, h) + x for x in ok]
                log.rec["selections_identical"] += int(not ok)
            if k_eff > 0 and strict:
                # vs the oracle's fully independent selection (its own q_hat)
                dq = qh[b, h] - ref.q_hat.ravel()
                sref, eref = score_error_bound(st.proxy[: t + 1], ref.q_hat.ravel(), r, extra_dq=dq)
                omega_ref = np.sort(ref.omega)
                bad2, ok2 = near_tie_diff(sref[:lite_lo], eref[:lite_lo], got[got < lite_lo],
                                          omega_ref[omega_ref < lite_lo], k_eff)
                assert not bad2, f"selection differs from the oracle's beyond near-ties at t={t}: {bad2[:5]}"
                log.rec["excused_ref_qhat"] += [(t, b, h) + x for x in ok2]
                log.rec["selections_identical_ref_qhat"] += int(not ok2)
            # ---- hit/miss counters: the reference replay rule, bit-exact ------------
            before = set(prev_res.tolist()) | {t}
            want_miss = len(set(got.tolist()) - before)
            assert int(miss[b, h]) == want_miss and int(tot[b, h]) == len(got)
            if np.array_equal(got, np.sort(ref.omega)):
                assert want_miss == ref.miss and len(got) == ref.total
            st.c_miss += want_miss - ref.miss
            st.c_total += len(got) - ref.total
            assert int(cmiss[b, h]) == st.c_miss
            # ---- attention on the identical index set --------------------------------
            want, _ = O.attend(q[None], st.K[got], st.V[got])
            eo = _rel(outs[b, h, :d], want.ravel())
            log.rec["max_out_rel"] = max(log.rec["max_out_rel"], eo)
            np.testing.assert_allclose(outs[b, h, :d], want.ravel(), rtol=RTOL[dtype],
                                       atol=RTOL[dtype] * np.abs(want).max())
            st.resident = got
            log.rec["head_steps"] += 1
        log.rec["steps"] += 1
        self.t += 1
