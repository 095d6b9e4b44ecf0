"""Batched drivers of the reference CLI's `factorize` and `simulate`
subcommands (ref: cli.py:167-251), with the same output files
(SURVEY §8(f) f3, f4):

    factorize:  lagrangian.csv (head,sweep,lagrangian), residuals.csv
    simulate:   report_hNNN.csv, cache_hNNN.csv, miss_hist.csv, summary.json

The reference runs one Python DecodeSession per head on a thread pool.  Here
all heads of a workload run as ONE device layer (every head its own
(sequence, q-head) session with its own K/V head): each decode step is one
fused lrqk_decode_step for every head; the prompt factorisation is the
float64 device prefill_run per head.  Per-step fidelity metrics (exact top-k
over the full history, full-history attention) are computed on the device
too.  With metrics off, the files are byte-identical to the reference's
whenever the selections match (tests/test_gpu_sim.py).
"""

from __future__ import annotations

import json
import math
import os
from dataclasses import asdict

import numpy as np
import torch

from . import dense as D
from .api import (CacheStats, PrefillConfig, SessionConfig, StepReport, _attention_device, _exact_topk_dev, as_matrix,
                  factor_residuals, prefill_run, selection_recall, summarize, write_report_csv, write_stats_csv)
from .engine import LayerShape, LayerState, pad_last


class HeadResult:
    """Per head: reports, CacheStats and the prefill run (the reference's
    SimulationResult without the session object)."""

    def __init__(self, reports, stats, run):
        self.reports, self.stats, self.run = reports, stats, run


def _stack(heads, idx):
    return np.stack([as_matrix(h[idx], "QKV"[idx]) for h in heads])


def prefill_heads(heads, cfg: PrefillConfig) -> list:
    """prefill_run per head (ref: prefill.py:197-223): the float64 device
    factorisation, so sweeps, convergence and the factors -- and through them
    every later selection -- follow the reference's."""
    return [prefill_run(h[0], h[1], cfg) for h in heads]


def factorize(heads, cfg: PrefillConfig, out_dir) -> list:
    """`lrqk factorize` outputs (ref: cli.py:167-185)."""
    runs = prefill_heads(heads, cfg)
    os.makedirs(out_dir, exist_ok=True)
    with open(os.path.join(out_dir, "lagrangian.csv"), "w", newline="") as fh:
        fh.write("head,sweep,lagrangian\n")
        for h, run in enumerate(runs):
            for sweep, value in enumerate(run.objective):
                fh.write(f"{h},{sweep},{value!r}\n")
    with open(os.path.join(out_dir, "residuals.csv"), "w", newline="") as fh:
        fh.write("head,rel_err_q,rel_err_k,rel_err_qk\n")
        for h, (run, (Q, K, _)) in enumerate(zip(runs, heads)):
            rq, rk, rqk = factor_residuals(Q, K, run.factors)
            fh.write(f"{h},{rq!r},{rk!r},{rqk!r}\n")
    return runs


def simulate_heads(heads, prompt_len: int, cfg: SessionConfig, steps=None, compute_metrics=True) -> list:
    """run_simulation for every head at once (ref: session.py:134-165)."""
    Q, K, V = _stack(heads, 0), _stack(heads, 1), _stack(heads, 2)
    H, total, d = Q.shape
    if not 1 <= prompt_len <= total:
        raise ValueError(f"prompt_len must be in [1, {total}], got {prompt_len}")
    avail = total - prompt_len
    steps = avail if steps is None else steps
    if steps > avail:
        raise ValueError(f"{steps} decode steps requested, only {avail} available")
    runs = prefill_heads([(Q[h, :prompt_len], K[h, :prompt_len], None) for h in range(H)], cfg.prefill)
    dc = cfg.decode
    shape = LayerShape(batch=1, n_q_heads=H, n_kv_heads=H, head_dim=d, rank=cfg.prefill.rank,
                       k_budget=cfg.k_budget, lite_budget=cfg.lite_budget, t_max=total + 1, dtype="f32")
    L = LayerState(shape, lambda_1=dc.lambda_1, lambda_2=dc.lambda_2, max_iter=dc.max_iter, tol=dc.tol)
    dev = L.device
    f32 = lambda x: torch.as_tensor(x, dtype=torch.float32, device=dev)  # noqa: E731
    L.load_prompt(f32(np.stack([r.factors.A_K for r in runs]))[None], f32(np.stack([r.factors.B_Q for r in runs]))[None],
                  f32(np.stack([r.factors.B_K for r in runs]))[None], f32(K[:, :prompt_len])[None],
                  f32(V[:, :prompt_len])[None])
    ds = shape.dim_stride
    # token-major [total, H, ds]: one contiguous [1, H, ds] row block per step
    Qd = pad_last(f32(Q), ds).transpose(0, 1).contiguous()
    Kd = pad_last(f32(K), ds).transpose(0, 1).contiguous()
    Vd = pad_last(f32(V), ds).transpose(0, 1).contiguous()
    out = torch.zeros(1, H, ds, dtype=torch.float32, device=dev)
    stats = [CacheStats() for _ in range(H)]
    reports = [[] for _ in range(H)]
    for i in range(prompt_len, prompt_len + steps):
        L.step(Qd[i:i + 1], Kd[i:i + 1], Vd[i:i + 1], out, advance=True)
        torch.cuda.synchronize()
        L.raise_status()
        miss = L.view("step_miss")[0].cpu().numpy()
        tot = L.view("step_total")[0].cpu().numpy()
        if compute_metrics:
            cnt = L.view("res_cnt")[0].cpu().numpy()
            idx = L.view("res_idx")[0].cpu().numpy()
            outs = out[0, :, :d].double().cpu().numpy()
        for h in range(H):
            stats[h].record(i, int(miss[h]), int(tot[h]))
            if compute_metrics:
                recall, err = _fidelity(L, h, Q[h, i], idx[h, : cnt[h]], outs[h], i, cfg.k_budget)
            else:
                recall, err = math.nan, math.nan
            reports[h].append(StepReport(step=i, selected_count=int(tot[h]), miss_count=int(miss[h]),
                                         recall_vs_exact=recall, output_err=err))
    return [HeadResult(reports[h], stats[h], runs[h]) for h in range(H)]


def _fidelity(L, h, q, omega, output, t, k_budget):
    """ref: session.py:119-131, on the device (float64 q K^T + select for the
    exact set; the attention kernel over the full stored history)."""
    d = L.shape.head_dim
    K = L.view("slow_k")[0, h, : t + 1, :d]
    V = L.view("slow_v")[0, h, : t + 1, :d]
    exact = _exact_topk_dev(D.t64(q.reshape(1, -1)), K.double().contiguous(), min(k_budget, t + 1))
    recall = selection_recall(omega, exact)
    full, _ = _attention_device(torch.as_tensor(q.reshape(1, -1), dtype=torch.float32, device=K.device),
                                K.contiguous()[None], V.contiguous()[None], d, want_weights=False)
    full = full[0, :d].double().cpu().numpy()
    denom = float(np.linalg.norm(full))
    diff = float(np.linalg.norm(output - full))
    return recall, (diff / denom if denom > 0 else (0.0 if diff == 0.0 else math.inf))


def simulate(heads, cfg: SessionConfig, out_dir, prompt_len=None, steps=None, compute_metrics=True) -> dict:
    """`lrqk simulate` outputs (ref: cli.py:188-251); returns summary.json's dict."""
    total = heads[0][0].shape[0]
    prompt_len = prompt_len if prompt_len is not None else total // 2
    results = simulate_heads(heads, prompt_len, cfg, steps=steps, compute_metrics=compute_metrics)
    os.makedirs(out_dir, exist_ok=True)
    per_head, rates = [], []
    for h, res in enumerate(results):
        write_report_csv(os.path.join(out_dir, f"report_h{h:03d}.csv"), res.reports)
        write_stats_csv(os.path.join(out_dir, f"cache_h{h:03d}.csv"), res.stats)
        per_head.append(summarize(res, cfg))
        rates += [m / s for _, m, s in res.stats.per_step if s]
    counts, edges = np.histogram(rates, bins=20, range=(0.0, 1.0))
    with open(os.path.join(out_dir, "miss_hist.csv"), "w", newline="") as fh:
        fh.write("bin_lo,bin_hi,count\n")
        for i, c in enumerate(counts):
            fh.write(f"{edges[i]!r},{edges[i + 1]!r},{int(c)}\n")
    c_miss = sum(r.stats.c_miss for r in results)
    c_total = sum(r.stats.c_total for r in results)
    errs = [x.output_err for r in results for x in r.reports]
    recalls = [x.recall_vs_exact for r in results for x in r.reports]
    have = compute_metrics and bool(errs) and not any(math.isnan(e) for e in errs)
    summary = {
        "heads": len(results),
        "prompt_len": prompt_len,
        "steps_per_head": len(results[0].reports),
        "mean_miss_rate": c_miss / c_total if c_total else None,
        "mean_recall": float(np.mean(recalls)) if have else None,
        "p50_output_err": float(np.percentile(errs, 50)) if have else None,
        "p95_output_err": float(np.percentile(errs, 95)) if have else None,
        "config": asdict(cfg),
        "per_head": per_head,
    }
    with open(os.path.join(out_dir, "summary.json"), "w") as fh:
        json.dump(summary, fh, indent=2, sort_keys=True)
        fh.write("\n")
    return summary
