"""Generate the golden fixtures that pin the oracle (and, through it, the
CUDA path) to the REFERENCE implementation.

Run in the development container, where the reference package is readable:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

It imports the reference ``lrqk`` package, drives its public API on seeded
inputs and stores inputs + outputs in ``tests/golden/*.npz``.  Nothing at test
or bench time reads /root/reference; only these committed files travel.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

import lrqk  # noqa: E402  (the reference)


def _save(name, **arrays):
    path = os.path.join(HERE, f"{name}.npz")
    np.savez_compressed(path, **arrays)
    return path


def gen_topk():
    rng = np.random.default_rng(1000)
    cases = []
    for _ in range(60):
        n = int(rng.integers(1, 300))
        k = int(rng.integers(1, n + 4))
        quant = int(rng.integers(0, 3))  # 0: raw, 1: 1-decimal, 2: heavy ties
        s = rng.standard_normal(n)
        if quant == 1:
            s = np.round(s, 1)
        elif quant == 2:
            s = np.round(s)
        if rng.random() < 0.2:
            s[rng.integers(0, n, size=max(1, n // 4))] = -0.0
        cases.append((s, k, lrqk.topk_indices(s, k)))
    flat = {}
    for i, (s, k, out) in enumerate(cases):
        flat[f"s{i}"] = s
        flat[f"k{i}"] = np.array(k)
        flat[f"o{i}"] = np.asarray(out, dtype=np.int64)
    flat["n"] = np.array(len(cases))
    _save("topk", **flat)


def gen_select():
    rng = np.random.default_rng(1001)
    flat = {}
    n = 80
    for i in range(n):
        t = int(rng.integers(0, 400))
        kb = int(rng.integers(1, 70))
        lb = int(rng.integers(1, 20))
        s = np.round(rng.standard_normal(t + 1), int(rng.integers(0, 3)))
        sel = lrqk.select_active(s, t, kb, lb)
        flat[f"s{i}"] = s
        flat[f"p{i}"] = np.array([t, kb, lb])
        flat[f"ok{i}"] = sel.omega_k.astype(np.int64)
        flat[f"ol{i}"] = sel.omega_l.astype(np.int64)
        flat[f"o{i}"] = sel.omega.astype(np.int64)
    flat["n"] = np.array(n)
    _save("select", **flat)


def gen_scores_attention():
    rng = np.random.default_rng(1002)
    flat = {}
    for i in range(10):
        t, r, d, n = int(rng.integers(1, 500)), [4, 16, 32][i % 3], [8, 64, 128][i % 3], int(rng.integers(1, 300))
        store = rng.standard_normal((t, r))
        qh = rng.standard_normal((1, r))
        flat[f"store{i}"] = store
        flat[f"qh{i}"] = qh
        flat[f"sc{i}"] = lrqk.proxy_scores(qh, store)
        q = rng.standard_normal((1, d))
        K = rng.standard_normal((n, d)) * (3.0 if i % 2 else 1.0)
        V = rng.standard_normal((n, d))
        res = lrqk.exact_attention(q, K, V)
        flat[f"q{i}"] = q
        flat[f"K{i}"] = K
        flat[f"V{i}"] = V
        flat[f"out{i}"] = res.output
        flat[f"w{i}"] = res.weights
    flat["n"] = np.array(10)
    _save("scores_attention", **flat)


def gen_compress():
    rng = np.random.default_rng(1003)
    flat = {}
    shapes = [(8, 3, 5), (16, 4, 0), (64, 16, 40), (128, 32, 272), (128, 32, 17)]
    i = 0
    for rep in range(3):
        for d, r, nres in shapes:
            f = lrqk.LowRankFactors(
                A_Q=np.zeros((1, r)), A_K=np.zeros((1, r)),
                B_Q=rng.standard_normal((r, d)) / np.sqrt(d),
                B_K=rng.standard_normal((r, d)) / np.sqrt(d),
            )
            step = lrqk.TokenStep(q=rng.standard_normal((1, d)), k=rng.standard_normal((1, d)),
                                  v=rng.standard_normal((1, d)))
            A_res = rng.standard_normal((nres, r))
            K_res = rng.standard_normal((nres, d))
            cfg = lrqk.DecodeConfig(max_iter=[2, 2, 5][rep], tol=[1e-2, 1e-2, 1e-6][rep])
            comp, ws = lrqk.decode_compress(step, f, A_res, K_res, cfg)
            ws2 = lrqk.DecodeWorkspace()
            new = lrqk.update_projections(step, comp, f, ws2)
            for key, val in dict(q=step.q, k=step.k, B_Q=f.B_Q, B_K=f.B_K, A_res=A_res, K_res=K_res,
                                 cfg=np.array([cfg.lambda_1, cfg.lambda_2, cfg.max_iter, cfg.tol]),
                                 q_hat=comp.q_hat, k_hat=comp.k_hat, M_rq=ws.M_rq, m_lq=ws.m_lq,
                                 B_Q_new=new.B_Q, B_K_new=new.B_K,
                                 eta=np.array([ws2.eta_Q, ws2.eta_K])).items():
                flat[f"{key}{i}"] = val
            i += 1
    flat["n"] = np.array(i)
    _save("compress", **flat)


def gen_spd():
    rng = np.random.default_rng(1004)
    flat = {}
    Ms = [np.eye(2), np.diag([2.0, 4.0]), np.array([[1.0, 1.0], [1.0, 1.0]])]
    RHSs = [np.array([[5.0, 7.0]]), np.array([[2.0, 4.0]]), np.array([[1.0, 1.0]])]
    for _ in range(6):
        A = rng.standard_normal((40, 32))
        Ms.append(A.T @ A + 0.1 * np.eye(32))
        RHSs.append(rng.standard_normal((1, 32)))
    # rank-deficient 32x32 (needs jitter)
    A = rng.standard_normal((8, 32))
    Ms.append(A.T @ A)
    RHSs.append(rng.standard_normal((1, 32)))
    for i, (M, R) in enumerate(zip(Ms, RHSs)):
        flat[f"M{i}"] = M
        flat[f"R{i}"] = R
        flat[f"X{i}"] = lrqk.solve_spd(M, R)
    flat["n"] = np.array(len(Ms))
    _save("spd", **flat)


def gen_prefill():
    flat = {}
    cases = [
        dict(l=64, d=16, r=4, seed=3, scale=1.0, max_iter=2, tol=1e-2, init="randn", iseed=0),
        dict(l=96, d=24, r=6, seed=4, scale=1.0, max_iter=5, tol=1e-30, init="top", iseed=0),
        dict(l=80, d=16, r=4, seed=5, scale=100.0, max_iter=25, tol=1e-12, init="topcol", iseed=0),
        dict(l=256, d=128, r=32, seed=6, scale=1.0, max_iter=2, tol=1e-2, init="randn", iseed=0),
    ]
    for i, c in enumerate(cases):
        spec = lrqk.SyntheticSpec(l=c["l"], d=c["d"], r_true=min(c["r"] * 2, c["d"]), seed=c["seed"],
                                  scale=c["scale"])
        Q, K, V = lrqk.gen_lowrank_qk(spec)
        rng = np.random.default_rng(77 + i)
        Q = Q + 0.01 * rng.standard_normal(Q.shape)
        K = K + 0.01 * rng.standard_normal(K.shape)
        cfg = lrqk.PrefillConfig(rank=c["r"], max_iter=c["max_iter"], tol=c["tol"],
                                 init=lrqk.InitStrategy(c["init"], c["iseed"]))
        run = lrqk.prefill_run(Q, K, cfg)
        f = run.factors
        flat.update({f"Q{i}": Q, f"K{i}": K, f"A_Q{i}": f.A_Q, f"A_K{i}": f.A_K, f"B_Q{i}": f.B_Q,
                     f"B_K{i}": f.B_K, f"obj{i}": np.array(run.objective),
                     f"sweeps{i}": np.array(run.sweeps), f"conv{i}": np.array(run.converged),
                     f"res{i}": np.array(lrqk.factor_residuals(Q, K, f)),
                     f"cfg{i}": np.array([c["r"], c["max_iter"], c["tol"]]),
                     f"init{i}": np.array(c["init"])})
    flat["n"] = np.array(len(cases))
    _save("prefill", **flat)


def gen_sessions():
    """Full DecodeSession runs; every per-step observable is stored."""
    flat = {}
    cases = [
        dict(l=120, prompt=60, d=16, r=4, kb=8, lb=4, seed=5, recency=0.0),
        dict(l=200, prompt=100, d=32, r=8, kb=24, lb=8, seed=6, recency=2.0),
        dict(l=360, prompt=300, d=128, r=32, kb=64, lb=16, seed=7, recency=2.0),
    ]
    for i, c in enumerate(cases):
        spec = lrqk.SyntheticSpec(l=c["l"], d=c["d"], r_true=min(2 * c["r"], c["d"]), decay=0.95,
                                  seed=c["seed"], recency_strength=c["recency"],
                                  scale=float(np.sqrt(c["l"])))
        Q, K, V = lrqk.gen_recency_biased(spec)
        # float32-representable inputs, like a trace file carries
        Q, K, V = (x.astype(np.float32).astype(np.float64) for x in (Q, K, V))
        cfg = lrqk.SessionConfig(prefill=lrqk.PrefillConfig(rank=c["r"]), decode=lrqk.DecodeConfig(),
                                 k_budget=c["kb"], lite_budget=c["lb"])
        sess = lrqk.DecodeSession(cfg)
        f0 = sess.prefill(Q[: c["prompt"]], K[: c["prompt"]], V[: c["prompt"]])
        f0 = f0.copy()
        omegas, outs, misses, totals, qh, kh, BQ, BK = [], [], [], [], [], [], [], []
        for t in range(c["prompt"], c["l"]):
            rep = sess.decode_step(Q[t], K[t], V[t], compute_metrics=False)
            omegas.append(sess.last_selection.omega.astype(np.int64))
            outs.append(sess.last_output.ravel())
            misses.append(rep.miss_count)
            totals.append(rep.selected_count)
            kh.append(sess.cache.proxy_store[t].copy())
            BQ.append(sess.factors.B_Q.copy())
            BK.append(sess.factors.B_K.copy())
        steps = c["l"] - c["prompt"]
        width = max(len(o) for o in omegas)
        om = np.full((steps, width), -1, dtype=np.int64)
        for j, o in enumerate(omegas):
            om[j, : len(o)] = o
        flat.update({f"Q{i}": Q, f"K{i}": K, f"V{i}": V,
                     f"A_Q0_{i}": f0.A_Q, f"A_K0_{i}": f0.A_K, f"B_Q0_{i}": f0.B_Q, f"B_K0_{i}": f0.B_K,
                     f"omega{i}": om, f"out{i}": np.array(outs), f"miss{i}": np.array(misses),
                     f"total{i}": np.array(totals), f"khat{i}": np.array(kh),
                     f"BQ{i}": np.array(BQ[::10] + BQ[-1:]), f"BK{i}": np.array(BK[::10] + BK[-1:]),
                     f"cfg{i}": np.array([c["prompt"], c["r"], c["kb"], c["lb"]]),
                     f"c_miss{i}": np.array(sess.stats.c_miss), f"c_total{i}": np.array(sess.stats.c_total)})
    flat["n"] = np.array(len(cases))
    _save("sessions", **flat)


def gen_dense():
    """The per-call linear algebra of the reference: gram, fro_norm_sq,
    update_B/AK/AQ, lagrangian_value, factor_residuals, khat_initial_guess,
    update_qhat/khat, and top-k on float64 scores closer than float32 can
    resolve."""
    rng = np.random.default_rng(1007)
    flat = {}
    i = 0
    for l, d, r, lq, lk in [(64, 16, 4, 1.0, 1.0), (200, 32, 8, 0.5, 2.0), (300, 128, 32, 1.0, 1.0),
                            (40, 24, 6, 0.0, 0.0)]:
        Q = rng.standard_normal((l, d))
        K = rng.standard_normal((l, d)) * 2.0
        f = lrqk.LowRankFactors(A_Q=rng.standard_normal((l, r)), A_K=rng.standard_normal((l, r)),
                                B_Q=rng.standard_normal((r, d)) / np.sqrt(d), B_K=rng.standard_normal((r, d)) / np.sqrt(d))
        cfg = lrqk.PrefillConfig(rank=r, lambda_q=lq, lambda_k=lk)
        flat.update({f"Q{i}": Q, f"K{i}": K, f"A_Q{i}": f.A_Q, f"A_K{i}": f.A_K, f"B_Q{i}": f.B_Q, f"B_K{i}": f.B_K,
                     f"lam{i}": np.array([lq, lk]),
                     f"gram{i}": lrqk.gram(f.A_Q), f"gramT{i}": lrqk.gram(f.B_K.T), f"fro{i}": np.array(lrqk.fro_norm_sq(Q)),
                     f"uB{i}": lrqk.update_B(f.A_Q, Q), f"uAK{i}": lrqk.update_AK(Q, K, f, cfg),
                     f"uAQ{i}": lrqk.update_AQ(Q, K, f, cfg), f"lag{i}": np.array(lrqk.lagrangian_value(Q, K, f, cfg)),
                     f"res{i}": np.array(lrqk.factor_residuals(Q, K, f))})
        # decode-side closed forms on a resident set
        nres = [5, 0, 272, 3][i]
        step = lrqk.TokenStep(q=rng.standard_normal((1, d)), k=rng.standard_normal((1, d)), v=rng.standard_normal((1, d)))
        A_res, K_res = rng.standard_normal((nres, r)), rng.standard_normal((nres, d))
        dcfg = lrqk.DecodeConfig(lambda_1=[1.0, 0.5, 1.0, 2.0][i], lambda_2=[1.0, 1.5, 1.0, 0.0][i])
        comp = lrqk.CompressedToken(q_hat=rng.standard_normal((1, r)), k_hat=rng.standard_normal((1, r)))
        ws = lrqk.DecodeWorkspace()
        flat.update({f"q{i}": step.q, f"k{i}": step.k, f"v{i}": step.v, f"A_res{i}": A_res, f"K_res{i}": K_res,
                     f"dlam{i}": np.array([dcfg.lambda_1, dcfg.lambda_2]), f"qh_in{i}": comp.q_hat,
                     f"kh_in{i}": comp.k_hat,
                     f"kh0{i}": lrqk.khat_initial_guess(step.k, f.B_K),
                     f"uq{i}": lrqk.update_qhat(step, comp, f, A_res, K_res, dcfg, ws),
                     f"m_lq{i}": ws.m_lq, f"M_rq{i}": ws.M_rq,
                     f"uk{i}": lrqk.update_khat(step, comp, f, dcfg)})
        i += 1
    flat["n"] = np.array(i)
    # float64 scores that differ below float32 resolution
    base = rng.standard_normal(500)
    s = np.repeat(base[:50], 10) + np.tile(np.arange(10) * 1e-12, 50)
    rng.shuffle(s)
    flat["tk_s"] = s
    flat["tk_o"] = lrqk.topk_indices(s, 37)
    _save("dense", **flat)


CLI_SYNTH = ["--length", "128", "--dim", "32", "--rank-true", "32", "--decay", "0.95", "--recency", "2.0", "--scale", "11.3",
             "--seed", "5", "--heads", "3"]
CLI_SIM = ["--rank", "8", "--topk", "24", "--lite", "8", "--prompt-len", "64"]


def gen_cli():
    """Outputs of the reference CLI (`lrqk synth / factorize / simulate`) on a
    small recency-biased workload: the trace bytes and every output file."""
    import shutil
    import tempfile

    from lrqk.cli import main as cli_main

    root = os.path.join(HERE, "cli")
    shutil.rmtree(root, ignore_errors=True)
    os.makedirs(root)
    trace = os.path.join(root, "workload.lrqk")
    assert cli_main(["synth", *CLI_SYNTH, "--out", trace]) == 0
    with tempfile.TemporaryDirectory() as tmp:
        for name, argv in (("simulate_nometrics", ["simulate", "--trace", trace, *CLI_SIM, "--no-metrics"]),
                           ("simulate_metrics", ["simulate", "--trace", trace, *CLI_SIM, "--steps", "24"]),
                           ("factorize", ["factorize", "--trace", trace, "--rank", "8", "--max-iter", "6",
                                          "--tol", "1e-9"])):
            out = os.path.join(tmp, name)
            assert cli_main([*argv, "--out-dir", out]) == 0
            shutil.copytree(out, os.path.join(root, name))
    with open(os.path.join(root, "ARGS.json"), "w") as fh:
        json.dump({"synth": CLI_SYNTH, "simulate": CLI_SIM}, fh, indent=1)


def main():
    gen_topk()
    gen_select()
    gen_scores_attention()
    gen_compress()
    gen_spd()
    gen_prefill()
    gen_sessions()
    gen_dense()
    gen_cli()
    manifest = {"reference_version": lrqk.__version__, "numpy": np.__version__,
                "files": sorted(f for f in os.listdir(HERE) if f.endswith(".npz"))}
    with open(os.path.join(HERE, "MANIFEST.json"), "w") as fh:
        json.dump(manifest, fh, indent=1, sort_keys=True)
    print(json.dumps(manifest))


if __name__ == "__main__":
    main()
