"""`python -m paper_2510_23649_b200.cli {synth,factorize,simulate}`: the
reference CLI's workload, factorisation and simulation subcommands with the
same flags, defaults, output files and exit codes (ref: cli.py:283-343),
driving the batched device runners of sim.py.  Heads run together on the
GPU instead of on a thread pool, so LRQK_THREADS has no effect.
"""

from __future__ import annotations

import argparse
import sys
from pathlib import Path

from .api import DecodeConfig, InitStrategy, PrefillConfig, SessionConfig
from .errors import CorruptTraceError, UnsupportedVersionError
from .workload import SyntheticSpec, as_heads, gen_recency_biased, load_trace, save_trace

SYNTH = dict(length=256, dim=64, rank_true=16, decay=0.9, recency=0.0, scale=1.0, seed=0, heads=1)


def _synth_flags(p):
    for name, typ in (("length", int), ("dim", int), ("rank_true", int), ("decay", float), ("recency", float),
                      ("scale", float), ("seed", int), ("heads", int)):
        p.add_argument("--" + name.replace("_", "-"), type=typ, dest=name)


def _prefill_flags(p):
    d = PrefillConfig()
    p.add_argument("--rank", type=int, default=d.rank)
    p.add_argument("--lambda-pq", type=float, default=d.lambda_q)
    p.add_argument("--lambda-pk", type=float, default=d.lambda_k)
    p.add_argument("--max-iter", type=int, default=d.max_iter)
    p.add_argument("--tol", type=float, default=d.tol)
    p.add_argument("--init", choices=["randn", "top", "topcol"], default=d.init.kind)
    p.add_argument("--init-seed", type=int, default=d.init.seed)


def _spec(a, head):
    v = {k: (getattr(a, k) if getattr(a, k) is not None else dflt) for k, dflt in SYNTH.items()}
    return SyntheticSpec(l=v["length"], d=v["dim"], r_true=v["rank_true"], decay=v["decay"],
                         recency_strength=v["recency"], seed=v["seed"] + head, scale=v["scale"])


def _heads(a, parser):
    if getattr(a, "trace", None) is not None:
        given = [k for k in SYNTH if getattr(a, k) is not None]
        if given:
            parser.error("--trace and synthetic workload flags are mutually exclusive "
                         f"(got {', '.join('--' + k.replace('_', '-') for k in given)})")
        return as_heads(load_trace(a.trace))
    n = a.heads if a.heads is not None else SYNTH["heads"]
    return [gen_recency_biased(_spec(a, h)) for h in range(n)]


def _prefill_cfg(a):
    return PrefillConfig(rank=a.rank, lambda_q=a.lambda_pq, lambda_k=a.lambda_pk, max_iter=a.max_iter, tol=a.tol,
                         init=InitStrategy(kind=a.init, seed=a.init_seed))


def cmd_synth(a, parser):
    heads = _heads(a, parser)
    save_trace(a.out, [(role, m) for qkv in heads for role, m in zip("qkv", qkv)])
    print(f"wrote {len(heads)} head(s) to {a.out}")
    return 0


def cmd_factorize(a, parser):
    from .sim import factorize

    runs = factorize(_heads(a, parser), _prefill_cfg(a), a.out_dir)
    for h, run in enumerate(runs):
        print(f"head {h}: {run.sweeps} sweep(s), {'converged' if run.converged else 'max-iter'}, "
              f"objective {run.objective[-1]:.6g}")
    return 0


def cmd_simulate(a, parser):
    from .sim import simulate

    heads = _heads(a, parser)
    cfg = SessionConfig(prefill=_prefill_cfg(a),
                        decode=DecodeConfig(lambda_1=a.lambda_d1, lambda_2=a.lambda_d2, max_iter=a.max_iter,
                                            tol=a.tol),
                        k_budget=a.topk, lite_budget=a.lite)
    s = simulate(heads, cfg, a.out_dir, prompt_len=a.prompt_len, steps=a.steps, compute_metrics=not a.no_metrics)
    rate = s["mean_miss_rate"]
    print(f"{s['heads']} head(s), {s['steps_per_head']} step(s), "
          f"miss rate {rate if rate is None else format(rate, '.4f')}")
    return 0


def build_parser():
    parser = argparse.ArgumentParser(prog="lrqk-b200", description="LRQK decode path on B200: workloads, "
                                     "prompt factorisation and decode simulation.")
    sub = parser.add_subparsers(dest="command", required=True)
    p = sub.add_parser("synth", help="write a synthetic workload to a trace file")
    _synth_flags(p)
    p.add_argument("--out", type=Path, required=True)
    p.set_defaults(func=cmd_synth)
    p = sub.add_parser("factorize", help="factor the prompt and report residuals")
    p.add_argument("--trace", type=Path)
    _synth_flags(p)
    _prefill_flags(p)
    p.add_argument("--out-dir", type=Path, required=True)
    p.set_defaults(func=cmd_factorize)
    p = sub.add_parser("simulate", help="full prefill + decode cache simulation")
    p.add_argument("--trace", type=Path)
    _synth_flags(p)
    _prefill_flags(p)
    s = SessionConfig()
    p.add_argument("--topk", type=int, default=s.k_budget)
    p.add_argument("--lite", type=int, default=s.lite_budget)
    p.add_argument("--lambda-d1", type=float, default=s.decode.lambda_1)
    p.add_argument("--lambda-d2", type=float, default=s.decode.lambda_2)
    p.add_argument("--prompt-len", type=int)
    p.add_argument("--steps", type=int)
    p.add_argument("--no-metrics", action="store_true")
    p.add_argument("--out-dir", type=Path, required=True)
    p.set_defaults(func=cmd_simulate)
    return parser


def main(argv=None) -> int:
    parser = build_parser()
    a = parser.parse_args(argv)
    try:
        return a.func(a, parser)
    except (CorruptTraceError, UnsupportedVersionError, OSError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 1
    except ValueError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
