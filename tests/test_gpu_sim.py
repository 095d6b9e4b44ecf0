"""`simulate` / `factorize` outputs against the reference CLI's own files
(tests/golden/cli/, written by `lrqk simulate|factorize` on the committed
trace).  All heads run as one batched device layer (sim.py).

  * simulate --no-metrics: every file byte-identical (report_hNNN.csv,
    cache_hNNN.csv, miss_hist.csv, summary.json);
  * simulate with metrics: cache / miss-hist files byte-identical, the
    report's step, selected, miss and recall columns identical, output_err
    within 1e-4 relative (fp32 attention vs float64);
  * factorize: lagrangian.csv / residuals.csv within the fp32 prefill's
    tolerance;
  * load_trace_device equals load_trace.
"""

import csv
import json
import os

import numpy as np
import pytest
import torch

from paper_2510_23649_b200 import cli
from paper_2510_23649_b200.workload import load_trace, load_trace_device

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "cli")
TRACE = os.path.join(GOLD, "workload.lrqk")
SIM = json.load(open(os.path.join(GOLD, "ARGS.json")))["simulate"]


def _files(d):
    return sorted(os.listdir(d))


def test_load_trace_device():
    Q, K, V = load_trace_device(TRACE)
    recs = load_trace(TRACE)
    assert Q.shape == (3, 128, 32) and Q.dtype == torch.float32 and Q.is_cuda
    for i, (role, t) in enumerate(zip("qkv" * 3, [Q[0], K[0], V[0], Q[1], K[1], V[1], Q[2], K[2], V[2]])):
        assert recs[i].role == role
        np.testing.assert_array_equal(t.cpu().numpy().astype(np.float64), recs[i].data)


def test_simulate_no_metrics_is_byte_identical(tmp_path):
    out = tmp_path / "sim"
    assert cli.main(["simulate", "--trace", TRACE, *SIM, "--no-metrics", "--out-dir", str(out)]) == 0
    ref = os.path.join(GOLD, "simulate_nometrics")
    assert _files(out) == _files(ref)
    for name in _files(ref):
        assert (out / name).read_bytes() == open(os.path.join(ref, name), "rb").read(), name


def test_simulate_with_metrics(tmp_path):
    out = tmp_path / "sim"
    assert cli.main(["simulate", "--trace", TRACE, *SIM, "--steps", "24", "--out-dir", str(out)]) == 0
    ref = os.path.join(GOLD, "simulate_metrics")
    assert _files(out) == _files(ref)
    for name in _files(ref):
        got, want = (out / name).read_text(), open(os.path.join(ref, name)).read()
        if name.startswith("cache_") or name == "miss_hist.csv":
            assert got == want, name
        elif name.startswith("report_"):
            g, w = list(csv.reader(got.splitlines())), list(csv.reader(want.splitlines()))
            assert g[0] == w[0] and len(g) == len(w)
            for a, b in zip(g[1:], w[1:]):
                assert a[:4] == b[:4], (name, a, b)  # step, selected, miss, recall: exact
                assert float(a[4]) == pytest.approx(float(b[4]), rel=1e-4, abs=1e-7)
        else:
            g, w = json.loads(got), json.loads(want)
            for key in ("heads", "prompt_len", "steps_per_head", "mean_miss_rate", "mean_recall", "config"):
                assert g[key] == w[key], key
            for key in ("p50_output_err", "p95_output_err"):
                assert g[key] == pytest.approx(w[key], rel=1e-4)


def test_factorize_matches_reference(tmp_path):
    out = tmp_path / "fact"
    assert cli.main(["factorize", "--trace", TRACE, "--rank", "8", "--max-iter", "6", "--tol", "1e-9",
                     "--out-dir", str(out)]) == 0
    ref = os.path.join(GOLD, "factorize")
    g = list(csv.reader((out / "lagrangian.csv").read_text().splitlines()))
    w = list(csv.reader(open(os.path.join(ref, "lagrangian.csv")).read().splitlines()))
    assert g[0] == w[0] and [r[:2] for r in g] == [r[:2] for r in w]  # same sweeps per head
    for a, b in zip(g[1:], w[1:]):
        assert float(a[2]) == pytest.approx(float(b[2]), rel=2e-3, abs=1e-3)
    g = list(csv.reader((out / "residuals.csv").read_text().splitlines()))
    w = list(csv.reader(open(os.path.join(ref, "residuals.csv")).read().splitlines()))
    assert g[0] == w[0]
    for a, b in zip(g[1:], w[1:]):
        assert a[0] == b[0]
        for x, y in zip(a[1:], b[1:]):
            assert float(x) == pytest.approx(float(y), rel=2e-3, abs=2e-6)
