"""LRQK trace-file I/O and the synthetic workload generators against the
reference's own bytes (tests/golden/cli/workload.lrqk, written by the
reference CLI `lrqk synth`), and the reference's error classes for corrupt
files (ref: workload.py:145-216, cli.py:333-343).  Host code, no GPU."""

import json
import os
import struct

import numpy as np
import pytest

from paper_2510_23649_b200 import cli
from paper_2510_23649_b200.errors import CorruptTraceError, UnsupportedVersionError
from paper_2510_23649_b200.workload import (SyntheticSpec, as_heads, gen_lowrank_qk, gen_recency_biased, load_trace,
                                            save_trace)

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "cli")
TRACE = os.path.join(GOLD, "workload.lrqk")


def _synth_args():
    return json.load(open(os.path.join(GOLD, "ARGS.json")))["synth"]


def test_generators_reproduce_the_reference_trace_bytes(tmp_path):
    """`synth` with the reference's arguments writes the reference's bytes."""
    out = tmp_path / "w.lrqk"
    assert cli.main(["synth", *_synth_args(), "--out", str(out)]) == 0
    assert out.read_bytes() == open(TRACE, "rb").read()


def test_load_save_round_trip(tmp_path):
    recs = load_trace(TRACE)
    assert [r.role for r in recs] == ["q", "k", "v"] * 3
    heads = as_heads(recs)
    assert len(heads) == 3 and heads[0][0].shape == (128, 32) and heads[0][0].dtype == np.float64
    out = tmp_path / "rt.lrqk"
    save_trace(out, [(r.role, r.data) for r in recs])
    assert out.read_bytes() == open(TRACE, "rb").read()


def test_recency_zero_is_the_plain_generator():
    s = SyntheticSpec(l=40, d=8, r_true=4, seed=2)
    a, b = gen_lowrank_qk(s), gen_recency_biased(s)
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x, y)
    sv = np.linalg.svd(a[0], compute_uv=False)
    np.testing.assert_allclose(sv[:4], 0.9 ** np.arange(4), rtol=1e-10)
    with pytest.raises(ValueError):
        SyntheticSpec(l=4, d=4, r_true=5)


def test_corrupt_traces_raise_the_reference_errors(tmp_path):
    blob = open(TRACE, "rb").read()
    cases = {
        "magic": (b"XRQK" + blob[4:], CorruptTraceError),
        "version": (blob[:4] + struct.pack("<H", 2) + blob[6:], UnsupportedVersionError),
        "header": (blob[:6] + blob[6:10], CorruptTraceError),
        "payload": (blob[:-3], CorruptTraceError),
        "tag": (blob[:6] + bytes([7]) + blob[7:], CorruptTraceError),
        "short": (b"LRQ", CorruptTraceError),
    }
    for name, (data, exc) in cases.items():
        p = tmp_path / f"{name}.lrqk"
        p.write_bytes(data)
        with pytest.raises(exc):
            load_trace(p)
    # the CLI maps trace errors to exit code 1 (ref: cli.py:338-340)
    assert cli.main(["factorize", "--trace", str(tmp_path / "magic.lrqk"), "--out-dir", str(tmp_path / "o")]) == 1
    recs = load_trace(TRACE)
    with pytest.raises(CorruptTraceError, match="triples"):
        as_heads(recs[:4])
    with pytest.raises(CorruptTraceError, match="roles"):
        as_heads([recs[1], recs[0], recs[2]])
    with pytest.raises(ValueError, match="role"):
        save_trace(tmp_path / "bad.lrqk", [("x", np.zeros((2, 2)))])


def test_trace_and_synthetic_flags_are_exclusive(tmp_path):
    with pytest.raises(SystemExit):
        cli.main(["simulate", "--trace", TRACE, "--length", "10", "--out-dir", str(tmp_path)])
