"""Host-side pieces of bench.py that the JSON line depends on (CPU only):
the algorithmic-bytes model of SURVEY §8(d), workload overrides, and the
ncu traffic lookup being tied to the captured launch shape."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def _args(**kw):
    a = argparse.Namespace(workload="c4", ctx=None, layers=None, rank=None, topk=None)
    for k, v in kw.items():
        setattr(a, k, v)
    return a


def test_step_bytes_match_survey_budget():
    """C4 per sequence: 359 MB per layer, 11.49 GB per token over 32 layers
    (SURVEY §8(d)); A_K is ~81 % of it (here t = ctx + 1 scores)."""
    w = bench.workload(_args())
    t, S = w["ctx"], w["k"] + w["lite"]
    b = bench.step_bytes(w, 1, t, S, 2)
    assert abs(b["total"] / 1e6 - 359.2) < 1.0
    assert abs(b["total"] * w["layers"] / 1e9 - 11.49) < 0.03
    assert 0.74 < b["a_k"] / b["total"] < 0.76 or 0.80 < b["a_k"] / b["total"] < 0.82


def test_workload_overrides_are_named():
    w = bench.workload(_args(rank=64, topk=4096))
    assert w["r"] == 64 and w["k"] == 4096
    assert "overridden" in w["desc"] and "r=64" in w["desc"] and "top-k=4096" in w["desc"]
    assert "overridden" not in bench.workload(_args())["desc"]


def test_ncu_traffic_only_for_the_captured_shape():
    """roofline.traffic comes from the committed ncu capture of the same
    workload, scaled to this launch's algorithmic bytes when they are within
    2 % (a few decode steps apart); otherwise it is null with a reason."""
    import json
    rec = json.load(open(os.path.join(os.path.dirname(bench.__file__), "profiles", "roofline_traffic.json")))["c4"]
    alg = int(rec["algorithmic_bytes_per_launch"])
    assert alg % (32 * (32 * 2 + 4)) == 0  # B*Hq*(t+1)*(R*e + 4) at C4
    got, src = bench._ncu_traffic("c4", alg)
    assert got == int(rec["dram_bytes_per_launch"]) and 0 < got <= alg * 1.05 and "ncu" in src
    got2, _ = bench._ncu_traffic("c4", alg + 50 * 32 * 68)  # 50 tokens later: scaled
    assert got2 == round(rec["dram_bytes_per_launch"] * (alg + 50 * 32 * 68) / alg)
    assert bench._ncu_traffic("c4", alg // 2)[0] is None  # another context length
    assert bench._ncu_traffic("c2", alg)[0] is None       # no capture for that workload


def test_reference_arm_config_matches_ours():
    a = bench.argparse.Namespace(workload="c4", ctx=None, layers=None, rank=None, topk=None, batch_per_gpu=1,
                                 policy="hbm", data="random")
    c = bench.config_dict(a, 1)
    for key in ("workload", "ctx", "layers", "n_q_heads", "n_kv_heads", "head_dim", "rank", "top_k", "lite",
                "global_batch", "slow_tier", "parallelism"):
        assert key in c


def test_global_batch_config_and_kv_head_split():
    """--global-batch fixes the job (strong scaling); with fewer sequences
    than GPUs the plan splits each sequence by KV-head blocks."""
    from paper_2510_23649_b200.shard import plan_shards

    a = bench.argparse.Namespace(workload="c4", ctx=None, layers=None, rank=None, topk=None, batch_per_gpu=1,
                                 global_batch=None, policy="hbm", data="random")
    assert bench.global_batch(a, 8) == 8 and bench.config_dict(a, 8)["batch_per_gpu"] == 1
    a.global_batch = 1
    c = bench.config_dict(a, 2)
    assert c["global_batch"] == 1 and c["batch_per_gpu"] == 0.5 and "KV-head" in c["parallelism"]
    plan = plan_shards(1, 32, 8, 2)
    assert [(s.b0, s.b1, s.g0, s.g1) for s in plan] == [(0, 1, 0, 4), (0, 1, 4, 8)]
    assert all(s.n_q_heads == 16 for s in plan)
