"""Benchmark of the LRQK decode-time sparse-attention path on B200.

Metric (BASELINE.json): decode tokens/s at 128K context with LLaMA-3-8B
attention shapes (32 layers, 32 q / 8 kv heads, d=128, r=32, top-k 2048,
16 recent tokens, bf16), plus the proxy-score kernel's HBM GB/s.

A "step" is one decode token for every sequence through all 32 layers:
per layer compress -> B update -> append -> proxy scores -> top-k select ->
hit/miss -> gather-fused attention.  Synthetic Q/K/V, the
prompt factorised on the GPU by the prefill kernels (K1).

    python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]

Multi-GPU (torchrun): weak scaling, --batch-per-gpu sequences per rank,
sharded by batch with no collective inside the step; the per-step
last-layer outputs are all-gathered over NCCL.  Timing is CUDA events,
max over ranks.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # name: layers, Hq, Hkv, d, ctx, r, k, lite, dtype
    "c4": dict(layers=32, hq=32, hkv=8, d=128, ctx=131072, r=32, k=2048, lite=16, dtype="bf16",
               desc="C4: LLaMA-3-8B attention shapes, 32 layers, 128K ctx, r=32, top-k 2048, 16 recent, bf16"),
    "c2": dict(layers=32, hq=32, hkv=8, d=128, ctx=32768, r=32, k=1024, lite=16, dtype="bf16",
               desc="C2: LLaMA-3-8B shapes, 32 layers, 32K ctx, r=32, top-k 1024, bf16"),
    "c3": dict(layers=28, hq=28, hkv=4, d=128, ctx=65536, r=32, k=2048, lite=16, dtype="bf16",
               desc="C3: Qwen2.5-7B shapes, 28 layers, 64K ctx, r=32, top-k 2048, bf16"),
    "c1": dict(layers=1, hq=32, hkv=8, d=128, ctx=4096, r=32, k=256, lite=16, dtype="f32",
               desc="C1: one layer, LLaMA-3-8B head shape, 4K ctx, r=32, top-k 256, fp32"),
}


def _ncu_traffic(workload_key, algorithmic_bytes):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the score
    kernel, from the committed ncu --set full capture of this workload
    (profiles/roofline_traffic.json, keyed by workload).  The capture was
    taken a few decode steps into the run; when this run's launch has the
    same algorithmic bytes within 2 % (same workload, context within a few
    hundred tokens), the captured DRAM bytes are scaled by the ratio of
    algorithmic bytes.  Returns (bytes, source) or (None, reason)."""
    try:
        with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "roofline_traffic.json")) as f:
            rec = json.load(f)[workload_key]
        alg0 = int(rec["algorithmic_bytes_per_launch"])
        if abs(algorithmic_bytes - alg0) > 0.02 * alg0:
            return None, f"no capture within 2% of {algorithmic_bytes} algorithmic bytes"
        dram = int(rec["dram_bytes_per_launch"])
        return int(round(dram * algorithmic_bytes / alg0)), rec["source"] + f" (scaled x{algorithmic_bytes / alg0:.5f})"
    except (OSError, ValueError, KeyError) as e:
        return None, f"no ncu capture for {workload_key}: {e.__class__.__name__}"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=50)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--workload", choices=sorted(WORKLOADS), default="c4")
    p.add_argument("--batch-per-gpu", type=int, default=1)
    p.add_argument("--global-batch", type=int, default=None,
                   help="fixed job batch (strong scaling); fewer sequences than GPUs splits each sequence by KV-head "
                        "blocks (shard.plan_shards). Default: batch-per-gpu x GPUs (weak scaling)")
    p.add_argument("--ctx", type=int, default=None)
    p.add_argument("--layers", type=int, default=None)
    p.add_argument("--rank", type=int, default=None)
    p.add_argument("--topk", type=int, default=None)
    p.add_argument("--policy", choices=["hbm", "host"], default="hbm")
    p.add_argument("--data", choices=["random", "recency", "drift"], default="random",
                   help="random: i.i.d. N(0,1) Q/K/V; recency: the reference's gen_recency_biased structure; "
                        "drift: AR(1)-correlated queries (paper-like top-k miss rate)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-sample-s", type=float, default=15.0)
    p.add_argument("--profile-steps", type=int, default=0,
                   help="only run N eager steps after setup (for ncu); prints nothing else")
    return p.parse_args()


def workload(args):
    w = dict(WORKLOADS[args.workload])
    if args.ctx:
        w["ctx"] = args.ctx
    if args.layers:
        w["layers"] = args.layers
    if args.rank:
        w["r"] = args.rank
    if args.topk:
        w["k"] = args.topk
    base = WORKLOADS[args.workload]
    over = [f"{name}={w[key]}" for key, name in (("ctx", "ctx"), ("layers", "layers"), ("r", "r"), ("k", "top-k"))
            if w[key] != base[key]]
    if over:  # the description names the overrides
        w["desc"] = base["desc"] + " [overridden: " + ", ".join(over) + "]"
    return w


def global_batch(args, world):
    gb = getattr(args, "global_batch", None)
    return gb if gb else args.batch_per_gpu * world


def config_dict(args, world):
    """The `config` object of the JSON line; identical for both arms."""
    w = workload(args)
    GB = global_batch(args, world)
    if world == 1:
        par = "1 GPU"
    elif GB % world == 0:
        par = (f"batch-sharded over {world} GPUs ({GB // world} sequence(s) each), no collective inside the step; "
               f"NCCL all-gather of last-layer outputs per step")
    else:
        par = (f"(sequence, KV-head block) shards over {world} GPUs ({world // GB} per sequence), no collective "
               f"inside the step; NCCL all-gather of last-layer outputs per step")
    return dict(workload=w["desc"], ctx=w["ctx"], layers=w["layers"], n_q_heads=w["hq"], n_kv_heads=w["hkv"],
                head_dim=w["d"], rank=w["r"], top_k=w["k"], lite=w["lite"], batch_per_gpu=GB // world if GB % world == 0 else GB / world,
                global_batch=GB, slow_tier=args.policy, data=args.data, parallelism=par,
                l2="no flush: each step streams %.1f GB (> 126 MB L2)" % (
                    step_bytes(w, GB, w["ctx"], w["k"] + w["lite"], 2 if w["dtype"] == "bf16" else 4)["total"]
                    * w["layers"] / max(world, 1) / 1e9))


# --------------------------------------------------------------------------
# distributed plumbing
# --------------------------------------------------------------------------
def dist_init(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if args.impl == "ours":
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    return world, rank, local


# --------------------------------------------------------------------------
# clocks sampled during the timed region
# --------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index=0):
        self.proc = None
        self.path = os.path.join(tempfile.gettempdir(), f"lrqk_clocks_{os.getpid()}.csv")
        self.dev = device_index

    def start(self):
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=self.fh, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.fh.close()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[5:9]):
                if val.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# --------------------------------------------------------------------------
# algorithmic bytes
# --------------------------------------------------------------------------
def step_bytes(w, B, t, S, e):
    """Per layer: A_K read, scores write+read, attention K/V gather,
    resident K/A reads for compression, B factors read+write."""
    Hq, d, r = w["hq"], w["d"], w["r"]
    a_k = B * Hq * t * r * e
    scores = 2 * B * Hq * t * 4
    attn = B * Hq * S * 2 * d * e
    resid = B * Hq * S * (d + r) * e
    bfac = B * Hq * 2 * r * d * 4 * 2
    return dict(a_k=a_k, scores=scores, attn=attn, resid=resid, bfac=bfac,
                total=a_k + scores + attn + resid + bfac)


# --------------------------------------------------------------------------
# structured synthetic data: the reference's gen_recency_biased
# (workload.py:87-107) with r_true=64, decay 0.95, recency 2.0, scale sqrt(T),
# drawn on the GPU (input synthesis only).  The q-heads of one KV group share
# the group's query directions (plus 10 % independent noise), so every one of
# them sees the recency structure of the shared keys.
# --------------------------------------------------------------------------
def recency_biased_heads(B, Hq, Hkv, T, d, gen, dev, r_true=64, decay=0.95, strength=2.0):
    import torch

    G = Hq // Hkv
    sig = math.sqrt(T) * decay ** torch.arange(r_true, device=dev, dtype=torch.float32)

    def lowrank():
        U = torch.linalg.qr(torch.randn(T, r_true, device=dev, generator=gen))[0]
        W = torch.linalg.qr(torch.randn(d, r_true, device=dev, generator=gen))[0]
        return (U * sig) @ W.T

    Q = torch.empty(B * Hq, T, d, device=dev)
    K = torch.empty(B * Hkv, T, d, device=dev)
    V = torch.randn(B * Hkv, T, d, device=dev, generator=gen)
    for bg in range(B * Hkv):
        Qg = lowrank()
        Kg = lowrank()
        Qn = Qg / (Qg * Qg).sum(1, keepdim=True).add_(1e-30)
        for lag in range(min(T - 1, 40) + 1):
            Kg[: T - lag].add_(Qn[lag:], alpha=strength * math.exp(-lag) * math.sqrt(d))
        K[bg] = Kg
        for j in range(G):
            h = (bg // Hkv) * Hq + (bg % Hkv) * G + j
            Q[h] = Qg + 0.1 * Qg.std() * torch.randn(T, d, device=dev, generator=gen)
    return Q, K, V


def drift_heads(B, Hq, Hkv, T, d, gen, dev, rho=0.9, r_true=64, decay=0.95, strength=2.0):
    """Temporally correlated queries: each q-head's latent coefficients follow
    an AR(1) process z_t = rho z_{t-1} + sqrt(1 - rho^2) e_t over the KV
    group's rank-64 key subspace, so consecutive queries pick overlapping
    top-k sets.  rho = 0.9 gives a top-k miss rate of ~0.45 per step, the
    regime the paper reports (~0.40) and the one the GPU
    cache (K5) and the pinned host tier (K5b) are built for.  Keys: the
    group's low-rank subspace plus the reference's recency bias toward the
    group's queries (workload.py:87-107)."""
    import torch

    G = Hq // Hkv
    sq = decay ** torch.arange(r_true, device=dev, dtype=torch.float32)
    sk = math.sqrt(T) * sq
    Q = torch.empty(B * Hq, T, d, device=dev)
    K = torch.empty(B * Hkv, T, d, device=dev)
    V = torch.randn(B * Hkv, T, d, device=dev, generator=gen)
    for bg in range(B * Hkv):
        W = torch.linalg.qr(torch.randn(d, r_true, device=dev, generator=gen))[0]
        U = torch.linalg.qr(torch.randn(T, r_true, device=dev, generator=gen))[0]
        Kg = (U * sk) @ W.T
        for j in range(G):
            z = math.sqrt(1 - rho * rho) * torch.randn(T, r_true, device=dev, generator=gen)
            z[0] /= math.sqrt(1 - rho * rho)
            shift = 1
            while shift < T:  # z_t = sum_j rho^j e_{t-j}, by doubling
                z[shift:] += rho ** shift * z[:-shift].clone()
                shift *= 2
            h = (bg // Hkv) * Hq + (bg % Hkv) * G + j
            Q[h] = (z * sq) @ W.T
        Qg = Q[(bg // Hkv) * Hq + (bg % Hkv) * G]
        Qn = Qg / (Qg * Qg).sum(1, keepdim=True).add_(1e-30)
        for lag in range(min(T - 1, 40) + 1):
            Kg[: T - lag].add_(Qn[lag:], alpha=strength * math.exp(-lag) * math.sqrt(d))
        K[bg] = Kg
    return Q, K, V


# --------------------------------------------------------------------------
# our arm
# --------------------------------------------------------------------------
def run_ours(args, world, rank, local):
    import ctypes as C

    import torch
    import torch.distributed as dist

    from paper_2510_23649_b200 import _lib
    from paper_2510_23649_b200.engine import Engine, LayerShape, prefill_factorize_device

    from paper_2510_23649_b200.shard import gather_outputs, plan_shards

    w = workload(args)
    dev = torch.device("cuda", local)
    GB = global_batch(args, world)
    # this rank's (sequence, KV-head) block of the job: whole
    # sequences when the GPUs divide the batch, else KV-head blocks
    plan = plan_shards(GB, w["hq"], w["hkv"], world)
    shard = plan[rank]
    B = shard.batch
    L, d, ctx, r, k, lite = w["layers"], w["d"], w["ctx"], w["r"], w["k"], w["lite"]
    Hq, Hkv = shard.n_q_heads, shard.n_kv_heads
    extra_steps = args.warmup + args.steps + max(args.profile_steps, 0) + 64
    t_max = ctx + 2 * extra_steps
    shape = LayerShape(batch=B, n_q_heads=Hq, n_kv_heads=Hkv, head_dim=d, rank=r, k_budget=k, lite_budget=lite,
                       t_max=t_max, dtype=w["dtype"], policy=args.policy)
    eng = Engine(L, shape, device=dev)
    sdt = torch.bfloat16 if w["dtype"] == "bf16" else torch.float32
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234 + rank)

    # ---- prompt: synthetic Q/K/V, factorised by the GPU prefill kernels ----
    # recency data: `pool` rows past the prompt are the decode rows, so the
    # decode queries continue the prompt's structure
    pool = 8 if args.data == "random" else 64
    torch.cuda.synchronize()
    t0 = time.time()
    prefill_ms = 0.0
    prefill_layer_ms = []
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    q_pool = torch.empty(pool, L, B, Hq, d, device=dev, dtype=sdt)
    k_pool = torch.empty(pool, L, B, Hkv, d, device=dev, dtype=sdt)
    v_pool = torch.empty_like(k_pool)
    for li, layer in enumerate(eng.layers):
        if args.data != "random":
            gen_heads = recency_biased_heads if args.data == "recency" else drift_heads
            Qa, Ka, Va = gen_heads(B, Hq, Hkv, ctx + pool, d, gen, dev)
            q_pool[:, li] = Qa[:, ctx:].reshape(B, Hq, pool, d).permute(2, 0, 1, 3).to(sdt)
            k_pool[:, li] = Ka[:, ctx:].reshape(B, Hkv, pool, d).permute(2, 0, 1, 3).to(sdt)
            v_pool[:, li] = Va[:, ctx:].reshape(B, Hkv, pool, d).permute(2, 0, 1, 3).to(sdt)
            Qp, Kp, Vp = (x[:, :ctx].to(sdt).contiguous() for x in (Qa, Ka, Va))
            del Qa, Ka, Va
        else:
            Qp = torch.randn(B * Hq, ctx, d, device=dev, generator=gen).to(sdt)
            Kp = torch.randn(B * Hkv, ctx, d, device=dev, generator=gen).to(sdt)
            Vp = torch.randn(B * Hkv, ctx, d, device=dev, generator=gen).to(sdt)
        ev0.record()
        res = prefill_factorize_device(Qp, Kp, r, dtype=w["dtype"], group=Hq // Hkv, want_a_q=False)
        ev1.record()
        torch.cuda.synchronize()
        prefill_layer_ms.append(ev0.elapsed_time(ev1))
        prefill_ms += prefill_layer_ms[-1]
        layer.load_prompt(res["A_K"].reshape(B, Hq, ctx, r), res["B_Q"].reshape(B, Hq, r, d),
                          res["B_K"].reshape(B, Hq, r, d), Kp.view(B, Hkv, ctx, d), Vp.view(B, Hkv, ctx, d))
        del Qp, Kp, Vp, res
    torch.cuda.synchronize()
    setup_s = time.time() - t0

    # ---- per-step inputs: a pool of synthetic decode rows ------------------
    if args.data == "random":
        q_pool = torch.randn(pool, L, B, Hq, d, device=dev, generator=gen).to(sdt)
        k_pool = torch.randn(pool, L, B, Hkv, d, device=dev, generator=gen).to(sdt)
        v_pool = torch.randn(pool, L, B, Hkv, d, device=dev, generator=gen).to(sdt)

    def load_inputs(i):
        eng.q_buf[..., :d].copy_(q_pool[i % pool], non_blocking=True)
        eng.k_buf[..., :d].copy_(k_pool[i % pool], non_blocking=True)
        eng.v_buf[..., :d].copy_(v_pool[i % pool], non_blocking=True)

    if args.profile_steps > 0:  # eager steps for ncu
        for i in range(args.profile_steps):
            load_inputs(i)
            eng.decode_step()
        torch.cuda.synchronize()
        eng.raise_status()
        return None

    # ---- warm up, capture -----------------------------------------------------
    for i in range(2):
        load_inputs(i)
        eng.decode_step()
    torch.cuda.synchronize()
    eng.raise_status()
    eng.capture()
    gather_buf = None
    if world > 1:
        gather_buf = torch.empty(GB, w["hq"], shape.dim_stride, device=dev)

    def one_step(i):
        load_inputs(i)
        eng.replay()
        if world > 1:  # final per-head output gather over NVLink (NCCL)
            gather_outputs(eng.out_buf[-1], plan, out=gather_buf)

    step_i = 2
    for _ in range(args.warmup):
        one_step(step_i)
        step_i += 1
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    cm0, ct0 = eng.counters()
    miss0, tot0 = cm0.sum().item(), ct0.sum().item()  # cumulative CacheStats over layers and heads
    if world > 1:
        dist.barrier()
    start.record()
    for _ in range(args.steps):
        one_step(step_i)
        step_i += 1
    stop.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clock_info = clocks.stop()
    ms = start.elapsed_time(stop)
    # miss transfers of the timed steps: with the host slow tier every miss is
    # one K row + one V row read from pinned host memory over PCIe (K5b)
    cm1, ct1 = eng.counters()
    misses = cm1.sum().item() - miss0
    selected = ct1.sum().item() - tot0
    miss_bytes = misses * 2 * d * (2 if w["dtype"] == "bf16" else 4)
    eng.raise_status()
    t_now = int(eng.ctx[0].item())
    # selection path statistics (head-steps per mode, since the prompt)
    mstat = np.zeros(7, dtype=np.int64)
    for layer in eng.layers:
        m = layer.buf["sel_meta"].view(torch.int32)[: B * Hq * 48].view(B * Hq, 48)
        mstat += m[:, 33:40].sum(0).cpu().numpy()
    sel_modes = dict(zip(["sampled_radix", "all_fit", "unused", "window_scan", "unused4", "window_direct",
                          "exact_fallback"],
                         [int(x) for x in mstat]))

    # ---- end to end: host inputs in, host outputs out, per step ------------
    # the same input sequence as the timed loop (the whole pool, continuing at
    # step_i), so the selections -- and the host tier's misses -- match it
    q_host = q_pool.cpu().pin_memory()
    k_host = k_pool.cpu().pin_memory()
    v_host = v_pool.cpu().pin_memory()
    out_host = torch.empty(L, B, Hq, shape.dim_stride, dtype=torch.float32).pin_memory()
    h2d = (q_host[0].numel() + k_host[0].numel() + v_host[0].numel()) * q_host.element_size()
    d2h = out_host.numel() * 4
    e2e_steps = max(5, args.steps // 2)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(e2e_steps):
        j = (step_i + i) % pool
        eng.q_buf[..., :d].copy_(q_host[j], non_blocking=True)
        eng.k_buf[..., :d].copy_(k_host[j], non_blocking=True)
        eng.v_buf[..., :d].copy_(v_host[j], non_blocking=True)
        eng.replay()
        if world > 1:
            gather_outputs(eng.out_buf[-1], plan, out=gather_buf)
        out_host.copy_(eng.out_buf, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1)
    step_i += e2e_steps

    # ---- dominant kernel (proxy score) timed on its stream ------------------
    lib = _lib.lib()
    stream = torch.cuda.current_stream()
    sp = _lib.stream_ptr(stream)
    n_prof = 3
    evs = []
    for i in range(n_prof):
        load_inputs(step_i)
        step_i += 1
        for li, layer in enumerate(eng.layers):
            q, kk, vv, out = eng.q_buf[li], eng.k_buf[li], eng.v_buf[li], eng.out_buf[li]
            _lib.check(lib.lrqk_decode_compress(layer.ptr, q.data_ptr(), kk.data_ptr(), vv.data_ptr(), 1, sp), "compress")
            a, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            _lib.check(lib.lrqk_score(layer.ptr, sp), "score")
            b_.record(stream)
            evs.append((a, b_))
            _lib.check(lib.lrqk_select_attend(layer.ptr, q.data_ptr(), out.data_ptr(), sp), "select_attend")
            _lib.check(lib.lrqk_select(layer.ptr, sp), "select")
            _lib.check(lib.lrqk_attention(layer.ptr, q.data_ptr(), out.data_ptr(), sp), "attention")
        _lib.check(lib.lrqk_compress_prepare_layers(eng._dev_layers.data_ptr(), eng._host_layers, L, sp), "prepare")
        _lib.check(lib.lrqk_advance(eng.ctx.data_ptr(), B, sp), "advance")
    torch.cuda.synchronize()
    eng.raise_status()
    score_ms = float(np.mean([a.elapsed_time(b_) for a, b_ in evs]))

    # ---- the product's dominant kernel: fused score/select/attend ----------
    # (the step's K3+K4+K6; timed per launch on its stream, as above)
    fused_ms = None
    if eng.fused:
        evs = []
        for i in range(n_prof):
            load_inputs(step_i)
            step_i += 1
            for li, layer in enumerate(eng.layers):
                q, kk, vv, out = eng.q_buf[li], eng.k_buf[li], eng.v_buf[li], eng.out_buf[li]
                _lib.check(lib.lrqk_decode_compress(layer.ptr, q.data_ptr(), kk.data_ptr(), vv.data_ptr(), 1, sp),
                           "compress")
                a, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                _lib.check(lib.lrqk_score_attend(layer.ptr, q.data_ptr(), out.data_ptr(), sp), "score_attend")
                b_.record(stream)
                evs.append((a, b_))
                _lib.check(lib.lrqk_select(layer.ptr, sp), "select")
                _lib.check(lib.lrqk_attention(layer.ptr, q.data_ptr(), out.data_ptr(), sp), "attention")
            _lib.check(lib.lrqk_compress_prepare_layers(eng._dev_layers.data_ptr(), eng._host_layers, L, sp),
                       "prepare")
            _lib.check(lib.lrqk_advance(eng.ctx.data_ptr(), B, sp), "advance")
        torch.cuda.synchronize()
        eng.raise_status()
        fused_ms = float(np.mean([a.elapsed_time(b_) for a, b_ in evs]))

    # ---- fidelity of the last step (f1, outside every timed region) --------
    rec, err = eng.fidelity()
    fid = torch.stack([rec.mean(), err[torch.isfinite(err)].mean()]).double()

    # ---- aggregate over ranks ------------------------------------------------
    vals = torch.tensor([ms, e2e_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(vals, op=dist.ReduceOp.MAX)
        dist.all_reduce(fid, op=dist.ReduceOp.SUM)
        fid /= world
    ms, e2e_ms = float(vals[0]), float(vals[1])
    total_seq = GB
    ms_per_step = ms / args.steps
    tok_s = total_seq * args.steps / (ms / 1e3)
    e2e_tok_s = total_seq * e2e_steps / (e2e_ms / 1e3)

    S = k + lite
    e = 2 if w["dtype"] == "bf16" else 4
    t_mid = t_now  # context during the profile steps
    byt = step_bytes(dict(w, hq=Hq), B, t_mid, S, e)
    score_bytes = B * Hq * (t_mid + 1) * (r * e + 4)  # A_K read + key write per launch
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    score_gbs = score_bytes / (score_ms / 1e3) / 1e9
    traffic, traffic_src = _ncu_traffic(args.workload if args.policy == "hbm" else None, score_bytes)
    step_gbs = byt["total"] * L / (ms_per_step / 1e3) / 1e9
    peak_src = "MEASURED_PEAKS.json hbm_gbs (copy, burst)" if peaks else "fallback 6650"
    k3 = dict(bound="hbm", kernel="score_tma_kernel (split path: proxy scores + window histogram)",
              achieved=round(score_gbs, 1), peak=hbm_peak, unit="GB/s", frac=round(score_gbs / hbm_peak, 4),
              traffic=traffic, traffic_source=traffic_src, algorithmic_bytes_per_launch=score_bytes,
              avg_launch_ms=round(score_ms, 5), step_frac_of_hbm=round(step_gbs / hbm_peak, 4),
              step_algorithmic_GBps=round(step_gbs, 1), peak_source=peak_src)
    if fused_ms is not None:
        # fused kernel: A_K read + keys write/read + the selected rows' K, V
        # and proxy rows (SURVEY §8d terms a_k + scores + attn + the A half of resid)
        sa_bytes = B * Hq * ((t_mid + 1) * (r * e + 8) + S * (2 * d + r) * e)
        sa_gbs = sa_bytes / (fused_ms / 1e3) / 1e9
        sa_traffic, sa_src = _ncu_traffic(f"{args.workload}:score_attend" if args.policy == "hbm" else None, sa_bytes)
        roofline = dict(bound="hbm", kernel="score_attend_kernel (fused K3+K4+K6: proxy scores, top-k, attention)",
                        achieved=round(sa_gbs, 1), peak=hbm_peak, unit="GB/s", frac=round(sa_gbs / hbm_peak, 4),
                        traffic=sa_traffic, traffic_source=sa_src, algorithmic_bytes_per_launch=sa_bytes,
                        avg_launch_ms=round(fused_ms, 5), step_frac_of_hbm=round(step_gbs / hbm_peak, 4),
                        step_algorithmic_GBps=round(step_gbs, 1), peak_source=peak_src, split_path_score_kernel=k3)
    else:
        roofline = k3
    return dict(
        metric="decode tokens/s at 128K ctx (LLaMA-3-8B shape); proxy-score HBM GB/s",
        value=round(tok_s, 3), unit="tokens/s", n_gpus=world, steps=args.steps, warmup=args.warmup,
        ms_per_step=round(ms_per_step, 4), higher_is_better=True,
        scaling="strong" if args.global_batch else "weak", vs_baseline=None,
        dtype=w["dtype"],
        data={"random": "synthetic (random N(0,1) Q/K/V per layer; prompt factorised on GPU)",
              "recency": "synthetic recency-biased low-rank Q/K (reference gen_recency_biased structure, r_true=64, "
                         "decay 0.95, strength 2, scale sqrt(T)); decode rows continue the prompt; prompt factorised "
                         "on GPU",
              "drift": "synthetic AR(1)-correlated queries (rho 0.9) over a rank-64 key subspace with the reference's "
                       "recency bias; decode rows continue the prompt; prompt factorised on GPU"}[args.data],
        config=config_dict(args, world),
        roofline=roofline,
        miss_transfers=dict(misses_per_step=round(misses / max(args.steps, 1), 1),
                            miss_rate=round(misses / max(selected, 1), 4),
                            bytes_per_step=int(miss_bytes / max(args.steps, 1)),
                            host_tier_GBps=round(miss_bytes / (ms / 1e3) / 1e9, 2) if args.policy == "host" else None,
                            note="host policy: K5b zero-copy PCIe reads of the missed K/V rows; "
                                 "HBM policy: misses are counted, the rows are already in HBM"),
        e2e=dict(value=round(e2e_tok_s, 3), unit="tokens/s", h2d_bytes_per_step=int(h2d),
                 d2h_bytes_per_step=int(d2h), steps=e2e_steps,
                 path="Engine public API: pinned host q/k/v -> H2D -> graph replay -> D2H outputs"),
        gpu_launches=eng.launches_per_step() * args.steps,
        clocks=clock_info,
        prefill=dict(ms_total_gpu=round(prefill_ms, 2), heads=L * B * Hq, ctx=ctx, setup_s=round(setup_s, 2),
                     ms_first_layer=round(prefill_layer_ms[0], 2),
                     ms_per_layer_median=round(sorted(prefill_layer_ms)[len(prefill_layer_ms) // 2], 3),
                     note="per layer: B*Hq query heads and B*Hkv key heads of ctx rows through "
                          "prefill_factorize_device (A_Q not materialised: decode reads A_K, B_Q, B_K); "
                          "the first call includes the one-time module load and init-draw upload"),
        bytes_per_token_layer=byt,
        select_paths=sel_modes,
        fidelity=dict(recall_mean=round(float(fid[0]), 5), output_err_mean=round(float(fid[1]), 6),
                      heads=L * GB * w["hq"], step=t_now - 1,
                      note="Engine.fidelity on the device after the timed steps: Omega_t vs the exact top-k of q K^T "
                           "over the whole history, and output vs full-history attention (ref session.py:119-131)"),
    )


# --------------------------------------------------------------------------
# CPU arm: the oracle port of the reference (numpy fp64), bounded sample
# --------------------------------------------------------------------------
def _cpu_session(ctx, d, r, k, lite, seed):
    """One reference head session (oracle port) at `ctx` tokens of context."""
    from oracle import lrqk_oracle as O

    rng = np.random.default_rng(seed)
    K = rng.standard_normal((ctx, d))
    V = rng.standard_normal((ctx, d))
    P = rng.standard_normal((ctx, r))
    BQ = rng.standard_normal((r, d)) / math.sqrt(d)
    BK = rng.standard_normal((r, d)) / math.sqrt(d)
    st = O.seed_head(K, V, O.Factors(None, P, BQ, BK), k, lite)
    return st, rng


def _cpu_worker(argtuple):
    """warm + n timed head-steps of one session; returns seconds per step."""
    ctx, d, r, k, lite, warm, n_steps, seed = argtuple
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    from oracle import lrqk_oracle as O

    st, rng = _cpu_session(ctx, d, r, k, lite, seed)
    for _ in range(max(1, warm)):  # the first step fills the resident set to its steady-state size
        O.head_step(st, rng.standard_normal(d), rng.standard_normal(d), rng.standard_normal(d))
    t0 = time.perf_counter()
    for _ in range(n_steps):
        O.head_step(st, rng.standard_normal(d), rng.standard_normal(d), rng.standard_normal(d))
    return (time.perf_counter() - t0) / n_steps


def _thread_pool_rate(w, cores, n_steps):
    """The reference CLI's own fan-out: one session per thread on a
    ThreadPoolExecutor (cli.py:126-137).  Head-steps per second."""
    from concurrent.futures import ThreadPoolExecutor

    from oracle import lrqk_oracle as O

    sess = [_cpu_session(w["ctx"], w["d"], w["r"], w["k"], w["lite"], 100 + i) for i in range(cores)]
    for st, rng in sess:
        O.head_step(st, rng.standard_normal(w["d"]), rng.standard_normal(w["d"]), rng.standard_normal(w["d"]))

    def run(i):
        st, rng = sess[i]
        for _ in range(n_steps):
            O.head_step(st, rng.standard_normal(w["d"]), rng.standard_normal(w["d"]), rng.standard_normal(w["d"]))

    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=cores) as pool:
        list(pool.map(run, range(cores)))
    return cores * n_steps / (time.perf_counter() - t0)


def _cpu_prefill_s(w):
    """Oracle prefill_run of one head at the workload's context (1 core)."""
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    from oracle import lrqk_oracle as O

    rng = np.random.default_rng(7)
    Q = rng.standard_normal((w["ctx"], w["d"]))
    K = rng.standard_normal((w["ctx"], w["d"]))
    t0 = time.perf_counter()
    O.factorize(Q, K, rank=w["r"])
    return time.perf_counter() - t0


def _process_pool_rate(w, cores, warm, n_steps):
    import multiprocessing as mp

    # one BLAS thread per process: set before the spawned children import numpy
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    os.environ["OMP_NUM_THREADS"] = "1"
    with mp.get_context("spawn").Pool(cores) as pool:
        t0 = time.perf_counter()
        per = pool.map(_cpu_worker, [(w["ctx"], w["d"], w["r"], w["k"], w["lite"], warm, n_steps, 1 + i)
                                     for i in range(cores)])
        wall = time.perf_counter() - t0
    return cores / float(np.mean(per)), float(np.mean(per)), wall


def cpu_baseline(w, total_seq, budget_s=15.0):
    """Reference CPU path on this host's cores (reported next to our arm, not
    the target): the oracle port of DecodeSession.decode_step, one head
    session per process (processes = cores; the GIL makes the reference's
    own thread fan-out nearly serial), extrapolated to the whole job
    (layers x q-heads x sequences head sessions per token; heads are
    independent).  Also: the thread-pool variant the reference
    CLI uses, and the single-head prefill time."""
    cores = os.cpu_count() or 1
    probe = _cpu_worker((w["ctx"], w["d"], w["r"], w["k"], w["lite"], 1, 1, 0))
    n_steps = max(2, min(500, int(budget_s / max(probe, 1e-3) / 2)))
    rate, per, wall = _process_pool_rate(w, cores, 1, n_steps)
    sessions = w["layers"] * w["hq"] * total_seq
    tok_s = rate / sessions * total_seq
    threads = min(cores, 8)  # the GIL serialises them anyway; 8 sessions bound the host memory
    thr_steps = max(2, min(50, int(5.0 / max(probe * threads, 1e-3))))
    thr_rate = _thread_pool_rate(w, threads, thr_steps)
    pre_s = _cpu_prefill_s(w)
    return dict(value=round(tok_s, 5), unit="tokens/s", cores=cores, kind="port",
                sample=f"{cores} processes x 1 head session ({w['ctx']} ctx, k={w['k']}, r={w['r']}, fp64 numpy "
                       f"oracle) x {n_steps} timed decode steps after 1 warm step; {per * 1e3:.1f} ms/head-step; "
                       f"extrapolated to {sessions} head sessions per token (layers x q-heads x sequences)",
                ms_per_head_step=round(per * 1e3, 3), wall_s=round(wall, 1),
                thread_pool=dict(value=round(thr_rate / sessions * total_seq, 5), unit="tokens/s", threads=threads,
                                 head_steps_per_s=round(thr_rate, 2),
                                 sample=f"{threads} threads x {thr_steps} head-steps (reference cli.py:126-137 fan-out)"),
                prefill=dict(s_per_head=round(pre_s, 2), heads_per_token_batch=sessions,
                             sample=f"oracle prefill_run, one head, {w['ctx']} x {w['d']}, r={w['r']}, 1 core"))


def run_reference(args, world, rank):
    """--impl reference: the reference's CPU path timed on this host's cores.
    Each of the K timed steps is one decode step of `cores` independent head
    sessions (one per process) after W untimed ones; tokens/s is then
    extrapolated to the whole job's head sessions (reported explicitly)."""
    w = workload(args)
    total_seq = global_batch(args, world)
    if rank != 0:
        return None
    cores = os.cpu_count() or 1
    t0 = time.perf_counter()
    rate, per, _ = _process_pool_rate(w, cores, max(1, args.warmup), args.steps)
    wall = time.perf_counter() - t0
    sessions = w["layers"] * w["hq"] * total_seq
    tok_s = rate / sessions * total_seq
    cfg = config_dict(args, world)
    return dict(metric="decode tokens/s at 128K ctx (LLaMA-3-8B shape); proxy-score HBM GB/s",
                value=round(tok_s, 5), unit="tokens/s", n_gpus=world, steps=args.steps, warmup=args.warmup,
                ms_per_step=round(1e3 * total_seq / tok_s, 3), higher_is_better=True,
                scaling="strong" if args.global_batch else "weak", vs_baseline=None, dtype="f64", data="synthetic (random N(0,1) K/V/proxy rows per head session)",
                config=cfg, impl="reference",
                cpu_baseline=dict(value=round(tok_s, 5), unit="tokens/s", cores=cores, kind="port",
                                  sample=f"{cores} processes x 1 head session, {args.warmup} warm + {args.steps} timed "
                                         f"decode steps each ({w['ctx']} ctx, k={w['k']}, r={w['r']}, fp64 numpy "
                                         f"oracle); {per * 1e3:.1f} ms/head-step"),
                extrapolation=dict(head_sessions_per_token=sessions, timed_head_steps=cores * args.steps,
                                   processes=cores, rule="tokens/s = head-steps/s / head sessions per token x sequences"),
                e2e=dict(value=round(tok_s, 5), unit="tokens/s", h2d_bytes_per_step=0, d2h_bytes_per_step=0,
                         note="CPU path: inputs and outputs never leave host memory"),
                wall_s=round(wall, 1))


def main():
    args = parse()
    world, rank, local = dist_init(args)
    if args.impl == "reference":
        out = run_reference(args, world, rank)
        if out is not None:
            print(json.dumps(out), flush=True)
        return
    res = run_ours(args, world, rank, local)
    if res is None:
        return
    if rank == 0:
        if not args.no_cpu_baseline and world == 1:
            res["cpu_baseline"] = cpu_baseline(workload(args), res["config"]["global_batch"], args.cpu_sample_s)
        else:
            res["cpu_baseline"] = None
        print(json.dumps(res), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
