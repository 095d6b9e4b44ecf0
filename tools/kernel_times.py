"""Per-kernel CUDA-event timing of one LRQK layer at a given context
(development tool; prints one JSON line)."""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2510_23649_b200 import _lib
from paper_2510_23649_b200.engine import LayerShape, LayerState, prefill_factorize_device

p = argparse.ArgumentParser()
p.add_argument("--ctx", type=int, default=131072)
p.add_argument("--hq", type=int, default=32)
p.add_argument("--hkv", type=int, default=8)
p.add_argument("--batch", type=int, default=1)
p.add_argument("--rank", type=int, default=32)
p.add_argument("--topk", type=int, default=2048)
p.add_argument("--lite", type=int, default=16)
p.add_argument("--steps", type=int, default=6)
p.add_argument("--dtype", default="bf16")
p.add_argument("--policy", default="hbm")
p.add_argument("--no-prefill", action="store_true")
p.add_argument("--trace", default="compress")
a = p.parse_args()
dev = torch.device("cuda")
B, Hq, Hkv, d, r, l = a.batch, a.hq, a.hkv, 128, a.rank, a.ctx
sh = LayerShape(batch=B, n_q_heads=Hq, n_kv_heads=Hkv, head_dim=d, rank=r, k_budget=a.topk, lite_budget=a.lite,
                t_max=l + 64, dtype=a.dtype, policy=a.policy)
L = LayerState(sh, device=dev)
sdt = L.sdt
g = torch.Generator(device=dev); g.manual_seed(0)
Q = torch.randn(B * Hq, l, d, device=dev, generator=g).to(sdt)
K = torch.randn(B * Hkv, l, d, device=dev, generator=g).to(sdt)
V = torch.randn(B * Hkv, l, d, device=dev, generator=g).to(sdt)
if a.no_prefill:
    AK = torch.randn(B, Hq, l, r, device=dev, generator=g)
    BQ = torch.randn(B, Hq, r, d, device=dev, generator=g) / d ** 0.5
    BK = torch.randn(B, Hq, r, d, device=dev, generator=g) / d ** 0.5
    pf_ms = 0
else:
    t0 = time.time()
    res = prefill_factorize_device(Q, K, r, dtype=a.dtype, group=Hq // Hkv)
    torch.cuda.synchronize()
    pf_ms = (time.time() - t0) * 1e3
    AK, BQ, BK = res["A_K"].reshape(B, Hq, l, r), res["B_Q"].reshape(B, Hq, r, d), res["B_K"].reshape(B, Hq, r, d)
L.load_prompt(AK, BQ, BK, K.view(B, Hkv, l, d), V.view(B, Hkv, l, d))
lib = _lib.lib()
sp = _lib.stream_ptr()
q = torch.randn(B, Hq, d, device=dev, generator=g).to(sdt)
k = torch.randn(B, Hkv, d, device=dev, generator=g).to(sdt)
v = torch.randn(B, Hkv, d, device=dev, generator=g).to(sdt)
out = torch.zeros(B, Hq, d, device=dev)
names = ["compress", "score", "select_attend", "select", "gather", "attention", "prepare", "advance"]
calls = [lambda: lib.lrqk_decode_compress(L.ptr, q.data_ptr(), k.data_ptr(), v.data_ptr(), 1, sp),
         lambda: lib.lrqk_score(L.ptr, sp),
         lambda: lib.lrqk_select_attend(L.ptr, q.data_ptr(), out.data_ptr(), sp),
         lambda: lib.lrqk_select(L.ptr, sp),
         lambda: lib.lrqk_gather_misses(L.ptr, sp),
         lambda: lib.lrqk_attention(L.ptr, q.data_ptr(), out.data_ptr(), sp),
         lambda: lib.lrqk_compress_prepare(L.ptr, sp),
         lambda: lib.lrqk_advance(L.view("ctx_len").data_ptr(), B, sp)]
times = {n: [] for n in names}
for s in range(a.steps):
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(len(names) + 1)]
    torch.cuda._sleep(200000)  # let the host enqueue every launch before timing
    evs[0].record()
    for i, c in enumerate(calls):
        _lib.check(c(), names[i])
        evs[i + 1].record()
    torch.cuda.synchronize()
    for i, n in enumerate(names):
        times[n].append(evs[i].elapsed_time(evs[i + 1]) * 1e3)
st = int(L.view("status").item())
meta = L.buf["sel_meta"].view(torch.int32)[: B * Hq * 48].view(B * Hq, 48).cpu()
print("select modes", sorted(set(meta[:, 7].tolist())), "hint_ok", int(meta[:, 17].sum()), "fbin", meta[:4, 19].tolist(),
      "stats", meta[:, 33:40].sum(0).tolist())
import numpy as np
lib.lrqk_trace_enable(1)
ti = names.index(a.trace)
_lib.check(calls[ti](), a.trace)
torch.cuda.synchronize()
buf = np.zeros((65536, 2), dtype=np.uint64)
n = lib.lrqk_trace_read(buf.ctypes.data, 65536)
lib.lrqk_trace_enable(0)
rec = buf[:n]
t0 = rec[:, 1].min()
tags = (rec[:, 0] >> 48).astype(int)
for tag in sorted(set(tags)):
    ts = (rec[tags == tag, 1] - t0) / 1e3
    print(f"trace tag {tag}: n={len(ts)} min={ts.min():.1f}us med={np.median(ts):.1f}us max={ts.max():.1f}us")
res = {n: round(sum(v[1:]) / max(1, len(v) - 1), 2) for n, v in times.items()}
print(json.dumps(dict(us=res, status=st, prefill_ms=round(pf_ms, 1), miss=int(L.view("step_miss").sum()),
                      total=int(L.view("step_total").sum()), args=vars(a))))
