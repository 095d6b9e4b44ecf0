"""Time the K1 prefill factorisation (tcgen05 Gram pass + float64 solve +
tcgen05 materialize) at a BASELINE shape and report per-kernel shares from
CUDA events around the whole call.  Usage: python tools/prefill_bench.py
[--ctx 131072] [--heads 32] [--kv 8] [--rank 32] [--reps 5]"""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2510_23649_b200.engine import prefill_factorize_device

ap = argparse.ArgumentParser()
ap.add_argument("--ctx", type=int, default=131072)
ap.add_argument("--heads", type=int, default=32)
ap.add_argument("--kv", type=int, default=8)
ap.add_argument("--rank", type=int, default=32)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--dtype", default="bf16")
a = ap.parse_args()
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev); g.manual_seed(0)
dt = torch.bfloat16 if a.dtype == "bf16" else torch.float32
Q = torch.randn(a.heads, a.ctx, 128, device=dev, generator=g).to(dt)
K = torch.randn(a.kv, a.ctx, 128, device=dev, generator=g).to(dt)
res = prefill_factorize_device(Q, K, a.rank, dtype=a.dtype, group=a.heads // a.kv)  # warm-up
torch.cuda.synchronize()
ts = []
for _ in range(a.reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); res = prefill_factorize_device(Q, K, a.rank, dtype=a.dtype, group=a.heads // a.kv); e1.record()
    torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
ms = sorted(ts)[len(ts) // 2]
e = Q.element_size()
rs = 32 if a.rank <= 32 else 64
# algorithmic bytes: two streams of Q and K (gram + materialize) + A writes (fp32, RS columns)
byts = 2 * (Q.numel() + K.numel()) * e + 2 * a.heads * a.ctx * rs * 4
print(json.dumps(dict(ctx=a.ctx, heads=a.heads, kv=a.kv, rank=a.rank, dtype=a.dtype, ms=round(ms, 3),
                      all_ms=[round(t, 3) for t in ts], algorithmic_GB=round(byts / 1e9, 3),
                      GBps=round(byts / ms / 1e6, 1), sweeps=res["sweeps"][:4].tolist(),
                      obj=res["objective"][0].tolist())))
