"""In-graph timeline of one decode step (development tool): an Engine with
--layers layers at --ctx is captured in a CUDA graph, replayed, and the
kernels' %globaltimer phase traces are printed relative to the step start
(min/median/max over blocks; with >1 layer the slots of later layers
overwrite earlier ones, so use --layers 1 or 2)."""
import argparse, os, sys
_ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, _ROOT)
# the product library is built without the trace; `make trace` builds this one
os.environ.setdefault("LRQK_LIB_PATH", os.path.join(_ROOT, "paper_2510_23649_b200", "liblrqk_b200_trace.so"))
import numpy as np
import torch
from paper_2510_23649_b200 import _lib
from paper_2510_23649_b200.engine import Engine, LayerShape

p = argparse.ArgumentParser()
p.add_argument("--ctx", type=int, default=131072)
p.add_argument("--layers", type=int, default=1)
p.add_argument("--batch", type=int, default=1)
p.add_argument("--fused-names", action="store_true", help="label the score_attend kernel's tags")
a = p.parse_args()
dev = torch.device("cuda")
B, Hq, Hkv, d, r, l = a.batch, 32, 8, 128, 32, a.ctx
sh = LayerShape(batch=B, n_q_heads=Hq, n_kv_heads=Hkv, head_dim=d, rank=r, k_budget=2048, lite_budget=16,
                t_max=l + 64, dtype="bf16")
eng = Engine(a.layers, sh, device=dev)
g = torch.Generator(device=dev); g.manual_seed(0)
for layer in eng.layers:
    AK = torch.randn(B, Hq, l, r, device=dev, generator=g)
    BQ = torch.randn(B, Hq, r, d, device=dev, generator=g) / d ** 0.5
    BK = torch.randn(B, Hq, r, d, device=dev, generator=g) / d ** 0.5
    K = torch.randn(B, Hkv, l, d, device=dev, generator=g).bfloat16()
    V = torch.randn(B, Hkv, l, d, device=dev, generator=g).bfloat16()
    layer.load_prompt(AK, BQ, BK, K, V)
eng.q_buf[..., :d].copy_(torch.randn(a.layers, B, Hq, d, device=dev, generator=g))
eng.k_buf[..., :d].copy_(torch.randn(a.layers, B, Hkv, d, device=dev, generator=g))
eng.v_buf[..., :d].copy_(torch.randn(a.layers, B, Hkv, d, device=dev, generator=g))
for _ in range(3):
    eng.decode_step()
torch.cuda.synchronize()
eng.capture()
for _ in range(3):
    eng.replay()
torch.cuda.synchronize()
lib = _lib.lib()
s0, e0 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s0.record(); eng.replay(); e0.record()
torch.cuda.synchronize()
print("graph step without tracing: %.1f us" % (s0.elapsed_time(e0) * 1e3))
lib.lrqk_trace_enable(1)
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record(); eng.replay(); e.record()
torch.cuda.synchronize()
buf = np.zeros((65536, 2), dtype=np.uint64)
n = lib.lrqk_trace_read(buf.ctypes.data, 65536)
lib.lrqk_trace_enable(0)
rec = buf[:n]
t0 = rec[:, 1].min()
tags = (rec[:, 0] >> 48).astype(int)
names = {0: "compress start", 1: "compress staged", 4: "compress B-update done", 40: "score start", 41: "score stream done",
         42: "score last-block", 43: "score end", 50: "sel_attend start", 51: "sel_attend meta", 52: "sel_attend part done",
         53: "sel_attend last-block", 54: "sel_attend end", 55: "sa crit sorted", 56: "sa part scanned", 44: "sa classified", 45: "sa crit flushed", 46: "sa cmask read", 47: "sa cands listed", 48: "sa keys classified", 49: "sa scanned",
         57: "sa part YG written", 58: "sa own partial", 59: "sa parts max", 60: "sa merged", 20: "select start", 30: "attention start", 10: "prepare start", 13: "finish YG summed", 7: "finish kernel start", 39: "attention merged (mode 5)", 8: "reduce kernel start", 9: "reduce kernel end", 35: "finish hits counted", 36: "finish B staged", 37: "finish B updated", 38: "finish grams",
         11: "prepare reduce done", 14: "prepare finish start", 16: "prepare end", 17: "prep idx staged", 18: "prep first chunk in", 19: "prep mma done", 61: "prep R gram", 62: "prep R GJ", 63: "prep pre-sync"}
if a.fused_names:
    names.update({41: "sa stream done", 42: "sa B1 passed", 46: "sa gwin loaded", 47: "sa D found", 48: "sa offsets",
                  49: "sa cands listed", 55: "sa keys classified", 58: "sa winners scanned", 44: "sa classified",
                  45: "sa B2 passed", 56: "sa lists ready", 59: "sa chunk 0 in", 60: "sa chunk 3 in", 52: "sa attended",
                  57: "sa partial written", 53: "sa last block", 54: "sa end"})
for tag in sorted(set(tags), key=lambda x: np.median(rec[tags == x, 1])):
    ts = (rec[tags == tag, 1] - t0) / 1e3
    print(f"tag {tag:3d} {names.get(tag, ''):24s} n={len(ts):4d} min={ts.min():7.1f} med={np.median(ts):7.1f} max={ts.max():7.1f} us")
print("graph step (events): %.1f us" % (s.elapsed_time(e) * 1e3))
if os.environ.get("TL_DUMP_TAG"):
    blk = (rec[:, 0] & 0xFFFFFF).astype(int)
    sm = ((rec[:, 0] >> 32) & 0xFFFF).astype(int)
    for tg in [int(x) for x in os.environ["TL_DUMP_TAG"].split(",")]:
        sel = tags == tg
        np.save("gpurun_out/tl_dump_%d.npy" % tg, np.stack([blk[sel], (rec[sel, 1] - t0) / 1e3, sm[sel]], 1))
