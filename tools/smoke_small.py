import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2510_23649_b200.engine import LayerShape, LayerState
print("start", flush=True)
sh = LayerShape(batch=1, n_q_heads=2, n_kv_heads=1, head_dim=128, rank=32, k_budget=32, lite_budget=16, t_max=512, dtype="f32")
L = LayerState(sh)
l = 256
g = torch.Generator(device="cuda"); g.manual_seed(0)
AK = torch.randn(1, 2, l, 32, device="cuda", generator=g)
BQ = torch.randn(1, 2, 32, 128, device="cuda", generator=g) / 11
BK = torch.randn(1, 2, 32, 128, device="cuda", generator=g) / 11
K = torch.randn(1, 1, l, 128, device="cuda", generator=g)
V = torch.randn(1, 1, l, 128, device="cuda", generator=g)
L.load_prompt(AK, BQ, BK, K, V)
torch.cuda.synchronize(); print("seeded", flush=True)
q = torch.randn(1, 2, 128, device="cuda", generator=g)
k = torch.randn(1, 1, 128, device="cuda", generator=g)
v = torch.randn(1, 1, 128, device="cuda", generator=g)
out = torch.zeros(1, 2, 128, device="cuda")
from paper_2510_23649_b200 import _lib
lib = _lib.lib(); sp = _lib.stream_ptr()
for name, fn in [("compress", lambda: lib.lrqk_decode_compress(L.ptr, q.data_ptr(), k.data_ptr(), v.data_ptr(), 1, sp)),
                 ("score", lambda: lib.lrqk_score(L.ptr, sp)), ("select", lambda: lib.lrqk_select(L.ptr, sp)),
                 ("attention", lambda: lib.lrqk_attention(L.ptr, q.data_ptr(), out.data_ptr(), sp)),
                 ("prepare", lambda: lib.lrqk_compress_prepare(L.ptr, sp))]:
    _lib.check(fn(), name); torch.cuda.synchronize(); print(name, "ok", flush=True)
print("status", L.view("status").item(), out[0, 0, :4].tolist())
