import os, sys
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_2510_23649_b200 import _lib
from paper_2510_23649_b200.engine import LayerShape, LayerState
dev = torch.device("cuda")
B, Hq, Hkv, d, r, l = 1, 32, 8, 128, 32, 8192
sh = LayerShape(batch=B, n_q_heads=Hq, n_kv_heads=Hkv, head_dim=d, rank=r, k_budget=2048, lite_budget=16, t_max=l + 64, dtype="bf16")
L = LayerState(sh)
g = torch.Generator(device=dev); g.manual_seed(0)
L.load_prompt(torch.randn(B, Hq, l, r, device=dev, generator=g), torch.randn(B, Hq, r, d, device=dev, generator=g) / 11,
              torch.randn(B, Hq, r, d, device=dev, generator=g) / 11, torch.randn(B, Hkv, l, d, device=dev, generator=g).bfloat16(),
              torch.randn(B, Hkv, l, d, device=dev, generator=g).bfloat16())
q = torch.randn(B, Hq, d, device=dev, generator=g).bfloat16(); k = torch.randn(B, Hkv, d, device=dev, generator=g).bfloat16()
v = torch.randn(B, Hkv, d, device=dev, generator=g).bfloat16()
lib = _lib.lib(); sp = _lib.stream_ptr()
def run(n_rep, other):
    for _ in range(3):
        if other:  # evict the instruction cache with other kernels in between
            lib.lrqk_score(L.ptr, sp); lib.lrqk_select(L.ptr, sp)
        for _ in range(n_rep): lib.lrqk_decode_compress(L.ptr, q.data_ptr(), k.data_ptr(), v.data_ptr(), 0, sp)
    torch.cuda.synchronize()
    if other:
        lib.lrqk_score(L.ptr, sp); lib.lrqk_select(L.ptr, sp)
    torch.cuda.synchronize()
    for _ in range(n_rep - 1): lib.lrqk_decode_compress(L.ptr, q.data_ptr(), k.data_ptr(), v.data_ptr(), 0, sp)
    torch.cuda.synchronize()
    lib.lrqk_trace_enable(1)
    lib.lrqk_decode_compress(L.ptr, q.data_ptr(), k.data_ptr(), v.data_ptr(), 0, sp)
    torch.cuda.synchronize()
    buf = np.zeros((65536, 2), dtype=np.uint64); n = lib.lrqk_trace_read(buf.ctypes.data, 65536); lib.lrqk_trace_enable(0)
    rec = buf[:n]; t0 = rec[:, 1].min(); tags = (rec[:, 0] >> 48).astype(int)
    print("rep", n_rep, "other", other, " ".join(f"{t}:{np.median((rec[tags==t,1]-t0)/1e3):.1f}" for t in sorted(set(tags))))
run(1, True)
run(2, False)
run(3, False)
