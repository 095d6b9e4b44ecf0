"""Sanitizer target for the fused score/select/attend kernel (development
tool): one layer, 2 q-heads x 8K context, so each head has 4 score parts and
the per-head barriers, the bin-D ranking and the partial merge all run;
three decode steps (the first takes the sampled-radix path, the others the
fused one)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2510_23649_b200.engine import LayerShape, LayerState

for dtype in ("bf16", "f32"):
    sh = LayerShape(batch=1, n_q_heads=2, n_kv_heads=1, head_dim=128, rank=32, k_budget=256, lite_budget=16,
                    t_max=8192 + 8, dtype=dtype)
    L = LayerState(sh)
    l = 8192
    g = torch.Generator(device="cuda"); g.manual_seed(0)
    sdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    L.load_prompt(torch.randn(1, 2, l, 32, device="cuda", generator=g),
                  torch.randn(1, 2, 32, 128, device="cuda", generator=g) / 11,
                  torch.randn(1, 2, 32, 128, device="cuda", generator=g) / 11,
                  torch.randn(1, 1, l, 128, device="cuda", generator=g).to(sdt),
                  torch.randn(1, 1, l, 128, device="cuda", generator=g).to(sdt))
    out = torch.zeros(1, 2, 128, device="cuda")
    for step in range(3):
        q = torch.randn(1, 2, 128, device="cuda", generator=g).to(sdt)
        k = torch.randn(1, 1, 128, device="cuda", generator=g).to(sdt)
        v = torch.randn(1, 1, 128, device="cuda", generator=g).to(sdt)
        L.step(q, k, v, out)
        torch.cuda.synchronize()
        L.raise_status()
    modes = L.view("sel_meta")[0, :, 7].tolist()
    print(dtype, "modes", modes, "out", out[0, 0, :3].tolist(), flush=True)
    if os.environ.get("LRQK_FUSED", "1") != "0":
        assert all(m == 6 for m in modes), modes  # the last step ran the fused path
print("fused ok")
