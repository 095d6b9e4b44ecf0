import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2510_23649_b200 as lrqk
from paper_2510_23649_b200.workload import load_trace, as_heads
from paper_2510_23649_b200.engine import LayerShape, LayerState
from tests.lrqk_testlib import StepLocked, ParityLog, rows_dev
heads = as_heads(load_trace("tests/golden/cli/workload.lrqk"))
cfg = lrqk.PrefillConfig(rank=8)
H = 3
runs = [lrqk.prefill_run(h[0][:64], h[1][:64], cfg) for h in heads]
Q = np.stack([h[0] for h in heads])[None]; K = np.stack([h[1] for h in heads])[None]; V = np.stack([h[2] for h in heads])[None]
for hsel in [None]:
    sh = LayerShape(batch=1, n_q_heads=H, n_kv_heads=H, head_dim=32, rank=8, k_budget=24, lite_budget=8, t_max=130, dtype="f32")
    L = LayerState(sh)
    f32 = lambda x: torch.as_tensor(np.asarray(x), dtype=torch.float32, device="cuda")
    L.load_prompt(f32(np.stack([r.factors.A_K for r in runs]))[None], f32(np.stack([r.factors.B_Q for r in runs]))[None],
                  f32(np.stack([r.factors.B_K for r in runs]))[None], f32(K[:, :, :64]), f32(V[:, :, :64]))
    lock = StepLocked(L, Q, K, V, 64)
    log = ParityLog("dbg")
    out = torch.zeros(1, H, 32, device="cuda")
    for t in range(64, 80):
        L.step(rows_dev(Q[:, :, t], L), rows_dev(K[:, :, t], L), rows_dev(V[:, :, t], L), out)
        torch.cuda.synchronize(); L.raise_status()
        try:
            lock.check_step(out, log, "f32", rtol_hat=2e-3)
        except AssertionError as e:
            print("t", t, "FAIL", str(e)[:500]); break
        print("t", t, "ok", L.view("step_miss")[0].tolist())
    print({k: (len(v) if isinstance(v, list) else v) for k, v in log.rec.items()})
