import sys, os
sys.path.insert(0, "/root/repo")
import torch, numpy as np
from tests.lrqk_testlib import make_layer
from paper_2510_23649_b200.engine import prefill_factorize_device
r, kb = int(sys.argv[1]), int(sys.argv[2])
B, Hq, Hkv, d, lb, ctx = 1, 4, 1, 128, 16, 24000
dev = torch.device("cuda")
for trial in range(6):
    torch.manual_seed(1)
    Qp = torch.randn(B * Hq, ctx, d, device=dev).to(torch.bfloat16)
    Kp = torch.randn(B * Hkv, ctx, d, device=dev).to(torch.bfloat16)
    Vp = torch.randn(B * Hkv, ctx, d, device=dev).to(torch.bfloat16)
    res = prefill_factorize_device(Qp, Kp, r, dtype="bf16", group=Hq // Hkv)
    layer = make_layer(B, Hq, Hkv, d, r, kb, lb, t_max=ctx + 16, dtype="bf16")
    layer.load_prompt(res["A_K"].reshape(B, Hq, ctx, r), res["B_Q"].reshape(B, Hq, r, d),
                      res["B_K"].reshape(B, Hq, r, d), Kp.view(B, Hkv, ctx, d), Vp.view(B, Hkv, ctx, d))
    out = torch.zeros(B, Hq, d, device=dev)
    Kall, Vall = Kp.view(B, Hkv, ctx, d).float(), Vp.view(B, Hkv, ctx, d).float()
    for t in range(ctx, ctx + 6):
        q = torch.randn(B, Hq, d, device=dev).to(torch.bfloat16)
        k = torch.randn(B, Hkv, d, device=dev).to(torch.bfloat16)
        v = torch.randn(B, Hkv, d, device=dev).to(torch.bfloat16)
        layer.step(q, k, v, out)
        torch.cuda.synchronize()
        Kall = torch.cat([Kall, k.float()[:, :, None]], 2)
        Vall = torch.cat([Vall, v.float()[:, :, None]], 2)
        cnt = layer.view("res_cnt").cpu(); idx = layer.view("res_idx").cpu()
        meta = layer.buf["sel_meta"][: B * Hq * 48 * 4].view(torch.int32).cpu()
        for h in range(Hq):
            sel = idx[0, h, : int(cnt[0, h])].long().to(dev)
            Ks, Vs = Kall[0, 0][sel], Vall[0, 0][sel]
            w = torch.softmax(q[0, h].float() @ Ks.T / d ** 0.5, -1)
            ref = w @ Vs
            err = (out[0, h] - ref).abs().max().item()
            if err > 1e-2:
                m = meta.reshape(B, Hq, -1)[0, h]
                print(f"trial {trial} t {t} h {h} err {err:.3f} cnt {int(cnt[0,h])} mode {int(m[7])} nabove {int(m[20])} P {int(m[22])}")
                P = 11; tiles = (t + 1 + 31) // 32; tpp = (tiles + P - 1) // P
                s = sel.tolist()
                groups = {"certain": s[:255], "binD": s[255:256], "lite": s[256:]}
                for p_ in range(P):
                    groups[f"part{p_}"] = [x for x in s[:255] if p_ * tpp * 32 <= x < (p_ + 1) * tpp * 32]
                nslot = 17 if False else None
                asc = layer.buf["attn_scratch"].view(torch.float32)
                # slots per head = max(splits, P + 1); find by scanning: use M_ATT_PARTS and try splits
                for slots in (12, 17, 16, 18, 24, 32):
                    base = (h * slots) * (d + 2)
                    ok = True
                    res_parts = []
                    for p_ in range(P + 1):
                        part = asc[base + p_ * (d + 2): base + (p_ + 1) * (d + 2)]
                        l_ = part[1].item()
                        if not (l_ > 0): ok = False; break
                        res_parts.append(part[2:] / l_)
                    if not ok: continue
                    print("   slots", slots)
                    for p_ in range(P):
                        rows = groups[f"part{p_}"] + (groups["lite"] if p_ == P - 1 else [])
                        kk = torch.tensor(rows, device=dev)
                        w2 = torch.softmax(q[0, h].float() @ Kall[0, 0][kk].T / d ** 0.5, -1)
                        e2 = (res_parts[p_] - w2 @ Vall[0, 0][kk]).abs().max().item()
                        print(f"   part {p_} partial err {e2:.4f} (rows {len(rows)})")
                    kk = torch.tensor(groups["binD"], device=dev)
                    w2 = torch.softmax(q[0, h].float() @ Kall[0, 0][kk].T / d ** 0.5, -1)
                    print(f"   slot P (binD) err {(res_parts[P] - w2 @ Vall[0, 0][kk]).abs().max().item():.4f}")
                    break
                si = layer.buf["sure_idx"].view(torch.int32).cpu()
                for p_ in range(P):
                    reg = si[(h * P + p_) * kb:(h * P + p_ + 1) * kb]
                    nl = int(reg[kb - 1]); sl = int(reg[kb - 2])
                    lst = reg[:nl].tolist()
                    want = groups[f"part{p_}"] + (groups["lite"] if p_ == P - 1 else [])
                    print(f"   part {p_} shortlist {sl} nloc {nl} list==want {sorted(lst)==sorted(want)} dup {len(lst)-len(set(lst))} extra {sorted(set(lst)-set(want))[:6]} missing {sorted(set(want)-set(lst))[:6]}")
                for gname, gl in groups.items():
                    keep = [x for x in s if x not in set(gl)]
                    if not keep: continue
                    kk = torch.tensor(keep, device=dev)
                    w2 = torch.softmax(q[0, h].float() @ Kall[0, 0][kk].T / d ** 0.5, -1)
                    e2 = (out[0, h] - w2 @ Vall[0, 0][kk]).abs().max().item()
                    print(f"   without {gname} ({len(gl)} rows): err {e2:.4f}")
print("done")
