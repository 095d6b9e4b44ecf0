"""Per-source-line warp-stall breakdown of one kernel in an ncu report:
lines sorted by samples, with the top stall reasons of each."""
import csv, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur, hdr, res = None, None, []
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if len(r) > 3 and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[2] == "-":
        try:
            smp = float(r[hdr.index("Warp Stall Sampling (All Samples)")])
        except ValueError:
            continue
        if smp <= 0:
            continue
        stalls = {h[6:]: float(v) for h, v in zip(hdr, r) if h.startswith("stall_") and "Not Issued" not in h and v not in ("", "0")}
        res.append((smp, cur, r[0], r[1][:90], stalls))
tot = sum(x[0] for x in res) or 1
agg = {}
for x in res:
    for k, v in x[4].items():
        agg[k] = agg.get(k, 0) + v
print("samples", tot, " overall:", ", ".join(f"{k} {v/tot:.2f}" for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:8]))
for smp, f, ln, src, st in sorted(res, key=lambda x: -x[0])[:top]:
    s = ", ".join(f"{k} {v/smp:.2f}" for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:3])
    print(f"{smp/tot:6.3f} {f}:{ln:>4s} {src:90s} | {s}")
