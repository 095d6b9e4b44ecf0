"""Summarise an ncu report's per-source-line stall samples for one kernel."""
import csv, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur = None; hdr = None; res = []
for r in rows:
    if len(r) >= 2 and r[0] == "File Path": cur = r[1].split("/")[-1]; continue
    if len(r) >= 2 and r[0] == "Line No": hdr = r; continue
    if hdr and len(r) > 7 and r[2] == "-":
        try: res.append((float(r[4]), float(r[7]), cur, r[0], r[1][:100]))
        except ValueError: pass
tot = sum(x[0] for x in res) or 1
print("samples", tot)
for x in sorted(res, reverse=True)[:top]:
    print(f"{x[0]/tot:6.3f} inst={x[1]:>10.0f} {x[2]}:{x[3]:>4s} {x[4]}")
