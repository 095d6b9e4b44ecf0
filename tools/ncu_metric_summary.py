"""Summarise an `ncu --metrics ... --csv --log-file` launch list: per kernel,
launches, share of the summed duration, mean duration and per-launch means
of the other metrics (PCIe / DRAM bytes, and the GB/s they imply over the
kernel's own time).  Usage: python tools/ncu_metric_summary.py log.csv [top]"""
import collections
import csv
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 15
rows = list(csv.reader(open(path)))
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
agg = collections.defaultdict(lambda: collections.defaultdict(float))
ids = collections.defaultdict(set)
for d in data:
    k = d["Kernel Name"].split("(")[0][:60]
    v = float(d["Metric Value"].replace(",", "") or 0)
    agg[k][d["Metric Name"]] += v
    ids[k].add(d["ID"])
tot = sum(v.get("gpu__time_duration.sum", 0) for v in agg.values()) or 1
print(f"{'kernel':60s} {'n':>5s} {'share':>6s} {'mean_us':>9s}  per-launch means")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1].get("gpu__time_duration.sum", 0))[:top]:
    n = len(ids[k])
    t = v.get("gpu__time_duration.sum", 0)
    extra = []
    for m in sorted(v):
        if m == "gpu__time_duration.sum":
            continue
        extra.append(f"{m}={v[m] / n / 1e6:.2f}MB ({v[m] / max(t, 1):.1f} GB/s)")
    print(f"{k:60s} {n:5d} {t / tot:6.3f} {t / n / 1e3:9.2f}  " + "  ".join(extra))
