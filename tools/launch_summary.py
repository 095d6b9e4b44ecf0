"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV):
per-kernel launch count, mean and total time, and the share of the decode
step (LRQK kernels launched after the last prefill launch)."""
import collections, csv, sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
launches = [(r[ki].split("(")[0].replace("void ", ""), float(r[vi].replace(",", "")) * scale[r[ui]]) for r in rows[1:]]
agg = collections.defaultdict(list)
for k, v in launches:
    agg[k].append(v)
print(f"{'kernel':60s} {'n':>5s} {'mean_us':>10s} {'total_us':>12s}")
for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
    print(f"{k[:60]:60s} {len(v):5d} {sum(v)/len(v):10.2f} {sum(v):12.1f}")
last_pf = max((i for i, (k, _) in enumerate(launches) if "pf_" in k or "seed" in k), default=-1)
if len(sys.argv) > 2:  # steady state: skip the first N decode steps (ends of steps = advance_kernel)
    adv = [i for i, (k, _) in enumerate(launches) if "advance_kernel" in k and i > last_pf]
    if len(adv) > int(sys.argv[2]):
        last_pf = adv[int(sys.argv[2]) - 1]
dec = [(k, v) for k, v in launches[last_pf + 1:] if k.startswith("lrqk::")]
tot = sum(v for _, v in dec) or 1.0
dagg = collections.defaultdict(float)
for k, v in dec:
    dagg[k] += v
print(f"\ndecode steps (serialised, cold-cache ncu replay): {len(dec)} launches, {tot:.1f} us")
for k, v in sorted(dagg.items(), key=lambda x: -x[1]):
    print(f"  {k[:58]:58s} {v:10.1f} us  share {v/tot:6.3f}")
