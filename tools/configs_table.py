"""Markdown table of the §8(d) configuration bench lines written by
tools/gpu_round2.sh (cfg_*.json): tokens/s, end-to-end tokens/s, the fused
kernel's and the whole step's fraction of the HBM roofline, the top-k miss
rate and the recall against the exact top-k.
Usage: python tools/configs_table.py DIR > DIR/../configs.md"""
import glob
import json
import os
import sys

d = sys.argv[1]
print("| config | tokens/s | e2e tokens/s | kernel frac of HBM | step frac of HBM | miss rate | recall |")
print("|---|---|---|---|---|---|---|")
for f in sorted(glob.glob(os.path.join(d, "cfg_*.json"))):
    lines = [l for l in open(f).read().strip().splitlines() if l.startswith("{")]
    if not lines:
        print(f"| {os.path.basename(f)[4:-5]} | (no line) | | | | | |")
        continue
    j = json.loads(lines[-1])
    rf = j.get("roofline") or {}
    print("| %s | %.1f | %.1f | %.3f | %.3f | %.2f | %.3f |" % (
        os.path.basename(f)[4:-5], j["value"], j["e2e"]["value"], rf.get("frac", float("nan")),
        rf.get("step_frac_of_hbm", float("nan")), j["miss_transfers"]["miss_rate"], j["fidelity"]["recall_mean"]))
