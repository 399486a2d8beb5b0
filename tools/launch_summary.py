"""Per-kernel launch count, total and mean time, and share of the dialsort kernels' time from an
ncu launch list (--metrics gpu__time_duration.sum --csv).  Usage: launch_summary.py launches.csv"""
import csv
import sys
from collections import defaultdict

lines = [l for l in open(sys.argv[1]) if l.startswith('"')]  # skip ==PROF== lines
rows = [r for r in csv.DictReader(lines) if r.get("Metric Name") == "gpu__time_duration.sum"]
agg = defaultdict(lambda: [0, 0.0])
for r in rows:
    name = r["Kernel Name"].split("(")[0].replace("void ", "")
    scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}[r["Metric Unit"]]
    agg[name][0] += 1
    agg[name][1] += float(r["Metric Value"].replace(",", "")) * scale
ours = {k: v for k, v in agg.items() if k.startswith("ds::") or k.startswith("k_")}
tot = sum(v[1] for v in ours.values()) or 1.0
print(f"{'kernel':40s} {'launches':>8s} {'total us':>10s} {'mean us':>9s} {'share':>6s}")
for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    share = f"{t / tot:6.3f}" if k in ours else "     -"
    print(f"{k[:40]:40s} {c:8d} {t:10.2f} {t / c:9.3f} {share}")
print("(share: of the DialSort kernels' summed time; ncu times are serialised and cold-cache)")
