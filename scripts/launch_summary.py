"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv): launches, total and
mean time and share per kernel.  python scripts/launch_summary.py launches.csv "header note"."""
import collections
import csv
import sys

path = sys.argv[1]
note = sys.argv[2] if len(sys.argv) > 2 else path
rows = []
with open(path, newline="") as fh:
    lines = [l for l in fh if not l.startswith("==")]
rd = csv.DictReader(lines)
tot = collections.defaultdict(lambda: [0, 0.0])
for r in rd:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    v = float(r["Metric Value"].replace(",", ""))
    unit = r.get("Metric Unit", "ns")
    us = v / 1e3 if unit in ("ns", "nsecond") else v if unit in ("us", "usecond") else v * 1e3
    k = r["Kernel Name"]
    tot[k][0] += 1
    tot[k][1] += us
total = sum(t for _, t in tot.values())
print(f"# {note}")
print("kernel | launches | total us | mean us | share")
for k, (n, t) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
    print(f"{k} | {n} | {t:.1f} | {t / n:.2f} | {100 * t / total:.2f}%")
