"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv): launches, mean ms and share per kernel.

usage: python tools/launch_summary.py launches.csv "header line"
"""
import collections, csv, sys

rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if l.startswith('"'))]
h = rows[0]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
tot, cnt = collections.Counter(), collections.Counter()
for r in rows[1:]:
    scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}[r[ui]]
    t = float(r[vi].replace(",", "")) * scale
    tot[r[ki][:60]] += t
    cnt[r[ki][:60]] += 1
all_ms = sum(tot.values())
if len(sys.argv) > 2:
    print(sys.argv[2])
print(f"{'kernel':60s} {'launches':>8s} {'mean ms':>10s} {'share':>7s}")
for k in tot:
    print(f"{k:60s} {cnt[k]:8d} {tot[k] / cnt[k]:10.4f} {tot[k] / all_ms:7.3f}")
