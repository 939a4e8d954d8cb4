"""Aggregate an ncu launch list (gpu__time_duration.sum csv) by kernel name."""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if l.startswith('"'))]
hdr = rows[0]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
tot = defaultdict(float)
cnt = defaultdict(int)
for r in rows[1:]:
    name = r[ki].split("(")[0]
    tot[name] += float(r[vi]) / 1e3
    cnt[name] += 1
all_us = sum(tot.values())
print(f"{'kernel':48s} {'launches':>8s} {'total us':>12s} {'share':>7s}")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"{k:48s} {cnt[k]:8d} {v:12.1f} {100 * v / all_us:6.1f}%")
print(f"{'TOTAL':48s} {sum(cnt.values()):8d} {all_us:12.1f}")
