"""Aggregate an ncu source page (cuda,sass csv) of the DMMA tile kernel by phase line ranges.

usage: ncu_phase_agg.py src.csv voxels
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
nvox = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
cur = None
hdr = None
out = []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split('/')[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) > 7 and r[0] and r[2] == "-":
        try:
            s = int(r[4])
            i = int(r[7] or 0)
        except ValueError:
            continue
        out.append((cur, int(r[0]), s, i))
# function line ranges in vx_gpr.cu, given as "name=lo-hi" arguments after the voxel count
ranges = {}
for a in sys.argv[3:]:
    n, lh = a.split("=")
    lo, hi = lh.split("-")
    ranges[n] = (int(lo), int(hi))
agg = {}
for f, l, s, i in out:
    k = f if f != "vx_gpr.cu" else next((n for n, (a, b) in ranges.items() if a <= l <= b), "other")
    a = agg.setdefault(k, [0, 0])
    a[0] += s
    a[1] += i
ts = sum(v[0] for v in agg.values()) or 1
ti = sum(v[1] for v in agg.values()) or 1
for k, v in sorted(agg.items(), key=lambda x: -x[1][0]):
    print(f"{k:16s} stall-samples {100 * v[0] / ts:5.1f}%  inst {100 * v[1] / ti:5.1f}%  {v[1] / nvox:9.0f} warp-inst/voxel")
