"""Sum ncu source-page stall samples / instructions of one file over line ranges.

usage: ncu_phases.py source.csv file.cu name:lo-hi [name:lo-hi ...]
(source.csv = `ncu -i X.ncu-rep --page source --csv --print-source cuda,sass`)
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
target = sys.argv[2]
ranges = []
for a in sys.argv[3:]:
    n, r = a.split(":")
    lo, hi = map(int, r.split("-"))
    ranges.append((n, lo, hi))
cur = None
hdr = None
acc = {n: [0, 0] for n, _, _ in ranges}
other = [0, 0]
tot = [0, 0]
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) > 7 and r[0] and r[2] == "-":
        try:
            s = int(r[4])
            i = int(r[7] or 0)
            ln = int(r[0])
        except (ValueError, IndexError):
            continue
        tot[0] += s
        tot[1] += i
        hit = False
        if cur == target:
            for n, lo, hi in ranges:
                if lo <= ln <= hi:
                    acc[n][0] += s
                    acc[n][1] += i
                    hit = True
                    break
        if not hit:
            other[0] += s
            other[1] += i
for n, _, _ in ranges:
    print(f"{n:12s} stalls {100 * acc[n][0] / tot[0]:5.1f}%  inst {100 * acc[n][1] / tot[1]:5.1f}%")
print(f"{'other':12s} stalls {100 * other[0] / tot[0]:5.1f}%  inst {100 * other[1] / tot[1]:5.1f}%")
