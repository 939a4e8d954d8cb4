"""Summarise an ncu source page (cuda,sass csv) by source line: stall samples and instructions."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
out = []
cur_file = None
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) > 7 and r[0] and r[2] == "-":
        try:
            samples = int(r[4]); inst = int(r[7] or 0)
        except (ValueError, IndexError):
            continue
        out.append((samples, inst, f"{cur_file}:{r[0]}", r[1][:90]))
tot = sum(o[0] for o in out) or 1
toti = sum(o[1] for o in out) or 1
out.sort(reverse=True)
print(f"total samples {tot}, warp instructions {toti}")
for s, i, loc, src in out[:int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    print(f"{100*s/tot:5.1f}% {100*i/toti:5.1f}%i  {loc:22s} {src}")
