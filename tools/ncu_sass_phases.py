"""Attribute ncu SASS-level samples / instructions to phases of a kernel by
source-line ranges of its main file, following inlined helpers by address
order (a SASS instruction of an inlined helper belongs to the phase of the
closest preceding main-file instruction).

usage: ncu_sass_phases.py source.csv main.cu name:lo-hi [name:lo-hi ...]
(source.csv = `ncu -i X.ncu-rep --page source --csv --print-source cuda,sass`)
"""
import csv
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    main_file = sys.argv[2]
    ranges = []
    for a in sys.argv[3:]:
        n, r = a.split(":")
        lo, hi = map(int, r.split("-"))
        ranges.append((n, lo, hi))
    cur_file, cur_line = None, None
    sass = []   # (addr, samples, inst, file, line)
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            cur_file = r[1].split("/")[-1]
            continue
        if r[0] in ("Function Name", "Line No"):
            continue
        if len(r) > 7 and r[0] and r[2] == "-":
            try:
                cur_line = int(r[0])
            except ValueError:
                cur_line = None
            continue
        if len(r) > 7 and r[0] == "" and r[2].startswith("0x"):
            try:
                s, i = int(r[6]), int(r[7])
            except ValueError:
                continue
            sass.append((int(r[2], 16), s, i, cur_file, cur_line))
    sass.sort()
    acc = {n: [0, 0] for n, _, _ in ranges}
    acc["other"] = [0, 0]
    phase = "other"
    for addr, s, i, f, ln in sass:
        if f == main_file and ln is not None:
            phase = next((n for n, lo, hi in ranges if lo <= ln <= hi), "other")
        acc[phase][0] += s
        acc[phase][1] += i
    ts = sum(v[0] for v in acc.values()) or 1
    ti = sum(v[1] for v in acc.values()) or 1
    print(f"total samples {ts}, warp instructions {ti}")
    for n, (s, i) in acc.items():
        print(f"{n:12s} samples {100 * s / ts:5.1f}%  instructions {100 * i / ti:5.1f}%  ({i})")


if __name__ == "__main__":
    main()
