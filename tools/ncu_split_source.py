"""Split a multi-kernel ncu source-page csv into one csv per profiled launch.

usage: ncu_split_source.py all.csv out_prefix   ->  out_prefix<i>.csv (i = launch index)
"""
import sys

lines = open(sys.argv[1]).read().splitlines(keepends=True)
k = -1
cur_fn = None
seen = set()
pending = None
out = {}
for ln in lines:
    if ln.startswith('"File Path"'):
        pending = ln
        continue
    if ln.startswith('"Function Name"'):
        fn = ln
        fpath = pending
        if fn != cur_fn or fpath in seen:
            k += 1
            cur_fn = fn
            seen = set()
        seen.add(fpath)
        out.setdefault(k, []).extend([fpath, ln])
        continue
    if k >= 0:
        out[k].append(ln)
for i, body in out.items():
    open(f"{sys.argv[2]}{i}.csv", "w").writelines(body)
    print(i, body[1].strip()[:110])
