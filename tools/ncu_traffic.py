"""DRAM traffic per solved voxel of each GPR kernel, from one `ncu --set full`
capture of `bench.py --voxels V --steps 1 --warmup 1` (first densify only).

    python tools/ncu_traffic.py <report.ncu-rep> <V> > profiles/<round>_traffic.json

The bucket voxel counts are recomputed from the same seeded workload, so the
bytes/voxel figure can be scaled to any launch of the same kernel (bench.py
reports `roofline.traffic` that way).
"""
import csv
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import bench  # noqa: E402

rep, V = sys.argv[1], int(sys.argv[2])
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[0]
col = {h: i for i, h in enumerate(hdr)}
_, _, counts, *_ = bench.make_workload(V, 0)
sol = counts[counts >= bench.TAU]
buckets = [("gpr_tile_kernel<20,", (128, 160), "gpr_n160"),
           ("gpr_tile_kernel<12,", (64, 96), "gpr_n96"),
           ("gpr_wdmma_kernel<32", (24, 32), "gpr_n32"),
           ("gpr_panel_kernel", (160, 10 ** 9), "gpr_n_large"),
           ("gpr_tile_kernel<16, 1, 6", (96, 128), "gpr_n128"),
           ("gpr_tile_kernel<8,", (32, 64), "gpr_n64"),
           ("gpr_wdmma_kernel<24", (16, 24), "gpr_n24"),
           ("gpr_wdmma_kernel<16", (0, 16), "gpr_n16")]
res = {}
for r in rows[2:]:
    name = r[col["Kernel Name"]]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    tot = sum(float(r[col[m]]) * scale.get(rows[1][col[m]], 1)     # per-column units
              for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
    for key, (lo, hi), label in buckets:
        if key in name and label not in res:
            n = int(((sol > lo) & (sol <= hi)).sum())
            res[label] = {"dram_bytes": tot, "voxels": n, "bytes_per_voxel": tot / max(n, 1),
                          "kernel": name}
            break
print(json.dumps(res, indent=1))
