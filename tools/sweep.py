"""Config 5: GPR sample-grid and kernel sweep for roofline characterisation.

    python tools/sweep.py [--voxels 200000] [--out profiles/r1_sweep.json]

For (n_s, n_r) in {(2,2),(3,2),(4,2),(3,3),(4,3),(4,4)} (grid 4..16 per
axis, n* = 16..256) and kernel in {se (reference), matern32, matern52
(extensions)}: one ingest of a synthetic planar map (points-per-voxel
histogram of the 32-beam scan) into an empty map on cuda:0, timed with CUDA
events (median of 3 after one warm-up).  Reports the GPR stage time (sum of
the size-bucket kernels, library stage timers), the algorithmic FP64 flops of
the solves at that n* (SURVEY §8(d) G6 formula with n* in place of 81) and
the achieved fraction of the FP64 peak measured in the same run.
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def flops(n, m):
    n = np.asarray(n, dtype=np.float64)
    return n ** 3 / 3 + n * n * m + n * n + 4 * n * m + 6 * (n * (n + 1) / 2 + n * m)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--voxels", type=int, default=200_000)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    import torch
    import paper_2410_17084_b200 as vx
    from paper_2410_17084_b200 import _native as N

    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    pos, col, counts, keys, owner, cam_d, img = bench.make_workload(args.voxels, 0)
    cam = vx.Camera(cam_d["fx"], cam_d["fy"], cam_d["cx"], cam_d["cy"], cam_d["width"],
                    cam_d["height"], cam_d["R"], cam_d["t"])
    d_xyz = torch.from_numpy(pos).to(dev)
    d_rgb = torch.from_numpy(col).to(dev)
    d_img = torch.from_numpy(img).to(dev)
    sol = counts[counts >= bench.TAU]
    peak = N.fp64_peak_tflops()
    rows = []
    for ns, nr in ((2, 2), (3, 2), (4, 2), (3, 3), (4, 3), (4, 4)):
        m = (ns * nr) ** 2
        for kern in ("se", "matern32", "matern52"):
            cfg = vx.PipelineConfig(voxel_size=0.5, n_s=ns, n_r=nr, kernel=kern)
            eng = vx.MappingEngine(cfg)
            res = []
            for it in range(4):
                eng.reset()
                torch.cuda.synchronize()
                N.profile(True)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                rep = eng.ingest_device(d_xyz, d_rgb, len(pos), cam, d_img)
                e1.record()
                torch.cuda.synchronize()
                prof = N.profile_read()
                N.profile(False)
                if it:
                    gpr_ms = sum(v[0] for k, v in prof.items() if k.startswith("gpr_"))
                    res.append((e0.elapsed_time(e1), gpr_ms, prof))
            step_ms = float(np.median([r[0] for r in res]))
            gpr_ms = float(np.median([r[1] for r in res]))
            f = float(flops(sol, m).sum())
            row = {"n_s": ns, "n_r": nr, "grid_per_axis": ns * nr, "n_star": m, "kernel": kern,
                   "voxels_solved": int(rep.voxels_solved), "step_ms": step_ms, "gpr_ms": gpr_ms,
                   "voxels_per_s": rep.voxels_solved / (step_ms / 1e3),
                   "gpr_tflops": f / (gpr_ms / 1e3) / 1e12,
                   "frac_fp64_peak": f / (gpr_ms / 1e3) / 1e12 / peak,
                   "stage_ms": {k: round(v[0], 3) for k, v in res[-1][2].items() if v[0] > 0}}
            rows.append(row)
            print(json.dumps(row), flush=True)
    out = {"workload": f"config5: {args.voxels}-voxel planar map, one ingest per point",
           "fp64_peak_tflops_measured": peak, "rows": rows}
    if args.out:
        json.dump(out, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
