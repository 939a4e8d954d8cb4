"""Large-n panel kernel probe: the config-4 tail map (Livox n-histogram) with
`--voxels` voxels ingested `--reps` times; prints the gpr_n_large stage time
and its FP64 rate.  Used under ncu (one launch) and for A/B timing."""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from workloads import scenes  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--voxels", type=int, default=100_000)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    import torch
    import paper_2410_17084_b200 as vx
    from paper_2410_17084_b200 import _native as N
    pos, col, counts, keys, owner = scenes.planar_map(a.voxels, voxel_size=0.5, seed=5,
                                                      bins=scenes.TAIL_BINS, probs=scenes.TAIL_PROBS)
    cam = vx.Camera(500.0, 500.0, 319.5, 239.5, 640, 480)
    img = torch.zeros((480, 640, 3), dtype=torch.float64, device="cuda")
    dx, dc = torch.from_numpy(pos).cuda(), torch.from_numpy(col).cuda()
    eng = vx.MappingEngine(vx.PipelineConfig(voxel_size=0.5))
    sol = counts[counts >= 10]
    big = sol[sol > 160]
    flops = float(bench.gpr_flops(big).sum())
    for r in range(a.reps):
        eng.reset()
        N.profile(True)
        eng.ingest_device(dx, dc, len(pos), cam, img)
        torch.cuda.synchronize()
        prof = N.profile_read()
        N.profile(False)
        ms = prof["gpr_n_large"][0]
        print(f"rep {r}: gpr_n_large {ms:.2f} ms, {len(big)} voxels, "
              f"{flops / ms / 1e9:.2f} TF/s", flush=True)


if __name__ == "__main__":
    main()
