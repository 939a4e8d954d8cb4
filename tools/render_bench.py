"""Renderer measurement: device render time on the
mapping path's own Gaussian maps, the host-API time, and the CPU oracle.

    python tools/render_bench.py [--out profiles/r1_render.json]

* config-1 map: one 60k-ray 32-beam scan ingested with its camera and image
  (~13.6k Gaussians), rendered at 640x480 from the scan camera.
* config-4 map: the bench's 1M-voxel planar map (9M Gaussians), rendered at
  640x480 from the bench's downward camera.
Device times: CUDA events around `render_device` (records already in HBM,
images left in HBM), median of 20 after warm-up.  Host-API time: `render()`
on the engine's device records including the D2H of the three images.
CPU: the oracle restatement (tests' checker) on the config-1 map, one run,
one core.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from workloads import scenes  # noqa: E402


def time_device(fn, reps=20):
    import torch
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--no-oracle", action="store_true")
    args = ap.parse_args()
    import torch
    import paper_2410_17084_b200 as vx
    from paper_2410_17084_b200 import renderer as R
    torch.cuda.set_device(0)
    res = {}
    # config-1
    sc = scenes.OutdoorScene.make(0)
    pin = scenes.camera_for(0, 640, 480, 400.0)
    img = scenes.render_image(sc, pin)
    cam = vx.Camera(pin.fx, pin.fy, pin.cx, pin.cy, pin.width, pin.height, pin.R, pin.t)
    pos, col = scenes.config1_scan(seed=0, frame=0)
    eng = vx.MappingEngine(vx.PipelineConfig(voxel_size=0.5))
    eng.ingest(pos, col, cam, img)
    g = eng.gaussians_device()
    ms = time_device(lambda: R.render_device(g, cam))
    t0 = time.perf_counter()
    for _ in range(10):
        buf = R.render(g, cam)
    host_ms = (time.perf_counter() - t0) / 10 * 1e3
    row = {"workload": "config1 map: one 32-beam scan's Gaussians, 640x480 from the scan camera",
           "gaussians": eng.num_gaussians, "device_ms": ms, "host_api_ms": host_ms,
           "covered_pixels": int((buf.silhouette > 0).sum())}
    if not args.no_oracle:
        from oracle import voxsplat_oracle as O
        h = {k: v.cpu().numpy() for k, v in g.items()}
        ocam = dict(fx=cam.fx, fy=cam.fy, cx=cam.cx, cy=cam.cy, width=640, height=480,
                    R=cam.rotation, t=cam.translation)
        t0 = time.perf_counter()
        oc, od, osil, _ = O.render_splats(h["position"], h["scale"], h["rotation"], h["opacity"],
                                          h["color"], ocam)
        row["cpu_oracle_ms"] = (time.perf_counter() - t0) * 1e3
        row["cpu_cores"] = 1
        row["max_abs_diff_vs_oracle"] = float(max(np.abs(buf.color - oc).max(),
                                                  np.abs(buf.silhouette - osil).max()))
    res["config1"] = row
    print(json.dumps(row), flush=True)
    # config-4
    pos, col, counts, keys, owner, cam_d, img4 = bench.make_workload(1_000_000, 0)
    cam4 = vx.Camera(cam_d["fx"], cam_d["fy"], cam_d["cx"], cam_d["cy"], cam_d["width"],
                     cam_d["height"], cam_d["R"], cam_d["t"])
    eng = vx.MappingEngine(vx.PipelineConfig(voxel_size=0.5, tau=bench.TAU),
                           voxel_capacity=1_050_000, point_capacity=int(len(pos) * 1.6),
                           gaussian_capacity=9_100_000)
    eng.ingest_device(torch.from_numpy(pos).cuda(), torch.from_numpy(col).cuda(), len(pos), cam4,
                      torch.from_numpy(img4).cuda())
    g = eng.gaussians_device()
    ms = time_device(lambda: R.render_device(g, cam4), reps=10)
    buf = R.render(g, cam4)
    row = {"workload": "config4 map: 1M voxels / 9M Gaussians, 640x480 from the bench camera",
           "gaussians": eng.num_gaussians, "device_ms": ms,
           "covered_pixels": int((buf.silhouette > 0).sum()),
           "gaussians_per_s": eng.num_gaussians / (ms / 1e3)}
    res["config4"] = row
    print(json.dumps(row), flush=True)
    if args.out:
        json.dump(res, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
