"""Per-call wall times of the drop-in VoxelMap path vs MappingEngine on the
config-2 trajectory (where do the drop-in's milliseconds go?)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_2410_17084_b200 as vx  # noqa: E402
from workloads import scenes  # noqa: E402

cfg = vx.PipelineConfig(voxel_size=0.5, eta=2e-5, iterations=0)
frames = [scenes.config1_scan(seed=0, frame=f, rays=60000) for f in range(12)]
vmap = vx.VoxelMap.from_config(cfg)
eng = vx.MappingEngine(cfg)
for i, (pos, col) in enumerate(frames):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    up = vmap.store_frame(vx.PointCloud(pos, col, np.zeros(len(pos))))
    t1 = time.perf_counter()
    cand = [k for k in up if vmap.cells[k].state == vx.VoxelState.READY]
    t2 = time.perf_counter()
    preds = vx.densify_frame(up, vmap, cfg)
    t3 = time.perf_counter()
    cells = [vmap.cells[p.key] for p in preds]
    t4 = time.perf_counter()
    torch.cuda.synchronize()
    t5 = time.perf_counter()
    e = eng.ingest(pos, col)
    t6 = time.perf_counter()
    print(f"frame {i}: store {1e3*(t1-t0):6.1f}  state-scan {1e3*(t2-t1):6.1f} ({len(up)} keys)  "
          f"densify {1e3*(t3-t2):6.1f} ({len(preds)} solved)  cells {1e3*(t4-t3):6.1f}  engine {1e3*(t6-t5):6.1f}")

# expansion loop of pipeline.py:154-171 on the last frame's first solves
import gc
gc.disable()
cam = vx.Camera(100.0, 100.0, 79.5, 59.5, 160, 120)
img = np.zeros((120, 160, 3))
gm = vx.GaussianMap()
pos, col = scenes.config1_scan(seed=0, frame=12, rays=60000)
up = vmap.store_frame(vx.PointCloud(pos, col, np.zeros(len(pos))))
t0 = time.perf_counter()
first = {k for k in up if vmap.cells[k].state == vx.VoxelState.READY}
t1 = time.perf_counter()
preds = vx.densify_frame(up, vmap, cfg)
t2 = time.perf_counter()
newly = [p.key for p in preds if p.key in first]
n = 0
for key in newly:
    cell = vmap.cells[key]
    prims = vx.init_gaussians_for_voxel(cell.last_prediction, cam, img, cfg)
    gm.extend(prims)
    n += len(prims)
t3 = time.perf_counter()
_ = gm.positions
t4 = time.perf_counter()
print(f"gc off: state-scan {1e3*(t1-t0):.1f} ({len(up)} keys)  densify {1e3*(t2-t1):.1f} ({len(preds)})  "
      f"expansion {1e3*(t3-t2):.1f} ({len(newly)} voxels, {n} prims)  settle {1e3*(t4-t3):.1f}")
