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
