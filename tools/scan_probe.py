"""Single-scan latency split (configs 1 and 3): wall time of MappingEngine.ingest
(H2D + device work + host syncs) vs the device time of its stages."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_2410_17084_b200 as vx  # noqa: E402
from paper_2410_17084_b200 import _native as N  # noqa: E402
from workloads import scenes  # noqa: E402

cam = vx.Camera(400.0, 400.0, 319.5, 239.5, 640, 480)
img = np.zeros((480, 640, 3))
for name, (pos, col) in (("config1", scenes.config1_scan(seed=0, frame=0)),
                         ("config3", scenes.config3_scan(seed=0, frame=0))):
    eng = vx.MappingEngine(vx.PipelineConfig(voxel_size=0.5))
    walls = []
    for i in range(12):
        eng.reset()
        torch.cuda.synchronize()
        if i == 10:
            N.profile(True)
        l0 = N.launch_count()
        t0 = time.perf_counter()
        eng.ingest(pos, col, cam, img)
        torch.cuda.synchronize()
        walls.append((time.perf_counter() - t0) * 1e3)
        if i == 10:
            prof = N.profile_read()
            N.profile(False)
            launches = N.launch_count() - l0
    st = {k: round(v[0], 3) for k, v in prof.items() if v[0] > 0}
    print(f"{name}: wall {np.median(walls[2:]):.3f} ms, launches {launches}, stages {st}")
