cat > /tmp/cfg3.py <<'PY'
import sys, time, numpy as np, torch
sys.path.insert(0, ".")
import paper_2410_17084_b200 as vx
from paper_2410_17084_b200 import _native as N
from workloads import scenes
pos, col = scenes.config3_scan(seed=0, frame=0)
cam = vx.Camera(400.0, 400.0, 319.5, 239.5, 640, 480)
img = np.zeros((480, 640, 3))
eng = vx.MappingEngine(vx.PipelineConfig(voxel_size=0.5))
walls = []
for i in range(10):
    eng.reset(); torch.cuda.synchronize()
    if i == 8: N.profile(True)
    t0 = time.perf_counter(); eng.ingest(pos, col, cam, img); torch.cuda.synchronize(); walls.append(time.perf_counter() - t0)
    if i == 8:
        p = N.profile_read(); N.profile(False)
c = np.bincount(np.unique(np.floor(pos / 0.5).astype(np.int64), axis=0, return_counts=True)[1] > 160)
print(f"wall {np.median(walls[3:])*1e3:.3f} ms, n_large {p['gpr_n_large'][0]:.3f} ms, voxels n>160: {c}")
PY
for C in auto 8 16; do if [ $C = auto ]; then unset VX_PANEL_C; else export VX_PANEL_C=$C; fi; echo "C=$C"; timeout 120 python /tmp/cfg3.py; done
