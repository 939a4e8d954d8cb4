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
for i in range(8):
    eng.reset(); torch.cuda.synchronize()
    if i == 5: N.profile(True)
    t0 = time.perf_counter(); eng.ingest(pos, col, cam, img); dt = time.perf_counter() - t0
    if i >= 5:
        p = N.profile_read(); print(f"scan {dt*1e3:.2f} ms", {k: round(v[0], 3) for k, v in p.items() if v[0] > 0}); N.profile(True)
PY
VX_LIB_PATH=$PWD/build/pt/libvoxgpr.so timeout 120 python tools/diag_bench.py
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "size_buckets or large_n or config3" 2>&1 | tail -2
timeout 300 python tools/panel_probe.py --voxels 100000 --reps 2
timeout 120 python /tmp/cfg3.py | tail -2
