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
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_r2.py -x -q -p no:cacheprovider -k "size_buckets or large_n or config3 or huge or threshold or c05" > gpurun_out/pytest_pi.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_pi.log
timeout 300 python tools/panel_probe.py --voxels 100000 --reps 3 > gpurun_out/panel_probe.log 2>&1; cat gpurun_out/panel_probe.log
for C in 1 8; do VX_PANEL_C=$C VX_LIB_PATH=$PWD/build/pt/libvoxgpr.so timeout 300 python tools/panel_phases.py; done
for C in auto 4 8; do if [ $C = auto ]; then unset VX_PANEL_C; else export VX_PANEL_C=$C; fi; timeout 120 python /tmp/cfg3.py > gpurun_out/cfg3_$C.log 2>&1; echo "C=$C"; tail -1 gpurun_out/cfg3_$C.log; done
