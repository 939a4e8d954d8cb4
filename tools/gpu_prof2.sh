set -x
python -m paper_2410_17084_b200.build
timeout 600 python -m pytest tests/test_gpu_r2.py -q -p no:cacheprovider -k stream > gpurun_out/pytest_stream.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_stream.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gpr_panel_kernel -s 1 -c 1 -o gpurun_out/panel_v2 python tools/panel_probe.py --voxels 100000 --reps 2 > gpurun_out/ncu_panel2.log 2>&1; echo "ncu rc=$?"
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
for C in 2 4 8; do VX_PANEL_C=$C timeout 120 python /tmp/cfg3.py > gpurun_out/cfg3_$C.log 2>&1; echo "C=$C"; cat gpurun_out/cfg3_$C.log; done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gpr_panel_kernel -s 3 -c 1 -o gpurun_out/panel_cfg3 python /tmp/cfg3.py > gpurun_out/ncu_cfg3.log 2>&1; echo "ncu3 rc=$?"
