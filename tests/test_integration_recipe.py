"""INTEGRATION.md §1 executed: the reference's own `MappingPipeline.ingest_frame`
(pipeline.py:139-187, unmodified, from the pip-installed reference in
baseline/_ref) with `voxsplat.{errors,config,camera,voxel_map,gpr,splat_init,
renderer}` substituted by this package before the pipeline is imported.

Ten frames of the config-2 trajectory (eta = 2e-5: re-fits from raw ∪ pseudo
points) must produce the same reports, the same transition log and the same
Gaussian map, record for record, as `MappingEngine` (the fused device path).
Runs in a subprocess so the substitution does not leak into other tests;
skipped when baseline/_ref (the reference install) is absent.
"""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")

pytestmark = pytest.mark.gpu

SCRIPT = r'''
import json, sys, time
import numpy as np
sys.path.insert(0, ROOT)
sys.path.insert(0, REF)
import paper_2410_17084_b200 as vx
from paper_2410_17084_b200 import camera, config, errors, gpr, renderer, splat_init, voxel_map
for name, mod in (("voxsplat.errors", errors), ("voxsplat.config", config),
                  ("voxsplat.camera", camera), ("voxsplat.voxel_map", voxel_map),
                  ("voxsplat.gpr", gpr), ("voxsplat.splat_init", splat_init),
                  ("voxsplat.renderer", renderer)):
    sys.modules[name] = mod
import voxsplat.pipeline as P
assert P.densify_frame is gpr.densify_frame and P.VoxelMap is voxel_map.VoxelMap
from workloads import scenes

cfg = vx.PipelineConfig(voxel_size=0.5, eta=2e-5, iterations=0)
sc = scenes.OutdoorScene.make(0)
frames = []
for f in range(NFRAMES):
    pos, col = scenes.config1_scan(seed=0, frame=f, rays=RAYS)
    pin = scenes.camera_for(f, 160, 120, 100.0)
    cam = vx.Camera(pin.fx, pin.fy, pin.cx, pin.cy, pin.width, pin.height, pin.R, pin.t)
    frames.append((pos, col, cam, scenes.render_image(sc, pin)))
pipe = P.MappingPipeline(cfg)
eng = vx.MappingEngine(cfg, record_log=True)
reps, ereps, dt, edt = [], [], [], []
for i, (pos, col, cam, img) in enumerate(frames):
    fs = P.FrameSample(float(i), vx.PointCloud(pos, col, np.zeros(len(pos))), img, cam)
    t0 = time.perf_counter()
    r = pipe.ingest_frame(fs)
    dt.append(time.perf_counter() - t0)
    reps.append([r.voxels_touched, r.voxels_solved, r.newly_active, r.newly_converged,
                 r.primitives_added, len(r.errors)])
    t0 = time.perf_counter()
    e = eng.ingest(pos, col, cam, img)
    edt.append(time.perf_counter() - t0)
    ereps.append([e.voxels_touched, e.voxels_solved, e.newly_active, e.newly_converged,
                  e.primitives_added, 0])
g = pipe.gmap
eg = eng.gaussian_map()
same = {k: bool(np.array_equal(getattr(g, k), getattr(eg, k))) for k in
        ("positions", "scales", "rotations", "opacities", "colors", "source_keys")}
tr = [(t.frame, tuple(t.key), int(t.old), int(t.new)) for t in pipe.vmap.transitions]
etr = [(t.frame, tuple(t.key), int(t.old), int(t.new)) for t in eng.vmap.transitions]
print(json.dumps({"reps": reps, "ereps": ereps, "same": same, "n": len(g),
                  "transitions_equal": tr == etr, "n_transitions": len(tr),
                  "audits": pipe.vmap.audit_transitions() + pipe.vmap.audit_converged_resolves(),
                  "ms_per_frame": [1e3 * x for x in dt],
                  "engine_ms_per_frame": [1e3 * x for x in edt]}))
'''


def run_recipe(nframes=10, rays=20000):
    code = (f"ROOT = {ROOT!r}\nREF = {REF!r}\nNFRAMES = {nframes}\nRAYS = {rays}\n" + SCRIPT)
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                         timeout=900, cwd=ROOT)
    if out.returncode != 0:
        raise RuntimeError(out.stderr[-4000:])
    return json.loads(out.stdout.strip().splitlines()[-1])


def test_reference_pipeline_on_substituted_modules_equals_engine():
    if not os.path.isdir(os.path.join(REF, "voxsplat")):
        pytest.skip("baseline/_ref (pip-installed reference) is absent")
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    r = run_recipe()
    assert r["reps"] == r["ereps"]
    assert all(r["same"].values()), r["same"]
    assert r["n"] > 0 and r["transitions_equal"] and r["n_transitions"] > 0
    assert r["audits"] == []
    refits = sum(x[1] - x[2] for x in r["reps"])
    assert refits > 0
