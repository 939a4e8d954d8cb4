import sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_2410_17084_b200 as vx
cam = vx.Camera(100.0, 100.0, 79.5, 59.5, 160, 120)
img = np.random.default_rng(0).uniform(0, 1, (120, 160, 3))
eng = vx.MappingEngine(vx.PipelineConfig(voxel_size=0.5))
r = eng.ingest(np.empty((0, 3)), np.empty((0, 3)), cam, img); print("empty", r.voxels_touched, r.primitives_added)
rng = np.random.default_rng(1)
pos = np.concatenate([rng.uniform(0.01, 0.49, (3000, 3)), rng.uniform(-10, 10, (2000, 3))])
col = rng.uniform(0, 1, pos.shape)
r = eng.ingest(pos, col, cam, img); print("big voxel", r.voxels_touched, r.voxels_solved, r.primitives_added)
r = eng.ingest(pos[:5], col[:5], cam, img); print("tiny", r.voxels_touched, r.voxels_solved, r.primitives_added)
try:
    eng.ingest(pos, col, cam, img[:100])
except IndexError as e:
    print("small image ->", type(e).__name__)
r = eng.ingest(pos, col, cam, np.pad(img, ((0, 5), (0, 7), (0, 1)))); print("large image ok", r.voxels_solved)
print("gaussians", eng.num_gaussians)
