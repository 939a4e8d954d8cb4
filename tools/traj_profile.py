"""Stage breakdown of the config-2 trajectory (bench --traj-scans) on one GPU."""
import sys, os, json
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch, numpy as np
import bench
import paper_2410_17084_b200 as vx
from paper_2410_17084_b200 import _native as N
from workloads import scenes
sc = scenes.OutdoorScene.make(0)
frames = []
for f in range(20):
    pos, col = scenes.config1_scan(seed=0, frame=f)
    pin = scenes.camera_for(f, 160, 120, 100.0)
    img = scenes.render_image(sc, pin)
    cam = vx.Camera(pin.fx, pin.fy, pin.cx, pin.cy, pin.width, pin.height, pin.R, pin.t)
    frames.append((torch.from_numpy(pos).pin_memory(), torch.from_numpy(col).pin_memory(), cam,
                   torch.from_numpy(img).pin_memory()))
eng = vx.MappingEngine(vx.PipelineConfig(voxel_size=0.5, eta=2e-5))
eng.ingest_stream(frames); eng.reset(); torch.cuda.synchronize()
N.profile(True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); reps = eng.ingest_stream(frames); e1.record(); torch.cuda.synchronize()
prof = N.profile_read(); N.profile(False)
print("ms/scan", e0.elapsed_time(e1) / len(frames))
print(json.dumps({k: round(v[0] / len(frames), 4) for k, v in prof.items()}))
print("max_train", max(r.voxels_solved for r in reps))
v = eng.vmap.device_view()
cnt = N.view_tensor(v.raw_count, (int(v.num_voxels),), np.int32).cpu().numpy()
print("raw count percentiles", np.percentile(cnt[cnt >= 10], [50, 90, 99, 100]))
