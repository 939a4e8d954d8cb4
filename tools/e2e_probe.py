import os, sys, time, json
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import bench
import paper_2410_17084_b200 as vx
torch.cuda.set_device(0)
dev = torch.device("cuda", 0)
pos, col, counts, keys, owner, cam_d, img = bench.make_workload(1_000_000, 0)
cam = vx.Camera(cam_d["fx"], cam_d["fy"], cam_d["cx"], cam_d["cy"], cam_d["width"], cam_d["height"], cam_d["R"], cam_d["t"])
cfg = vx.PipelineConfig(voxel_size=0.5, tau=10)
eng = vx.MappingEngine(cfg, voxel_capacity=1_050_000, point_capacity=int(len(pos) * 1.6), gaussian_capacity=9_100_000)
h = [torch.from_numpy(a).pin_memory() for a in (pos, col, img)]
d = [t.to(dev) for t in h]
def t_dev(k):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(k):
        eng.reset(); eng.ingest_device(d[0], d[1], len(pos), cam, d[2])
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / k * 1e3
def t_stream(frames, k):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    eng.ingest_stream([frames] * k, reset_each=True)
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / k * 1e3
def t_copy(k):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(k):
        for a, b in zip(d, h): a.copy_(b, non_blocking=True)
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / k * 1e3
for _ in range(2): t_dev(2); t_stream((h[0], h[1], cam, h[2]), 2)
print(json.dumps({"device_loop_ms": t_dev(5), "stream_pinned_ms": t_stream((h[0], h[1], cam, h[2]), 5),
                  "stream_devframes_ms": t_stream((d[0], d[1], cam, d[2]), 5), "h2d_only_ms": t_copy(5)}))
# compute loop on the current stream with an independent H2D stream running beside it
cs = torch.cuda.Stream()
torch.cuda.synchronize(); t0 = time.perf_counter()
with torch.cuda.stream(cs):
    for _ in range(8):
        for a, b in zip(d, h): a.copy_(b, non_blocking=True)
ms = t_dev(5)
torch.cuda.synchronize()
print(json.dumps({"device_loop_with_concurrent_h2d_ms": ms, "total_s": time.perf_counter() - t0,
                  "current_stream": str(torch.cuda.current_stream()), "side": str(cs)}))
