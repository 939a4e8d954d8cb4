import sys, time, torch, numpy as np
sys.path.insert(0, '.')
import bench
import paper_2410_17084_b200 as vx
pos, col, counts, keys, owner, cam_d, img = bench.make_workload(1000000, 0)
cam = vx.Camera(cam_d["fx"], cam_d["fy"], cam_d["cx"], cam_d["cy"], cam_d["width"], cam_d["height"], cam_d["R"], cam_d["t"])
h_xyz = torch.from_numpy(pos).pin_memory(); h_rgb = torch.from_numpy(col).pin_memory(); h_img = torch.from_numpy(img).pin_memory()
dev = torch.device('cuda')
d_xyz = torch.empty_like(h_xyz, device=dev); d_rgb = torch.empty_like(h_rgb, device=dev); d_img = h_img.to(dev)
eng = vx.MappingEngine(vx.PipelineConfig(voxel_size=0.5), voxel_capacity=1100000, point_capacity=41000000, gaussian_capacity=9100000)
def T(fn, k=3):
    fn(); torch.cuda.synchronize(); t=time.perf_counter()
    for _ in range(k): fn()
    torch.cuda.synchronize(); return (time.perf_counter()-t)/k*1e3
print('h2d', T(lambda: (d_xyz.copy_(h_xyz, non_blocking=True), d_rgb.copy_(h_rgb, non_blocking=True))))
def comp():
    eng.reset(); eng.ingest_device(d_xyz, d_rgb, len(pos), cam, d_img)
print('compute', T(comp))
s2 = torch.cuda.Stream()
def both():
    with torch.cuda.stream(s2):
        d2 = torch.empty_like(h_xyz, device=dev); d2.copy_(h_xyz, non_blocking=True); d3 = torch.empty_like(h_rgb, device=dev); d3.copy_(h_rgb, non_blocking=True)
    comp()
print('overlap', T(both))
print('stream', T(lambda: eng.ingest_stream([(h_xyz, h_rgb, cam, h_img)]*3, reset_each=True), 1)/3)
