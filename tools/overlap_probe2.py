"""Where does the e2e leg lose time against the device-resident step?

Times the config-4 step (a) alone, (b) with a concurrent 1.23 GB H2D on a side
stream, (c) with concurrent H2D + 1.22 GB D2H, with the per-stage CUDA-event
profile of each, and the wall time of the host part of ingest_device.

    python tools/overlap_probe2.py
"""
import sys
import time

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2410_17084_b200 as vx  # noqa: E402
from paper_2410_17084_b200 import _native as N  # noqa: E402


def main():
    pos, col, counts, keys, owner, cam_d, img = bench.make_workload(1_000_000, 0)
    cam = vx.Camera(cam_d["fx"], cam_d["fy"], cam_d["cx"], cam_d["cy"], cam_d["width"],
                    cam_d["height"], cam_d["R"], cam_d["t"])
    dev = torch.device("cuda", 0)
    h_xyz = torch.from_numpy(pos).pin_memory()
    h_rgb = torch.from_numpy(col).pin_memory()
    d_xyz, d_rgb, d_img = h_xyz.to(dev), h_rgb.to(dev), torch.from_numpy(img).to(dev)
    x2, r2 = torch.empty_like(d_xyz), torch.empty_like(d_rgb)
    nrec = 9_000_000 * 136
    d_out = torch.empty(nrec, dtype=torch.uint8, device=dev)
    h_out = torch.empty(nrec, dtype=torch.uint8).pin_memory()
    eng = vx.MappingEngine(vx.PipelineConfig(voxel_size=0.5, tau=bench.TAU),
                           voxel_capacity=1_100_000, point_capacity=int(len(pos) * 1.6),
                           gaussian_capacity=9_100_000)
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()

    def comp():
        eng.reset()
        return eng.ingest_device(d_xyz, d_rgb, len(pos), cam, d_img)

    def run(tag, h2d, d2h, k=3):
        comp()
        torch.cuda.synchronize()
        walls, host = [], []
        N.profile(True)
        for _ in range(k):
            if h2d:
                with torch.cuda.stream(s_in):
                    x2.copy_(h_xyz, non_blocking=True)
                    r2.copy_(h_rgb, non_blocking=True)
            if d2h:
                with torch.cuda.stream(s_out):
                    h_out.copy_(d_out, non_blocking=True)
            t0 = time.perf_counter()
            comp()
            t1 = time.perf_counter()
            torch.cuda.synchronize()
            t2 = time.perf_counter()
            host.append((t1 - t0) * 1e3)
            walls.append((t2 - t0) * 1e3)
        prof = N.profile_read()
        N.profile(False)
        st = {k2: round(v[0] / k, 2) for k2, v in prof.items() if v[0] > 0}
        print(f"{tag:10s} wall {sum(walls) / k:7.2f} ms  host-in-ingest {sum(host) / k:7.2f} ms  stages {st}")

    for _ in range(2):
        run("alone", False, False)
        run("+h2d", True, False)
        run("+h2d+d2h", True, True)
        run("+d2h", False, True)


if __name__ == "__main__" and len(sys.argv) == 1:
    main()


def stream_timeline():
    """Host timeline of MappingEngine.ingest_stream(fetch_records=True)."""
    pos, col, counts, keys, owner, cam_d, img = bench.make_workload(1_000_000, 0)
    cam = vx.Camera(cam_d["fx"], cam_d["fy"], cam_d["cx"], cam_d["cy"], cam_d["width"],
                    cam_d["height"], cam_d["R"], cam_d["t"])
    h_xyz = torch.from_numpy(pos).pin_memory()
    h_rgb = torch.from_numpy(col).pin_memory()
    h_img = torch.from_numpy(img).pin_memory()
    solved = int((counts >= bench.TAU).sum())
    eng = vx.MappingEngine(vx.PipelineConfig(voxel_size=0.5, tau=bench.TAU),
                           voxel_capacity=1_050_000, point_capacity=int(len(pos) * 1.6),
                           gaussian_capacity=9 * solved + 1024)
    marks = []
    t0 = [time.perf_counter()]
    orig = eng.ingest_device

    def wrapped(*a, **k):
        s = time.perf_counter()
        r = orig(*a, **k)
        marks.append(("ingest", (s - t0[0]) * 1e3, (time.perf_counter() - t0[0]) * 1e3))
        return r
    eng.ingest_device = wrapped

    def on_rec(rep, host):
        marks.append(("records", (time.perf_counter() - t0[0]) * 1e3, 0))
    for k in (3, 6):
        marks.clear()
        torch.cuda.synchronize()
        t0[0] = time.perf_counter()
        eng.ingest_stream([(h_xyz, h_rgb, cam, h_img)] * k, reset_each=True, fetch_records=True,
                          on_records=on_rec)
        torch.cuda.synchronize()
        tot = (time.perf_counter() - t0[0]) * 1e3
        print(f"stream x{k}: {tot:.1f} ms = {tot / k:.1f} ms/frame")
        for m in marks:
            print("   ", m[0], f"{m[1]:8.1f} {m[2]:8.1f}")


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "stream":
    stream_timeline()
