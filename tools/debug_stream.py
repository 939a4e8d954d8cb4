import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_2410_17084_b200 as vx
from paper_2410_17084_b200 import formats
sdir = os.path.join(ROOT, "tests", "golden", "stream")
ref = [formats.read_ply_device(os.path.join(sdir, f"{i:06d}.ply")) for i in range(3)]
frames = list(vx.stream.stream_frames(sdir))
eng = vx.MappingEngine(vx.PipelineConfig(voxel_size=0.2))
orig = eng.ingest_device
k = [0]
def spy(dx, dc, n, cam, di):
    torch.cuda.synchronize()
    i = k[0]; k[0] += 1
    rx, rc, rn = ref[i]
    print("frame", i, "n", n, rn, "xyz equal", bool(torch.equal(dx, rx)), "rgb equal", bool(torch.equal(dc, rc)),
          "absmax", float(dx.abs().max()), "ptrs", dx.data_ptr(), dc.data_ptr(), None if di is None else di.data_ptr(), flush=True)
    try:
        return orig(dx, dc, n, cam, di)
    except Exception as e:
        torch.cuda.synchronize()
        print("  failed:", e, "xyz equal after", bool(torch.equal(dx, rx)), float(dx.abs().max()), flush=True)
        raise
eng.ingest_device = spy
try:
    eng.ingest_stream(iter(frames))
except Exception as e:
    print("ERR", e)
eng2 = vx.MappingEngine(vx.PipelineConfig(voxel_size=0.2))
for i in range(3):
    rx, rc, rn = ref[i]
    try:
        r = eng2.ingest_device(rx, rc, rn, frames[i][2], frames[i][3].cuda())
        print("host-decoded frame", i, "ok", r.voxels_solved)
    except Exception as e:
        print("host-decoded frame", i, "ERR", e)
