"""Per-phase SM cycles of the DMMA tile kernel, per voxel, for single-bucket maps.

Run on a GPU box from the repo root (rebuilds the library as a diagnostics
build, so do not commit the resulting .so):

    VX_EXTRA_NVCC_FLAGS=-DVX_PHASE_TIMING python -m paper_2410_17084_b200.build --force
    python tools/phase_timing.py

Each row: training-set sizes, voxels, then cycles per voxel per CTA for
staging+tables, kernel matrix, panel Cholesky, diagonal inverses, forward
substitution, epilogue (thread 0's clock64 between the phase barriers; two
CTAs share an SM, so the sum is the CTA's latency per voxel, not SM time).
"""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_2410_17084_b200 as vx  # noqa: E402
from paper_2410_17084_b200 import _native as N  # noqa: E402
from workloads import scenes  # noqa: E402

PHASES = ("stage", "fill", "chol", "linv", "trsm", "epilogue", "f.loads", "f.chain", "f.publish",
          "f.rows", "c.update", "c.barrier")


def main():
    lib = N.lib()
    fn = lib.vx_phase_cycles
    fn.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
    buf = (ctypes.c_ulonglong * 12)()
    for lo, hi in ((33, 64), (65, 96), (97, 128)):
        pos, col, counts, keys, owner = scenes.planar_map(20000, voxel_size=0.5, seed=1,
                                                          bins=[(lo, hi + 1)], probs=[1.0])
        eng = vx.MappingEngine(vx.PipelineConfig(voxel_size=0.5))
        eng.ingest(pos, col)                     # warm-up (and JIT of nothing)
        eng = vx.MappingEngine(vx.PipelineConfig(voxel_size=0.5))
        fn(buf, 12)
        rep = eng.ingest(pos, col)
        import torch
        torch.cuda.synchronize()
        fn(buf, 12)
        solved = max(int(getattr(rep, "voxels_solved", len(counts))), 1)
        cyc = np.array(buf[:12], dtype=np.float64) / solved
        print(f"n {lo:3d}-{hi:3d} voxels {solved:6d} " +
              " ".join(f"{p}={c:8.0f}" for p, c in zip(PHASES, cyc)) + f" total={cyc[:6].sum():8.0f}")


if __name__ == "__main__":
    main()
