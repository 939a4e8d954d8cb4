"""Per-phase cycles of the large-n panel kernel (diagnostics build):

    VX_EXTRA_NVCC_FLAGS=-DVX_PHASE_TIMING python -m paper_2410_17084_b200.build --out=build/pt/libvoxgpr.so
    VX_LIB_PATH=$PWD/build/pt/libvoxgpr.so python tools/panel_phases.py

Thread 0 of every CTA adds clock64 deltas per panel phase: A (GEMM waves),
barrier after A, diagonal factorisation + inverse, B (triangular update),
barrier after B.  Printed as microseconds per CTA per voxel-panel at the
measured clock, for the config-3 scan (latency) and a tail map (throughput).
"""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_2410_17084_b200 as vx  # noqa: E402
from paper_2410_17084_b200 import _native as N  # noqa: E402
from workloads import scenes  # noqa: E402

NAMES = ("A2", "syncA2", "diag||A1", "B", "syncB")


def run(tag, pos, col, reps=2):
    import torch
    lib = N.lib()
    fn = lib.vx_phase_cycles
    fn.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
    buf = (ctypes.c_ulonglong * 20)()
    eng = vx.MappingEngine(vx.PipelineConfig(voxel_size=0.5))
    eng.ingest(pos, col)
    torch.cuda.synchronize()
    fn(buf, 20)
    for _ in range(reps):
        eng.reset()
        eng.ingest(pos, col)
    torch.cuda.synchronize()
    fn(buf, 20)
    cyc = np.array(buf[12:17], dtype=np.float64) / reps
    tot = cyc.sum()
    print(f"{tag}: " + " ".join(f"{n}={c / 1.965e3:10.1f}us({100 * c / tot:4.1f}%)"
                                for n, c in zip(NAMES, cyc)) + "  (sum over CTAs)")


def main():
    pos, col = scenes.config3_scan(seed=0, frame=0)
    run("config3", pos, col)
    pos, col, *_ = scenes.planar_map(100000, voxel_size=0.5, seed=5, bins=scenes.TAIL_BINS,
                                     probs=scenes.TAIL_PROBS)
    run("tail100k", pos, col, reps=1)


if __name__ == "__main__":
    main()
