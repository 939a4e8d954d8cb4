"""Cycles of one 32x32 diagonal-block factorisation + inverse (diagnostics build):
VX_LIB_PATH=$PWD/build/pt/libvoxgpr.so python tools/diag_bench.py"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_2410_17084_b200 import _native as N  # noqa: E402

lib = N.lib()
out = ctypes.c_ulonglong(0)
for iters in (1, 10, 100):
    lib.vx_diag_bench(iters, ctypes.byref(out))
    print(f"iters {iters}: {out.value & ((1 << 62) - 1)} cycles per call, ok={not (out.value >> 62)}")

parts = (ctypes.c_ulonglong * 8)()
lib.vx_diag_parts(parts)
lib.vx_diag_bench(100, ctypes.byref(out))
lib.vx_diag_parts(parts)
names = ("load", "update", "factor8", "solve+publish", "inv_diag", "inv_offdiag")
print("per call:", {n: parts[i] // 100 for i, n in enumerate(names)})
