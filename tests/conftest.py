"""Shared pytest setup: the `gpu` marker and repo-root imports."""

import os
import sys

for _v in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS"):
    os.environ.setdefault(_v, "1")      # oracle speed: single-threaded small LAPACK calls

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def pytest_configure(config):
    config.addinivalue_line(
        "markers", "gpu: needs a B200 (sm_100a) and the built CUDA extension")


def pytest_sessionstart(session):
    """Build libvoxgpr.so in-tree if it is missing or stale (nvcc cross-compiles
    without a GPU); the C-ABI export checks need the library."""
    try:
        from paper_2410_17084_b200 import build as _b
        _b.build()
    except Exception as exc:   # surfaced by the tests that need the library
        print(f"[conftest] libvoxgpr build failed: {exc}")
