"""bench.py's N > 1 path (one map hash-sharded over the ranks, each rank holding
its slice of the scan, ShardedEngine.ingest_sliced + gather_frame) run with
two ranks on the box's single GPU over gloo (VX_BENCH_BACKEND=gloo; the driver
runs the same code with NCCL on N GPUs).  Checks the JSON contract of the
line rank 0 prints: every voxel solved, the sharded parallelism label, the
e2e H2D counting only this rank's slice."""

import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_bench_two_ranks_gloo():
    env = dict(os.environ, VX_BENCH_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", "2",
           "--steps", "3", "--warmup", "3", "--voxels", "50000", "--no-cpu", "--traj-scans", "0",
           "--scan-reps", "0", "--tail-voxels", "0"]
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["steps"] == 3 and d["value"] > 0
    assert d["config"]["solved_per_step"] == d["config"]["voxels"]
    assert "ingest_sliced" in d["config"]["parallelism"]
    # each rank copies its half of the scan (+ the image), not the whole scan
    assert d["e2e"]["h2d_bytes_per_step"] < 0.6 * 48 * d["config"]["points"] + 8e6
