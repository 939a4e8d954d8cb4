"""Hash-sharded mapping on the GPU: two shard processes == one unsharded map.

Two processes share the box's single B200 (gloo carries the collectives
through host memory; no kernel of one rank waits on the other).  Each rank
runs `ShardedEngine` over the same frames and keeps only its voxels; after
every frame `gather_frame` hands the frame's predictions and new Gaussian
records to rank 0 (gather-v + order-key sort, sharding.py).  Rank 0's merged
outputs must equal the unsharded `MappingEngine` run BIT FOR BIT and in the
same order (voxel_map.py:324-326, pipeline.py:139-171),
including re-fits (eta 2e-5) and a global expansion threshold.
"""

import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

FRAMES = 4
PRED = ("keys", "order", "positions", "colors", "variances")
GAUSS = ("position", "scale", "rotation", "opacity", "color", "source_key")


def _frames():
    from workloads import scenes
    sc = scenes.OutdoorScene.make(0)
    out = []
    for f in range(FRAMES):
        pos, col = scenes.config1_scan(seed=0, frame=f, rays=30000)
        pin = scenes.camera_for(f, 160, 120, 100.0)
        out.append((pos, col, pin, scenes.render_image(sc, pin)))
    return out


def _camera(pin):
    import paper_2410_17084_b200 as vx
    return vx.Camera(pin.fx, pin.fy, pin.cx, pin.cy, pin.width, pin.height, pin.R, pin.t)


def _config(threshold):
    import paper_2410_17084_b200 as vx
    return vx.PipelineConfig(voxel_size=0.5, eta=2e-5, expansion_threshold=threshold)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_main(rank, world, port, threshold, outdir, sliced=False):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2410_17084_b200 import sharding
        eng = sharding.ShardedEngine(_config(threshold), rank, world)
        for f, (pos, col, pin, img) in enumerate(_frames()):
            if sliced:
                # input slicing: this rank H2Ds rows [lo, hi) of the scan only
                lo, hi = rank * len(pos) // world, (rank + 1) * len(pos) // world
                dx = torch.from_numpy(np.ascontiguousarray(pos[lo:hi])).cuda()
                dc = torch.from_numpy(np.ascontiguousarray(col[lo:hi])).cuda()
                di = torch.from_numpy(img).cuda()
                eng.ingest_sliced(dx, dc, hi - lo, lo, _camera(pin), di)
            else:
                eng.ingest(pos, col, _camera(pin), img)
            out = eng.gather_frame(dst=0)
            if rank == 0:
                np.savez(os.path.join(outdir, f"frame{f}.npz"),
                         **{"p_" + k: v.cpu().numpy() for k, v in out["predictions"].items()},
                         **{"g_" + k: v.cpu().numpy() for k, v in out["gaussians"].items()})
        allrec = eng.gather(dst=0)
        if rank == 0:
            np.savez(os.path.join(outdir, "map.npz"), **{k: v.cpu().numpy() for k, v in allrec.items()})
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("threshold,sliced", [(1, False), (2500, False), (1, True), (2500, True)])
def test_two_shards_equal_unsharded(threshold, sliced):
    """sliced: each rank holds half of every scan and the points reach their
    owners through `ingest_sliced`'s all-to-all (order keys from the global
    row numbers); the outputs must still equal the unsharded run."""
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2410_17084_b200 as vx

    # unsharded reference run in this process
    eng = vx.MappingEngine(_config(threshold), track_order=True)
    want, first = [], 0
    for pos, col, pin, img in _frames():
        rep = eng.ingest(pos, col, _camera(pin), img)
        p = {k: v.cpu().numpy() for k, v in eng.frame_predictions().items()}
        g = {k: v[first:].cpu().numpy() for k, v in eng.gaussians_device().items()}
        first = eng.num_gaussians
        want.append((p, g, rep))
    want_map = {k: v.cpu().numpy() for k, v in eng.gaussians_device().items()}
    if threshold > 1:   # the threshold defers at least one frame's records
        assert any(r.primitives_added == 0 and r.newly_active for _, _, r in want)
    assert sum(r.voxels_solved - r.newly_active for _, _, r in want) > 0   # re-fits happened

    with tempfile.TemporaryDirectory() as d:
        ctx = mp.get_context("spawn")
        port = _free_port()
        procs = [ctx.Process(target=_rank_main, args=(r, 2, port, threshold, d, sliced))
                 for r in range(2)]
        for p in procs:
            p.start()
        for p in procs:
            p.join(timeout=600)
            assert p.exitcode == 0
        for f, (p, g, rep) in enumerate(want):
            got = np.load(os.path.join(d, f"frame{f}.npz"))
            assert len(got["p_keys"]) == rep.voxels_solved
            for k in PRED:
                np.testing.assert_array_equal(got["p_" + k], p[k], err_msg=f"frame {f} {k}")
            for k in GAUSS:
                np.testing.assert_array_equal(got["g_" + k], g[k], err_msg=f"frame {f} {k}")
        got = np.load(os.path.join(d, "map.npz"))
        for k in GAUSS:
            np.testing.assert_array_equal(got[k], want_map[k], err_msg=k)
