"""BASELINE config 4, Livox-tail variant, at FULL size on a B200.

The 1,000,000-voxel planar map with the points-per-voxel histogram of the
config-3 rosette scan (n from 10 to 742; ~62M points), one
scan through `MappingEngine.ingest` — the `tail` leg of bench.py, whose n > 160
voxels run on the augmented panel-Cholesky kernel.  Held to the size-
independent properties of test_full_size.py, plus 48 sampled voxels — the 10
largest of the map among them — replayed through the oracle:

* n <= 64: the parity tolerances of test_gpu_parity.py (positions 1e-11 m,
  variances rtol 1e-9 / atol 1e-12);
* n > 64: within 10x the disagreement between the oracle's own two FP64 routes
  (LAPACK Cholesky, gpr.py:187-198, vs the explicit inverse of the reference's
  test oracle, tests/_oracles.py:10-35): at cond(K + Sigma) ~ 1e6-1e7 no FP64
  route is closer to the exact answer than that;
* grid coordinates of every sampled prediction and the nearest-colour sources
  bit-exact, whatever the conditioning.
"""

import math

import numpy as np
import pytest

import paper_2410_17084_b200 as vx
from oracle import voxsplat_oracle as O
from paper_2410_17084_b200 import _native as N
from workloads import scenes

pytestmark = pytest.mark.gpu

RTOL, ATOL, POS_ATOL = 1e-9, 1e-12, 1e-11
PARAM_AXES = {0: (1, 2), 1: (2, 0), 2: (0, 1)}      # gpr.py:36


@pytest.fixture(scope="module")
def run():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    N.lib()
    nvox = 1_000_000
    pos, col, counts, keys, owner = scenes.planar_map(nvox, voxel_size=0.5, seed=5,
                                                      bins=scenes.TAIL_BINS,
                                                      probs=scenes.TAIL_PROBS)
    side = int(math.ceil(math.sqrt(nvox)))
    R, t = scenes.look_at((0.25 * side, 0.25 * side, 150.0),
                          (0.25 * side, 0.25 * side + 1e-3, 0.0), up=(0.0, 1.0, 0.0))
    cam = vx.Camera(500.0, 500.0, 319.5, 239.5, 640, 480, R, t)
    img = np.random.default_rng(98).uniform(0.0, 1.0, (480, 640, 3))
    config = vx.PipelineConfig(voxel_size=0.5)
    eng = vx.MappingEngine(config, voxel_capacity=int(nvox * 1.05),
                           point_capacity=int(len(pos) * 1.6), gaussian_capacity=9 * nvox + 1024)
    rep = eng.ingest(pos, col, cam, img)
    torch.cuda.synchronize()
    return dict(pos=pos, col=col, counts=counts, owner=owner, cam=cam, img=img, config=config,
                eng=eng, rep=rep, side=side, nvox=nvox)


def test_tail_map_report_and_properties(run):
    import torch
    counts, nvox = run["counts"], run["nvox"]
    assert counts.max() >= 700 and (counts > 160).sum() > 50000
    rep = run["rep"]
    assert rep.voxels_touched == nvox and rep.voxels_solved == nvox
    assert rep.primitives_added == 9 * nvox and rep.errors == []
    v = run["eng"].vmap.device_view()
    V, M = int(v.num_voxels), int(v.pred_points)
    assert int(v.solved) == nvox
    cnt = N.view_tensor(v.raw_count, (V,), np.int32).cpu().numpy()
    _, first = np.unique(run["owner"], return_index=True)
    order = np.argsort(first, kind="stable")
    np.testing.assert_array_equal(cnt, counts[order])            # per-voxel point sets
    var = N.view_tensor(v.pred_var, (V, M), np.float64)
    assert bool(((var >= 0) & (var <= 1)).all())
    st = N.view_tensor(v.state, (V,), np.uint8).cpu().numpy()
    mv = var.mean(dim=1).cpu().numpy()
    np.testing.assert_array_equal(st == 3, mv <= run["config"].eta)
    g = run["eng"].gaussians_device()
    assert bool(torch.isfinite(g["position"]).all())


def test_tail_sampled_voxels_incl_largest_against_oracle(run):
    nvox, owner, counts = run["nvox"], run["owner"], run["counts"]
    largest = np.argsort(counts, kind="stable")[-10:]
    rng = np.random.default_rng(6)
    rest = rng.choice(np.setdiff1d(np.arange(nvox), largest), 38, replace=False)
    sample = np.sort(np.concatenate([largest, rest]))
    mask = np.isin(owner, sample)
    cfg = run["config"]
    omap = O.OracleMap(cfg.voxel_size, cfg.sensor_var, cfg.tau, cfg.eta)
    res = O.ingest(omap, run["pos"][mask], run["col"][mask], O.DensifyConfig())
    assert len(res["predictions"]) == len(sample)
    inv = np.empty(nvox, dtype=np.int64)
    _, first = np.unique(owner, return_index=True)
    inv[np.argsort(first, kind="stable")] = np.arange(nvox)
    side = run["side"]
    v = run["eng"].vmap.device_view()
    V, M = int(v.num_voxels), int(v.pred_points)
    slots = N.view_tensor(v.pred_slot, (V,), np.int32)
    big = 0
    for pred in res["predictions"]:
        k = pred["key"]
        i = int(inv[k[0] + k[1] * side])
        s = int(slots[i].item())
        px = N.view_tensor(v.pred_xyz, (s + 1, M, 3), np.float64)[s].cpu().numpy()
        pc = N.view_tensor(v.pred_rgb, (s + 1, M, 3), np.float64)[s].cpu().numpy()
        pv = N.view_tensor(v.pred_var, (s + 1, M), np.float64)[s].cpu().numpy()
        ax = pred["value_axis"]
        other = list(PARAM_AXES[ax])
        np.testing.assert_array_equal(px[:, other], pred["positions"][:, other])
        np.testing.assert_array_equal(pc, pred["colors"])
        n = int(counts[k[0] + k[1] * side])
        if n <= 64:
            np.testing.assert_allclose(px, pred["positions"], rtol=RTOL, atol=POS_ATOL)
            np.testing.assert_allclose(pv, pred["variances"], rtol=RTOL, atol=ATOL)
            continue
        big += 1
        tp, tc, tn = omap.training(k)
        a2, f, x = O.select_axis(tp)
        assert a2 == ax
        mf = f.mean()
        pa, pb = PARAM_AXES[ax]
        lo = np.array(k, dtype=np.float64) * cfg.voxel_size
        xs = O.mesh_grid(((lo[pa], lo[pa] + cfg.voxel_size), (lo[pb], lo[pb] + cfg.voxel_size)),
                         cfg.n_s, cfg.n_r)
        mu2, var2 = O.dense_inverse_posterior(x, f - mf, tn, xs, cfg.kernel_lambda)[:2]
        mu1 = pred["positions"][:, ax] - mf
        var1 = pred["variances"]
        assert np.abs(px[:, ax] - pred["positions"][:, ax]).max() <= \
            10 * np.abs(mu2 - mu1).max() + POS_ATOL
        assert np.abs(pv - var1).max() <= 10 * np.abs(np.clip(var2, 0, None) - var1).max() + ATOL
    assert big >= 10
