"""Pin the CPU oracle to golden vectors produced by the real reference.

CPU-only.  If these pass, the oracle reproduces the reference
(`/root/reference/pkg/src/voxsplat`) on every fixture, so the GPU parity
tests that compare the CUDA path with the oracle are anchored to the
reference itself.
"""

import numpy as np
import pytest

from oracle import voxsplat_oracle as O
from tests import _fixtures as F

RTOL, ATOL = 1e-9, 1e-12     # reference tolerance, tests/test_gpr.py:170-174


@pytest.mark.parametrize("seed", [7, 101, 11])
def test_posterior_matches_reference(seed):
    for x, f, noise, xs, lam, mu, var, full in F.problems(seed):
        m, v, S = O.posterior(x, f, noise, xs, lam, full=full is not None)
        np.testing.assert_allclose(m, mu, rtol=RTOL, atol=ATOL)
        np.testing.assert_allclose(v, var, rtol=RTOL, atol=ATOL)
        if full is not None:
            np.testing.assert_allclose(S, full, rtol=RTOL, atol=ATOL)


def test_posterior_agrees_with_dense_inverse():
    for x, f, noise, xs, lam, *_ in F.problems(7)[:30]:
        m, v, _ = O.posterior(x, f, noise, xs, lam)
        m2, v2, _ = O.dense_inverse_posterior(x, f, noise, xs, lam)
        np.testing.assert_allclose(m, m2, rtol=RTOL, atol=ATOL)
        np.testing.assert_allclose(v, v2, rtol=RTOL, atol=ATOL)


def test_closed_form_and_interpolation():
    d = F.load("gpr_problems.npz")
    mu, var, _ = O.posterior([[0, 0]], [2.0], [0.25], [[0, 0]], 1.0)
    assert abs(mu[0] - 1.6) <= 1e-12 and abs(var[0] - 0.2) <= 1e-12
    np.testing.assert_array_equal(mu, d["closed_mu"])
    mu, var, _ = O.posterior(d["interp_x"], d["interp_f"], np.zeros(25),
                             d["interp_x"], 25.0)
    np.testing.assert_allclose(mu, d["interp_mu"], rtol=1e-9, atol=1e-10)


def test_keys_bit_exact():
    d = F.load("keys.npz")
    np.testing.assert_array_equal(O.keys_of(d["points"], 0.2), d["keys_02"])
    np.testing.assert_array_equal(O.keys_of(d["points"], 0.5), d["keys_05"])


def test_axis_selection_exact():
    for pts, axis in F.axis_sets():
        try:
            got = O.select_axis(pts)[0]
        except O.OracleError:
            got = -1
        assert got == axis


def test_mesh_grids_bit_exact():
    d = F.load("grids.npz")
    i = 0
    while f"g{i}_grid" in d.files:
        e = d[f"g{i}_extent"]
        ns, nr = (int(v) for v in d[f"g{i}_nsnr"])
        got = O.mesh_grid(((e[0, 0], e[0, 1]), (e[1, 0], e[1, 1])), ns, nr)
        np.testing.assert_array_equal(got, d[f"g{i}_grid"])
        i += 1


def test_subgrid_moments():
    d = F.load("subgrids.npz")
    for i in range(len(d["weights"])):
        p, phi = O.subgrid_moments(d["points"][i], d["weights"][i])
        np.testing.assert_array_equal(p, d["position"][i])
        np.testing.assert_allclose(phi, d["phi"][i], atol=1e-15)


def _camera(d, fr):
    fx, fy, cx, cy, w, h = d["camera_intrinsics"]
    return O.OracleCamera(fx, fy, cx, cy, int(w), int(h), d[f"f{fr}_R"], d[f"f{fr}_t"])


def test_scan_replay_matches_reference():
    """3-frame ingest replay: update order, transitions, predictions, Gaussians."""
    d = F.scan_frames()
    vs, eta, sv, tau, lam, jit = d["config"]
    omap = O.OracleMap(vs, sv, int(tau), eta)
    cfg = O.DensifyConfig(kernel_lambda=lam, jitter=jit)
    for fr in range(3):
        p = f"f{fr}_"
        ntr = len(omap.transitions)
        res = O.ingest(omap, d[p + "positions"], d[p + "colors"], cfg,
                       camera=_camera(d, fr), image=d[p + "image"])
        np.testing.assert_array_equal(np.array(res["update"]).reshape(-1, 3), d[p + "update"])
        tr = np.array([[*k, a, b] for _, k, a, b in omap.transitions[ntr:]]).reshape(-1, 5)
        np.testing.assert_array_equal(tr, d[p + "transitions"])
        preds = res["predictions"]
        np.testing.assert_array_equal(np.array([q["key"] for q in preds]).reshape(-1, 3),
                                      d[p + "pred_keys"])
        np.testing.assert_array_equal(np.array([q["value_axis"] for q in preds]),
                                      d[p + "pred_axis"])
        pos = np.stack([q["positions"] for q in preds])
        np.testing.assert_allclose(pos, d[p + "pred_positions"], rtol=RTOL, atol=ATOL)
        np.testing.assert_array_equal(np.stack([q["colors"] for q in preds]),
                                      d[p + "pred_colors"])
        np.testing.assert_allclose(np.stack([q["variances"] for q in preds]),
                                   d[p + "pred_variances"], rtol=RTOL, atol=ATOL)
        g = res["gaussians"]
        if g:
            gp = np.concatenate([x["position"] for x in g])
            np.testing.assert_allclose(gp, d[p + "g_positions"], atol=ATOL)
            np.testing.assert_allclose(np.concatenate([x["scale"] for x in g]),
                                       d[p + "g_scales"], atol=ATOL)
            np.testing.assert_array_equal(np.concatenate([x["color"] for x in g]),
                                          d[p + "g_colors"])
            np.testing.assert_array_equal(np.concatenate([x["source_key"] for x in g]),
                                          d[p + "g_source_keys"])
        else:
            assert len(d[p + "g_positions"]) == 0
    keys = sorted(omap.cells)
    np.testing.assert_array_equal(np.array(keys), d["final_keys"])
    np.testing.assert_array_equal([len(omap.cells[k].raw_pos) for k in keys], d["final_counts"])
    np.testing.assert_array_equal([omap.cells[k].state for k in keys], d["final_states"])


@pytest.mark.parametrize("tag", ["a", "b", "c"])
def test_oracle_renderer_matches_reference_golden(tag):
    """Renderer restatement vs the reference's render()/project_points()."""
    g = F.load("render.npz")
    cv = g[f"{tag}_cam"]
    cam = dict(fx=cv[0], fy=cv[1], cx=cv[2], cy=cv[3], width=int(cv[4]), height=int(cv[5]),
               R=cv[6:15].reshape(3, 3), t=cv[15:18])
    color, depth, sil, pr = O.render_splats(g[f"{tag}_pos"], g[f"{tag}_scale"], g[f"{tag}_rot"],
                                            g[f"{tag}_opacity"], g[f"{tag}_sh0"], cam)
    np.testing.assert_array_equal(pr["valid"], g[f"{tag}_valid"])
    np.testing.assert_array_equal(pr["bbox"], g[f"{tag}_bbox"])
    v = g[f"{tag}_valid"]
    np.testing.assert_allclose(pr["mean2d"][v], g[f"{tag}_mean2d"][v], rtol=1e-12, atol=1e-9)
    np.testing.assert_allclose(pr["cov2d"][v], g[f"{tag}_cov2d"][v], rtol=1e-9, atol=1e-9)
    np.testing.assert_allclose(color, g[f"{tag}_color"], atol=1e-12)
    np.testing.assert_allclose(depth, g[f"{tag}_depth"], atol=1e-11)
    np.testing.assert_allclose(sil, g[f"{tag}_sil"], atol=1e-12)
