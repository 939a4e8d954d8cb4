"""Forward splat renderer on the device vs the reference (renderer.py:90-207).

Golden scenes come from the real reference (tests/golden/render.npz, made by
tests/golden/make_golden.py); larger scenes are checked against the pinned
oracle restatement.  Discrete outputs (validity, pixel bounding boxes, the
depth order) are exact; projections and images agree to FP64 rounding: the
per-pixel quadratic form and the blend follow NumPy's operation order, so
pixels differ only through exp() (<= 1 ulp) and the einsum order of the 3x3
covariance products.  The reference's own renderer tests
(tests/test_renderer.py) are restated at their tolerances.
"""

import numpy as np
import pytest

import paper_2410_17084_b200 as vx
from oracle import voxsplat_oracle as O
from paper_2410_17084_b200 import renderer as R
from paper_2410_17084_b200.splat_init import GaussianPrimitive
from tests import _fixtures as F

pytestmark = pytest.mark.gpu

IMG_ATOL = 1e-12


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2410_17084_b200 import _native as N
    N.lib()


def _scene(g, tag):
    cv = g[f"{tag}_cam"]
    cam = vx.Camera(fx=cv[0], fy=cv[1], cx=cv[2], cy=cv[3], width=int(cv[4]), height=int(cv[5]),
                    rotation=cv[6:15].reshape(3, 3), translation=cv[15:18])
    gm = vx.GaussianMap.from_arrays(g[f"{tag}_pos"], g[f"{tag}_scale"], g[f"{tag}_rot"],
                                    g[f"{tag}_opacity"], g[f"{tag}_sh0"],
                                    np.zeros((len(g[f"{tag}_pos"]), 3), dtype=np.int64))
    return cam, gm


@pytest.mark.parametrize("tag", ["a", "b", "c"])
def test_projection_matches_reference_golden(tag):
    g = F.load("render.npz")
    cam, _ = _scene(g, tag)
    ps = R.project_points(g[f"{tag}_pos"], g[f"{tag}_scale"], g[f"{tag}_rot"], cam)
    np.testing.assert_array_equal(ps.valid, g[f"{tag}_valid"])
    np.testing.assert_array_equal(ps.bbox, g[f"{tag}_bbox"])
    v = ps.valid
    np.testing.assert_allclose(ps.mean2d[v], g[f"{tag}_mean2d"][v], rtol=1e-12, atol=1e-9)
    np.testing.assert_allclose(ps.cov2d[v], g[f"{tag}_cov2d"][v], rtol=1e-9, atol=1e-9)
    np.testing.assert_allclose(ps.depth, g[f"{tag}_pdepth"], rtol=1e-14, atol=1e-14)
    np.testing.assert_allclose(ps.radius[v], g[f"{tag}_radius"][v], rtol=1e-9)


@pytest.mark.parametrize("tag", ["a", "b", "c"])
def test_render_matches_reference_golden(tag):
    g = F.load("render.npz")
    cam, gm = _scene(g, tag)
    buf = R.render(gm, cam)
    np.testing.assert_allclose(buf.color, g[f"{tag}_color"], atol=IMG_ATOL)
    np.testing.assert_allclose(buf.depth, g[f"{tag}_depth"], atol=10 * IMG_ATOL)
    np.testing.assert_allclose(buf.silhouette, g[f"{tag}_sil"], atol=IMG_ATOL)


def _random_map(rng, n, spread=3.0):
    pos = rng.uniform([-spread, -spread, -0.5], [spread, spread, 1.5], (n, 3))
    scl = rng.uniform(0.01, 0.3, (n, 3))
    rot = rng.normal(size=(n, 4))
    rot /= np.linalg.norm(rot, axis=1, keepdims=True)
    opa = rng.uniform(0.05, 1.0, n)
    sh0 = (rng.uniform(0, 1, (n, 3)) - 0.5) / 0.28209479177
    return pos, scl, rot, opa, sh0


@pytest.mark.parametrize("n,w,h", [(3000, 160, 120), (20000, 333, 197)])
def test_render_matches_oracle_large(n, w, h):
    """Many overlapping splats over ragged tiles (image not a multiple of 16):
    exercises the tile lists, chunked staging and the early-termination."""
    rng = np.random.default_rng(n)
    pos, scl, rot, opa, sh0 = _random_map(rng, n)
    cam = vx.Camera.looking_at((0.2, -7.0, 2.5), (0.0, 0.0, 0.3), fx=0.8 * w, fy=0.8 * w,
                               cx=(w - 1) / 2, cy=(h - 1) / 2, width=w, height=h)
    gm = vx.GaussianMap.from_arrays(pos, scl, rot, opa, sh0, np.zeros((n, 3), dtype=np.int64))
    buf = R.render(gm, cam)
    ocam = dict(fx=cam.fx, fy=cam.fy, cx=cam.cx, cy=cam.cy, width=w, height=h, R=cam.rotation,
                t=cam.translation)
    color, depth, sil, _ = O.render_splats(pos, scl, rot, opa, sh0, ocam)
    np.testing.assert_allclose(buf.color, color, atol=1e-11)
    np.testing.assert_allclose(buf.depth, depth, atol=1e-10)
    np.testing.assert_allclose(buf.silhouette, sil, atol=1e-11)
    assert buf.silhouette.max() > 0.99          # saturated pixels occurred


def test_device_records_render_like_host_map():
    """render() on the engine's device records (no host round trip) equals the host map."""
    from workloads import scenes
    pos, col = scenes.config1_scan(seed=0, frame=0, rays=20000)
    eng = vx.MappingEngine(vx.PipelineConfig(voxel_size=0.5))
    sc = scenes.OutdoorScene.make(0)
    pin = scenes.camera_for(0, 160, 120, 100.0)
    cam = vx.Camera(pin.fx, pin.fy, pin.cx, pin.cy, pin.width, pin.height, pin.R, pin.t)
    eng.ingest(pos, col, cam, scenes.render_image(sc, pin))
    assert eng.num_gaussians > 0
    dev = R.render(eng.gaussians_device(), cam)
    gm = eng.gaussian_map()
    host = R.render(gm, cam)
    np.testing.assert_array_equal(dev.color, host.color)
    np.testing.assert_array_equal(dev.silhouette, host.silhouette)
    assert dev.silhouette.max() > 0.5


# ---------------------------------------------------------------------------
# the reference's own renderer cases (tests/test_renderer.py), same tolerances
# ---------------------------------------------------------------------------
def _splat(position, color=(1.0, 1.0, 1.0), opacity=1.0, scale=0.05):
    return GaussianPrimitive(position=np.asarray(position, dtype=float), scale=np.full(3, scale),
                             rotation=np.array([1.0, 0.0, 0.0, 0.0]), opacity=opacity,
                             color=(np.asarray(color, dtype=float) - 0.5) / 0.28209479177)


def _center_camera():
    return vx.Camera(fx=100, fy=100, cx=50, cy=50, width=100, height=100)


def _camera(width=100, height=100, fx=100.0, fy=100.0):
    return vx.Camera(fx=fx, fy=fy, cx=(width - 1) / 2, cy=(height - 1) / 2, width=width, height=height)


def test_projection_hand_cases():
    p = R.project_gaussian(_splat((0.0, 0.0, 1.0)), _center_camera())
    np.testing.assert_allclose(p.mean2d, [50.0, 50.0])
    assert p.depth == 1.0
    assert R.project_gaussian(_splat((0.0, 0.0, -1.0)), _center_camera()) is None
    assert R.project_gaussian(_splat((0.0, 0.0, 0.005)), _center_camera()) is None
    s, z = 0.03, 2.0
    p = R.project_gaussian(_splat((0.0, 0.0, z), scale=s), _center_camera())
    e = (100.0 * s / z) ** 2 + R.COV_DILATION
    np.testing.assert_allclose(p.cov2d, np.diag([e, e]), atol=1e-6)
    assert R.project_gaussian(_splat((50.0, 0.0, 1.0)), _center_camera()) is None


def test_single_opaque_and_two_splat_blend():
    cam = _center_camera()
    buf = R.render([_splat((0.0, 0.0, 1.5), color=(0.3, 0.6, 0.9), opacity=1.0, scale=0.2)], cam)
    np.testing.assert_allclose(buf.silhouette[50, 50], 0.99, atol=1e-12)
    np.testing.assert_allclose(buf.color[50, 50], 0.99 * np.array([0.3, 0.6, 0.9]), atol=1e-9)
    np.testing.assert_allclose(buf.depth[50, 50], 0.99 * 1.5, atol=1e-9)
    front = _splat((0.0, 0.0, 1.0), color=(1, 0, 0), opacity=0.5, scale=0.2)
    back = _splat((0.0, 0.0, 2.0), color=(0, 0, 1), opacity=0.5, scale=0.4)
    buf = R.render([front, back], cam)
    np.testing.assert_allclose(buf.color[50, 50], [0.5, 0.0, 0.25], atol=1e-6)
    np.testing.assert_allclose(buf.silhouette[50, 50], 0.75, atol=1e-6)
    np.testing.assert_allclose(buf.depth[50, 50], 0.5 * 1.0 + 0.25 * 2.0, atol=1e-6)


def test_empty_map():
    buf = R.render([], _camera())
    assert np.all(buf.color == 0) and np.all(buf.depth == 0) and np.all(buf.silhouette == 0)


def _random_scene(rng, n):
    return [_splat(position=rng.uniform([-0.6, -0.6, 0.8], [0.6, 0.6, 3.0]),
                   color=rng.uniform(0, 1, 3), opacity=float(rng.uniform(0.2, 1.0)),
                   scale=float(rng.uniform(0.02, 0.15))) for _ in range(n)]


def test_silhouette_identity_and_permutation_invariance():
    rng = np.random.default_rng(0)
    cam = _camera(64, 64, fx=64, fy=64)
    prims = _random_scene(rng, 30)
    buf = R.render(prims, cam)
    ps = R.project_points(np.stack([p.position for p in prims]), np.stack([p.scale for p in prims]),
                          np.stack([p.rotation for p in prims]), cam)
    opac = np.array([p.opacity for p in prims])
    one_minus = np.ones((64, 64))
    for i in R.depth_order(ps.depth, ps.valid):
        x0, x1, y0, y1 = ps.bbox[i]
        a = R.alpha_patch(ps.mean2d[i], ps.cov2d[i], opac[i], x0, x1, y0, y1)
        T = one_minus[y0:y1, x0:x1]
        one_minus[y0:y1, x0:x1] = np.where(T >= 1e-4, T * (1 - a), T)
    np.testing.assert_allclose(buf.silhouette, 1.0 - one_minus, atol=1e-6)
    perm = rng.permutation(len(prims))
    shuffled = R.render([prims[i] for i in perm], cam)
    np.testing.assert_array_equal(shuffled.color, buf.color)
    np.testing.assert_array_equal(shuffled.depth, buf.depth)
    a = _splat((-0.05, 0.0, 1.0), color=(1, 0, 0), opacity=0.6, scale=0.1)
    b = _splat((0.05, 0.0, 1.0), color=(0, 1, 0), opacity=0.6, scale=0.1)
    np.testing.assert_array_equal(R.render([a, b], cam).color, R.render([a, b], cam).color)


def test_monotone_silhouette_bounded_color_and_skip_threshold():
    rng = np.random.default_rng(1)
    cam = _camera(64, 64, fx=64, fy=64)
    prims = _random_scene(rng, 20)
    before = R.render(prims, cam).silhouette
    extra = _splat(rng.uniform([-0.3, -0.3, 1.0], [0.3, 0.3, 2.0]), opacity=0.7, scale=0.1)
    after = R.render(prims + [extra], cam).silhouette
    assert np.all(after >= before - 1e-12)
    rng = np.random.default_rng(2)
    prims = _random_scene(rng, 30)
    buf = R.render(prims, cam)
    for ch in range(3):
        top = max(np.array([0.28209479177 * p.color[ch] + 0.5 for p in prims]).max(), 0.0)
        assert np.all(buf.color[:, :, ch] <= buf.silhouette * top + 1e-6)
    cam = _center_camera()
    faint = _splat((0.0, 0.0, 1.0), color=(1, 1, 1), opacity=R.ALPHA_SKIP * 0.5, scale=0.2)
    solid = _splat((0.0, 0.0, 2.0), color=(0, 1, 0), opacity=0.9, scale=0.4)
    np.testing.assert_array_equal(R.render([faint, solid], cam).color, R.render([solid], cam).color)


def test_depth_order_needs_low_word():
    """Depths that share the high 32 bits of their IEEE pattern but arrive out
    of order (1.0000001 before 1.0): the high-word fast path must fall back to
    the full 64-bit sort; exact ties keep index order."""
    cam = _center_camera()
    a = _splat((0.0, 0.0, 1.0000001), color=(1, 0, 0), opacity=0.6, scale=0.1)
    b = _splat((0.01, 0.0, 1.0), color=(0, 0, 1), opacity=0.6, scale=0.1)
    c = _splat((-0.01, 0.0, 1.0), color=(0, 1, 0), opacity=0.6, scale=0.1)   # exact tie with b
    prims = [a, b, c]
    buf = R.render(prims, cam)
    ocam = dict(fx=cam.fx, fy=cam.fy, cx=cam.cx, cy=cam.cy, width=cam.width, height=cam.height,
                R=cam.rotation, t=cam.translation)
    color, depth, sil, _ = O.render_splats(np.stack([p.position for p in prims]),
                                           np.stack([p.scale for p in prims]),
                                           np.stack([p.rotation for p in prims]),
                                           np.array([p.opacity for p in prims]),
                                           np.stack([p.color for p in prims]), ocam)
    np.testing.assert_allclose(buf.color, color, atol=1e-13)
    np.testing.assert_allclose(buf.silhouette, sil, atol=1e-13)
    # the front splat (b, nearest) dominates the centre pixel colour order
    assert buf.color[50, 50, 2] > buf.color[50, 50, 0]
