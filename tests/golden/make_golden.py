"""Generate golden vectors by running the REAL reference implementation.

Run in the build container only (it imports `voxsplat` from the read-only
reference tree):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Outputs small `.npz` fixtures next to this script.  They hold the inputs
and the reference's outputs, so the GPU box (which has no /root/reference)
can check both the oracle and the CUDA path against them.

Fixtures
  gpr_problems.npz   random problems of the reference tests (seeds 7, 101,
                     tests/_oracles.py:80-89) + closed form + interpolation;
                     outputs of voxsplat.gpr.gpr_solve (gpr.py:173-205)
  keys.npz           voxel_keys (voxel_map.py:136-143) incl. boundary values
  axis.npz           select_value_axis (gpr.py:57-78) on planar/degenerate sets
  grids.npz          make_mesh_grid (gpr.py:104-120) for several (n_s, n_r)
  subgrids.npz       init_position / init_covariance (splat_init.py:92-114)
  scan_frames.npz    3-frame mapping replay through MappingPipeline.ingest_frame
                     (pipeline.py:139-187): update order, per-voxel counts,
                     transitions, predictions, Gaussian map
  render.npz         project_points / render (renderer.py:90-207) on three
                     scenes: the reference tests' random scene, an
                     anisotropic rotated scene under a looking_at camera
                     (incl. behind-camera, off-image, equal-depth and faint
                     splats), and the Gaussian map of the scan replay
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
REF_TESTS = "/root/reference/pkg/tests"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF_SRC)
sys.path.insert(0, REF_TESTS)
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

from voxsplat import Camera, PipelineConfig  # noqa: E402
from voxsplat import gpr as rgpr  # noqa: E402
from voxsplat import splat_init as rsplat  # noqa: E402
from voxsplat import voxel_map as rvm  # noqa: E402
from voxsplat.errors import DegenerateGeometryError  # noqa: E402
from voxsplat.pipeline import FrameSample, MappingPipeline  # noqa: E402
from _oracles import random_gpr_problem  # noqa: E402

from workloads import scenes  # noqa: E402


def pack_problems(problems):
    n = np.array([len(p[0]) for p in problems], dtype=np.int64)
    m = np.array([len(p[3]) for p in problems], dtype=np.int64)
    return dict(
        n=n, m=m, lam=np.array([p[4] for p in problems]),
        x=np.concatenate([p[0] for p in problems]),
        f=np.concatenate([p[1] for p in problems]),
        noise=np.concatenate([p[2] for p in problems]),
        xs=np.concatenate([p[3] for p in problems]))


def gpr_fixture():
    out = {}
    for seed, count, nmax in ((7, 100, 64), (101, 100, 64), (11, 200, 24)):
        rng = np.random.default_rng(seed)
        probs = [random_gpr_problem(rng, n_max=nmax, m_max=81 if nmax > 24 else 36)
                 for _ in range(count)]
        pk = pack_problems(probs)
        mus, vs, fulls = [], [], []
        for i, (x, f, noise, xs, lam) in enumerate(probs):
            r = rgpr.gpr_solve(rgpr.GprProblem(x, f, noise, xs, lam),
                               return_full=(seed == 7 and i < 8))
            mus.append(r.mu_star)
            vs.append(r.sigma_star_diag)
            if r.sigma_star_full is not None:
                fulls.append(r.sigma_star_full.ravel())
        pk["mu"] = np.concatenate(mus)
        pk["var"] = np.concatenate(vs)
        if fulls:
            pk["full"] = np.concatenate(fulls)
        for k, v in pk.items():
            out[f"s{seed}_{k}"] = v
    # closed form (tests/test_gpr.py:143-147)
    r = rgpr.gpr_solve(rgpr.GprProblem(x=[[0, 0]], f=[2.0], noise_diag=[0.25],
                                       x_star=[[0, 0]]))
    out["closed_mu"], out["closed_var"] = r.mu_star, r.sigma_star_diag
    # noiseless interpolation (tests/test_gpr.py:149-162)
    rng = np.random.default_rng(6)
    gx, gy = np.meshgrid(np.linspace(0, 1, 5), np.linspace(0, 1, 5))
    x = np.column_stack([gx.ravel(), gy.ravel()]) + rng.uniform(-0.05, 0.05, (25, 2))
    f = np.sin(3 * x[:, 0]) + x[:, 1]
    r = rgpr.gpr_solve(rgpr.GprProblem(x=x, f=f, noise_diag=np.zeros(25),
                                       x_star=x, lam=25.0))
    out.update(interp_x=x, interp_f=f, interp_mu=r.mu_star, interp_var=r.sigma_star_diag)
    np.savez_compressed(os.path.join(HERE, "gpr_problems.npz"), **out)


def keys_fixture():
    rng = np.random.default_rng(20)
    pts = rng.uniform(-3, 3, (2000, 3))
    # exact lattice boundaries and near-boundary values
    grid = np.arange(-10, 11) * 0.2
    edge = np.stack([grid, grid[::-1], np.roll(grid, 3)], axis=1)
    nudged = np.concatenate([edge, np.nextafter(edge, -np.inf), np.nextafter(edge, np.inf)])
    pts = np.concatenate([pts, nudged, [[0.05, 0.19, -0.01], [0.0, 0.0, 0.0]]])
    np.savez_compressed(os.path.join(HERE, "keys.npz"), points=pts,
                        keys_02=rvm.voxel_keys(pts, 0.2), keys_05=rvm.voxel_keys(pts, 0.5))


def axis_fixture():
    rng = np.random.default_rng(21)
    sets, axes = [], []
    for i in range(300):
        n = int(rng.integers(3, 120))
        normal = rng.normal(size=3)
        normal /= np.linalg.norm(normal)
        basis = np.linalg.svd(normal[None, :])[2][1:]
        pts = rng.uniform(-0.25, 0.25, (n, 2)) @ basis
        pts += rng.uniform(0.0, 0.03) * rng.normal(size=(n, 1)) * normal
        pts += rng.uniform(-5, 5, 3)
        if i % 25 == 0:
            pts = np.full((n, 3), 0.3)            # coincident
        elif i % 25 == 1:
            pts = np.outer(np.linspace(0, 1, n), rng.normal(size=3))  # collinear
        sets.append(pts)
        try:
            axes.append(rgpr.select_value_axis(pts).value_axis)
        except DegenerateGeometryError:
            axes.append(-1)
    np.savez_compressed(os.path.join(HERE, "axis.npz"),
                        n=np.array([len(s) for s in sets]),
                        points=np.concatenate(sets), axis=np.array(axes))


def grids_fixture():
    out = {}
    cases = [((0.0, 0.2), (0.0, 0.2), 3, 3), ((0.4, 0.6), (-1.2, -1.0), 1, 1),
             ((-3.5, -3.0), (12.0, 12.5), 2, 2), ((0.0, 0.9), (0.0, 0.9), 4, 3),
             ((1.3, 1.8), (-0.5, 0.0), 4, 4), ((7.1, 7.3), (2.2, 2.4), 3, 2)]
    for i, (e0, e1, ns, nr) in enumerate(cases):
        out[f"g{i}_extent"] = np.array([e0, e1], dtype=np.float64)
        out[f"g{i}_nsnr"] = np.array([ns, nr])
        out[f"g{i}_grid"] = rgpr.make_mesh_grid((e0, e1), ns, nr)
    np.savez_compressed(os.path.join(HERE, "grids.npz"), **out)


def subgrid_fixture():
    rng = np.random.default_rng(106)
    pts = rng.uniform(-1, 1, (200, 9, 3))
    w = rng.uniform(0.05, 20.0, (200, 9))
    pos, phi, scale = [], [], []
    for i in range(200):
        g = rsplat.Subgrid(points=pts[i], weights=w[i], colors=np.full((9, 3), 0.5))
        p = rsplat.init_position(g)
        ph, s, _ = rsplat.init_covariance(g, p)
        pos.append(p)
        phi.append(ph)
        scale.append(s)
    np.savez_compressed(os.path.join(HERE, "subgrids.npz"), points=pts, weights=w,
                        position=np.array(pos), phi=np.array(phi), scale=np.array(scale))


def scan_fixture():
    """A small 3-frame replay of the reference ingest (store, densify, init).

    Small scene (ground + boxes + spheres seen from close range, 0.2 m voxels)
    with eta=2e-5 so frames 2 and 3 re-fit ACTIVE voxels from raw ∪ pseudo.
    """
    config = PipelineConfig(voxel_size=0.2, eta=2e-5, sensor_var=1e-4,
                            iterations=0, expansion_threshold=1)
    sc = scenes.OutdoorScene.make(3, n_boxes=6, n_spheres=6, half=12.0)
    pipe = MappingPipeline(config)
    out = {}
    for fr in range(3):
        eye = (0.3 * fr, 0.0, 1.8)
        pos, col = scenes.scan(sc, eye, (eye[0] + 10, 0.0, 1.8), 3, fr,
                               rays=6000, rows=16, fov_az=np.radians(60.0),
                               fov_el=np.radians(30.0))
        cam = Camera(fx=60.0, fy=60.0, cx=39.5, cy=29.5, width=80, height=60,
                     rotation=scenes.look_at(eye, (eye[0] + 10, 0.0, 1.8))[0],
                     translation=scenes.look_at(eye, (eye[0] + 10, 0.0, 1.8))[1])
        pin = scenes.Pinhole(60.0, 60.0, 39.5, 29.5, 80, 60, cam.rotation, cam.translation)
        image = scenes.render_image(sc, pin)
        ntr = len(pipe.vmap.transitions)
        nsolve = len(pipe.vmap.solve_log)
        ngs = len(pipe.gmap)
        # capture the update set and predictions exactly as ingest sees them
        captured = {}
        orig = rgpr.densify_frame

        def spy(update, vmap, cfg):
            captured["update"] = list(update)
            preds = orig(update, vmap, cfg)
            captured["preds"] = preds
            return preds
        import voxsplat.pipeline as rp
        rp.densify_frame = spy
        try:
            pipe.ingest_frame(FrameSample(float(fr), rvm.PointCloud(pos, col, np.zeros(len(pos))),
                                          image, cam))
        finally:
            rp.densify_frame = orig
        p = f"f{fr}_"
        out[p + "positions"], out[p + "colors"] = pos, col
        out[p + "R"], out[p + "t"], out[p + "image"] = cam.rotation, cam.translation, image
        out[p + "update"] = np.array(captured["update"], dtype=np.int64).reshape(-1, 3)
        tr = pipe.vmap.transitions[ntr:]
        out[p + "transitions"] = np.array(
            [[*t.key, int(t.old), int(t.new)] for t in tr], dtype=np.int64).reshape(-1, 5)
        preds = captured["preds"]
        out[p + "pred_keys"] = np.array([pr.key for pr in preds], dtype=np.int64).reshape(-1, 3)
        out[p + "pred_positions"] = np.stack([pr.positions for pr in preds])
        out[p + "pred_colors"] = np.stack([pr.colors for pr in preds])
        out[p + "pred_variances"] = np.stack([pr.variances for pr in preds])
        out[p + "pred_axis"] = np.array([pipe.vmap.cells[pr.key].value_axis for pr in preds])
        out[p + "solve_log_len"] = np.array(len(pipe.vmap.solve_log) - nsolve)
        g = pipe.gmap
        out[p + "g_positions"] = g.positions[ngs:]
        out[p + "g_scales"] = g.scales[ngs:]
        out[p + "g_rotations"] = g.rotations[ngs:]
        out[p + "g_opacities"] = g.opacities[ngs:]
        out[p + "g_colors"] = g.colors[ngs:]
        out[p + "g_source_keys"] = g.source_keys[ngs:]
    keys = sorted(pipe.vmap.cells)
    out["final_keys"] = np.array(keys, dtype=np.int64)
    out["final_counts"] = np.array([pipe.vmap.cells[k].point_count for k in keys])
    out["final_states"] = np.array([int(pipe.vmap.cells[k].state) for k in keys])
    out["camera_intrinsics"] = np.array([60.0, 60.0, 39.5, 29.5, 80, 60])
    out["config"] = np.array([config.voxel_size, config.eta, config.sensor_var,
                              config.tau, config.kernel_lambda, config.jitter])
    np.savez_compressed(os.path.join(HERE, "scan_frames.npz"), **out)


def ply_fixture():
    """PLY files written by the reference writer (formats.py:42-63) and the
    reference reader's output (formats.py:66-147)."""
    from voxsplat import formats as rformats
    rng = np.random.default_rng(30)
    pos = rng.uniform(-50, 50, (500, 3))
    col = rng.uniform(0, 1, (500, 3))
    cloud = rvm.PointCloud(pos, col, np.zeros(500))
    out = {}
    for binary, name in ((True, "scan_bin.ply"), (False, "scan_ascii.ply")):
        path = os.path.join(HERE, name)
        rformats.write_ply(path, cloud, binary=binary)
        back = rformats.read_ply(path, noise_var=0.25)
        out[name + "_positions"] = back.positions
        out[name + "_colors"] = back.colors
    np.savez_compressed(os.path.join(HERE, "ply_ref.npz"), **out)


def render_fixture():
    from voxsplat.renderer import project_points, render
    from voxsplat.splat_init import GaussianPrimitive, rgb_to_sh0
    out = {}

    def add(tag, pos, scl, rot, opa, sh0, cam):
        prims = [GaussianPrimitive(position=pos[i], scale=scl[i], rotation=rot[i] / np.linalg.norm(rot[i]),
                                   opacity=float(opa[i]), color=sh0[i]) for i in range(len(pos))]
        buf = render(prims, cam)
        ps = project_points(pos, scl, rot, cam)
        for k, v in (("pos", pos), ("scale", scl), ("rot", rot), ("opacity", opa), ("sh0", sh0),
                     ("color", buf.color), ("depth", buf.depth), ("sil", buf.silhouette),
                     ("mean2d", ps.mean2d), ("cov2d", ps.cov2d), ("pdepth", ps.depth),
                     ("radius", ps.radius), ("valid", ps.valid), ("bbox", ps.bbox)):
            out[f"{tag}_{k}"] = np.asarray(v)
        out[f"{tag}_cam"] = np.concatenate([[cam.fx, cam.fy, cam.cx, cam.cy, cam.width, cam.height],
                                            cam.rotation.reshape(-1), cam.translation])

    # (a) the reference tests' random scene (tests/test_renderer.py:76-86)
    rng = np.random.default_rng(0)
    n = 30
    pos = rng.uniform([-0.6, -0.6, 0.8], [0.6, 0.6, 3.0], (n, 3))
    col = rng.uniform(0, 1, (n, 3))
    opa = rng.uniform(0.2, 1.0, n)
    scl = np.repeat(rng.uniform(0.02, 0.15, n)[:, None], 3, axis=1)
    rot = np.tile([1.0, 0.0, 0.0, 0.0], (n, 1))
    add("a", pos, scl, rot, opa, rgb_to_sh0(col), Camera(fx=64, fy=64, cx=31.5, cy=31.5, width=64, height=64))
    # (b) anisotropic, rotated primitives under a looking_at camera
    rng = np.random.default_rng(5)
    n = 400
    pos = rng.uniform([-3, -3, -0.5], [3, 3, 1.5], (n, 3))
    pos[:5] = [[0, -8, 1], [0, 30, 1], [40, 0, 0], [0.5, 0.5, 0.5], [0.5, 0.5, 0.5]]  # behind, far, off, ties
    scl = rng.uniform(0.01, 0.4, (n, 3))
    rot = rng.normal(size=(n, 4))
    opa = rng.uniform(0.05, 1.0, n)
    opa[5:10] = 0.5 / 255.0                                   # below the skip threshold
    sh0 = rgb_to_sh0(rng.uniform(0, 1, (n, 3)))
    cam = Camera.looking_at((0.3, -6.0, 2.0), (0.0, 0.0, 0.3), fx=80.0, fy=80.0, cx=47.5, cy=35.5,
                            width=96, height=72)
    add("b", pos, scl, rot, opa, sh0, cam)
    # (c) the Gaussian map of the scan replay fixture, seen by its camera
    sf = np.load(os.path.join(HERE, "scan_frames.npz"))
    g = {k: np.concatenate([sf[f"f{f}_g_{k}"] for f in range(3)])
         for k in ("positions", "scales", "rotations", "opacities", "colors")}
    fx, fy, cx, cy, w, h = sf["camera_intrinsics"]
    cam = Camera(fx=fx, fy=fy, cx=cx, cy=cy, width=int(w), height=int(h), rotation=sf["f2_R"],
                 translation=sf["f2_t"])
    add("c", g["positions"], g["scales"], g["rotations"], g["opacities"], g["colors"], cam)
    np.savez_compressed(os.path.join(HERE, "render.npz"), **out)


if __name__ == "__main__":
    if len(sys.argv) > 1:
        for name in sys.argv[1:]:
            globals()[name]()
        sys.exit(0)
    ply_fixture()
    gpr_fixture()
    keys_fixture()
    axis_fixture()
    grids_fixture()
    subgrid_fixture()
    scan_fixture()
    render_fixture()
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)))
