"""CPU oracle for the voxel-GPR hot path — TEST INFRASTRUCTURE, NOT PRODUCT.

A NumPy/SciPy restatement of the reference `voxsplat` mapping hot path
(`/root/reference/pkg/src/voxsplat/`: voxel_map.py, gpr.py, splat_init.py,
camera.py).  Only `tests/`, `__graft_entry__.smoke()` and the `cpu_baseline` /
`--impl reference` legs of `bench.py` may import this module, and only as the
checker (or as the timed CPU baseline).  The product package
`paper_2410_17084_b200` never imports it and has no CPU fallback.

Parity pinning: every function here is checked against golden vectors produced
by the real reference (`tests/golden/make_golden.py`, run in the build
container where `/root/reference` is importable) in
`tests/test_oracle_golden.py`.  Parity is therefore PINNED, not unpinned.

The linear algebra runs through the same third-party routines the reference
uses: `scipy.linalg.cho_factor/cho_solve` (LAPACK dpotrf/dpotrs) and
`numpy.linalg.eigh` (LAPACK dsyevd).  The data layout is deliberately
different from the reference: the map is a struct of plain dicts of arrays and
the functions are free functions, so the oracle shares no code with either the
reference or the product.

One deliberate algorithmic difference: the reference groups a frame's points
with an O(touched x points) mask loop (voxel_map.py:328-341); the oracle uses a
stable argsort, which yields the identical first-touch order and identical
per-voxel point order in O(points log points).  As a CPU baseline this makes
the oracle FASTER than the reference, i.e. the reported GPU/CPU ratio is
conservative.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
from scipy.linalg import LinAlgError, cho_factor, cho_solve

UNREADY, READY, ACTIVE, CONVERGED = 0, 1, 2, 3
STATE_NAMES = ("UNREADY", "READY", "ACTIVE", "CONVERGED")

# value axis -> (first parameter axis, second parameter axis); gpr.py:36
PARAM_AXES = ((1, 2), (2, 0), (0, 1))
SH0 = 0.28209479177          # splat_init.py:22
IDENTITY_Q = np.array([1.0, 0.0, 0.0, 0.0])  # geometry.py:10

OK, DEGENERATE, CHOL_FAIL = 0, 1, 2


class OracleError(Exception):
    pass


# ---------------------------------------------------------------------------
# H1 — lattice keys (voxel_map.py:125-143)
# ---------------------------------------------------------------------------

def keys_of(positions, voxel_size):
    """floor(p / voxel_size) as int64; true IEEE division, no reciprocal."""
    if voxel_size <= 0:
        raise OracleError("voxel_size must be positive")
    p = np.asarray(positions, dtype=np.float64).reshape(-1, 3)
    if p.size and not np.isfinite(p).all():
        raise OracleError("cannot hash non-finite positions")
    return np.floor(p / voxel_size).astype(np.int64)


# ---------------------------------------------------------------------------
# H2/H3/G10 — the voxel map as plain arrays (voxel_map.py:173-355)
# ---------------------------------------------------------------------------

@dataclass
class OracleCell:
    raw_pos: np.ndarray
    raw_col: np.ndarray
    raw_noise: np.ndarray
    pseudo_pos: np.ndarray | None = None
    pseudo_col: np.ndarray | None = None
    pseudo_noise: np.ndarray | None = None
    state: int = UNREADY
    value_axis: int | None = None
    pred: dict | None = None   # last prediction: positions/colors/variances


@dataclass
class OracleMap:
    voxel_size: float
    sensor_var: float
    tau: int
    eta: float
    cells: dict = field(default_factory=dict)
    transitions: list = field(default_factory=list)   # (frame, key, old, new)
    solve_log: list = field(default_factory=list)     # (frame, key)
    frame: int = -1

    def store_frame(self, positions, colors):
        """First-touch-ordered keys of one frame; appends points per voxel.

        Restates voxel_map.py:313-342: the update order is the order of each
        key's first occurrence (np.unique return_index, then a stable argsort,
        lines 324-326); within a voxel the points keep frame order (boolean
        mask, line 330); noise is replaced by sensor_var (line 332); a cell
        becomes READY when its raw count reaches tau (339-340).
        """
        self.frame += 1
        pos = np.asarray(positions, dtype=np.float64).reshape(-1, 3)
        col = np.asarray(colors, dtype=np.float64).reshape(-1, 3)
        if len(pos) == 0:
            return []
        k = keys_of(pos, self.voxel_size)
        uniq, first, inverse = np.unique(k, axis=0, return_index=True,
                                         return_inverse=True)
        inverse = inverse.reshape(-1)
        rank_of = np.empty(len(uniq), dtype=np.int64)
        rank_of[np.argsort(first, kind="stable")] = np.arange(len(uniq))
        point_rank = rank_of[inverse]
        order = np.argsort(point_rank, kind="stable")   # groups, frame order kept
        counts = np.bincount(point_rank, minlength=len(uniq))
        starts = np.concatenate([[0], np.cumsum(counts)])
        by_rank = np.empty_like(uniq)
        by_rank[rank_of] = uniq
        touched = []
        for r in range(len(uniq)):
            key = tuple(int(v) for v in by_rank[r])
            idx = order[starts[r]:starts[r + 1]]
            sp, sc = pos[idx], col[idx]
            sn = np.full(len(idx), self.sensor_var)
            cell = self.cells.get(key)
            if cell is None:
                cell = OracleCell(sp, sc, sn)
                self.cells[key] = cell
            else:
                cell.raw_pos = np.concatenate([cell.raw_pos, sp])
                cell.raw_col = np.concatenate([cell.raw_col, sc])
                cell.raw_noise = np.concatenate([cell.raw_noise, sn])
            if cell.state == UNREADY and len(cell.raw_pos) >= self.tau:
                self.transitions.append((self.frame, key, UNREADY, READY))
                cell.state = READY
            touched.append(key)
        return touched

    def training(self, key):
        """raw ∪ pseudo (voxel_map.py:196-200)."""
        c = self.cells[key]
        if c.pseudo_pos is None:
            return c.raw_pos, c.raw_col, c.raw_noise
        return (np.concatenate([c.raw_pos, c.pseudo_pos]),
                np.concatenate([c.raw_col, c.pseudo_col]),
                np.concatenate([c.raw_noise, c.pseudo_noise]))

    def apply_prediction(self, key, pred):
        """voxel_map.py:242-261 and 344-355 (fold back, reclassify, log)."""
        c = self.cells[key]
        if c.state not in (READY, ACTIVE):
            raise OracleError(f"cell {key} cannot accept a solve")
        before = c.state
        c.pseudo_pos = pred["positions"]
        c.pseudo_col = pred["colors"]
        c.pseudo_noise = np.clip(pred["variances"], 0.0, None)
        c.pred = pred
        c.state = CONVERGED if float(pred["variances"].mean()) <= self.eta else ACTIVE
        self.solve_log.append((self.frame, key))
        for s in range(before + 1, c.state + 1):
            self.transitions.append((self.frame, key, s - 1, s))


# ---------------------------------------------------------------------------
# G1 — value-axis selection by PCA (gpr.py:57-86)
# ---------------------------------------------------------------------------

def select_axis(points):
    """(value_axis, f, x) or raises OracleError('degenerate')."""
    p = np.asarray(points, dtype=np.float64).reshape(-1, 3)
    if len(p) < 3:
        raise OracleError("degenerate: fewer than 3 points")
    d = p - p.mean(axis=0)
    cov = d.T @ d / len(p)
    w, v = np.linalg.eigh(cov)
    if w[2] <= 1e-18 or w[1] <= 1e-9 * w[2]:
        raise OracleError("degenerate: coincident or collinear")
    a = np.abs(v[:, 0])
    axis = 2 - int(np.argmax(a[::-1]))        # ties prefer z, then y, then x
    pa, pb = PARAM_AXES[axis]
    return axis, p[:, axis].copy(), np.stack([p[:, pa], p[:, pb]], axis=1)


def rebuild_points(axis, x, f):
    """Inverse split (gpr.py:89-97)."""
    pa, pb = PARAM_AXES[axis]
    out = np.empty((len(x), 3))
    out[:, axis] = f
    out[:, pa] = x[:, 0]
    out[:, pb] = x[:, 1]
    return out


# ---------------------------------------------------------------------------
# G3/G4 — query grid and SE kernel (gpr.py:104-130)
# ---------------------------------------------------------------------------

def mesh_grid(extent, n_s, n_r):
    (lo0, hi0), (lo1, hi1) = extent
    m = n_s * n_r
    i = np.arange(m)
    c0 = lo0 + (i + 0.5) * (hi0 - lo0) / m
    c1 = lo1 + (i + 0.5) * (hi1 - lo1) / m
    b = np.arange(m * m)
    sr, rem = np.divmod(b, n_s * n_r * n_r)
    sc, rem = np.divmod(rem, n_r * n_r)
    fr, fc = np.divmod(rem, n_r)
    return np.stack([c0[sr * n_r + fr], c1[sc * n_r + fc]], axis=1)


def se_kernel(xa, xb, lam):
    xa = np.asarray(xa, dtype=np.float64).reshape(-1, 2)
    xb = np.asarray(xb, dtype=np.float64).reshape(-1, 2)
    d2 = ((xa[:, None, :] - xb[None, :, :]) ** 2).sum(axis=2)
    return np.exp(-lam * d2)


def matern_kernel(xa, xb, lam, nu):
    """Matérn-nu (nu in {1.5, 2.5}) with unit amplitude, length 1/sqrt(lam).

    North-star extension (no reference oracle, parity unpinned): r = sqrt(lam
    d2); nu=1.5: (1+√3 r)e^{-√3 r}; nu=2.5: (1+√5 r+5r²/3)e^{-√5 r}.
    k(q, q) = 1, which the posterior-variance shortcut relies on.
    """
    xa = np.asarray(xa, dtype=np.float64).reshape(-1, 2)
    xb = np.asarray(xb, dtype=np.float64).reshape(-1, 2)
    d2 = ((xa[:, None, :] - xb[None, :, :]) ** 2).sum(axis=2)
    r = np.sqrt(lam * d2)
    if nu == 1.5:
        s = math.sqrt(3.0) * r
        return (1.0 + s) * np.exp(-s)
    if nu == 2.5:
        s = math.sqrt(5.0) * r
        return (1.0 + s + s * s / 3.0) * np.exp(-s)
    raise OracleError("nu must be 1.5 or 2.5")


def kernel_fn(kind):
    if kind == "se":
        return se_kernel
    nu = {"matern32": 1.5, "matern52": 2.5}[kind]
    return lambda a, b, lam: matern_kernel(a, b, lam, nu)


# ---------------------------------------------------------------------------
# G6/G7 — posterior (gpr.py:173-255)
# ---------------------------------------------------------------------------

def posterior(x, f, noise, xs, lam, jitter=1e-10, full=False, kind="se"):
    """(mu, var_diag, full_or_None); raises OracleError('cholesky') on failure.

    Jitter is added only after a failed factorisation and the factorisation
    is retried exactly once (gpr.py:186-194).
    """
    kern = kernel_fn(kind)
    x = np.asarray(x, dtype=np.float64).reshape(-1, 2)
    xs = np.asarray(xs, dtype=np.float64).reshape(-1, 2)
    f = np.asarray(f, dtype=np.float64).reshape(-1)
    A = kern(x, x, lam) + np.diag(np.asarray(noise, dtype=np.float64).reshape(-1))
    try:
        fac = cho_factor(A, lower=True, check_finite=False)
    except LinAlgError:
        try:
            fac = cho_factor(A + jitter * np.eye(len(A)), lower=True,
                             check_finite=False)
        except LinAlgError as exc:
            raise OracleError("cholesky") from exc
    Ks = kern(x, xs, lam)
    mu = Ks.T @ cho_solve(fac, f, check_finite=False)
    V = cho_solve(fac, Ks, check_finite=False)
    var = 1.0 - np.einsum("ij,ij->j", Ks, V)
    Sfull = kern(xs, xs, lam) - Ks.T @ V if full else None
    return mu, var, Sfull


def dense_inverse_posterior(x, f, noise, xs, lam, jitter=1e-10):
    """Independent explicit-inverse route (mirrors tests/_oracles.py:10-35)."""
    x = np.asarray(x, dtype=np.float64).reshape(-1, 2)
    xs = np.asarray(xs, dtype=np.float64).reshape(-1, 2)
    A = se_kernel(x, x, lam) + np.diag(np.asarray(noise, dtype=np.float64))
    try:
        np.linalg.cholesky(A)
    except np.linalg.LinAlgError:
        A = A + jitter * np.eye(len(A))
    Ai = np.linalg.inv(A)
    Ks = se_kernel(x, xs, lam)
    S = se_kernel(xs, xs, lam) - Ks.T @ Ai @ Ks
    return Ks.T @ Ai @ np.asarray(f, dtype=np.float64), np.diag(S).copy(), S


# ---------------------------------------------------------------------------
# G9 — frame densification (gpr.py:262-311)
# ---------------------------------------------------------------------------

@dataclass
class DensifyConfig:
    n_s: int = 3
    n_r: int = 3
    kernel_lambda: float = 1.0
    jitter: float = 1e-10
    kernel: str = "se"


def densify(update_keys, omap: OracleMap, cfg: DensifyConfig):
    """Returns (predictions list of dicts in update order, skipped dict key->reason)."""
    preds, skipped = [], {}
    for key in update_keys:
        cell = omap.cells[key]
        if cell.state not in (READY, ACTIVE):
            continue
        tp, tc, tn = omap.training(key)
        try:
            axis, f, x = select_axis(tp)
        except OracleError:
            skipped[key] = DEGENERATE
            continue
        mean_f = f.mean()
        pa, pb = PARAM_AXES[axis]
        lo = np.array(key, dtype=np.float64) * omap.voxel_size
        hi = lo + omap.voxel_size
        xs = mesh_grid(((lo[pa], hi[pa]), (lo[pb], hi[pb])), cfg.n_s, cfg.n_r)
        try:
            mu, var, _ = posterior(x, f - mean_f, tn, xs, cfg.kernel_lambda,
                                   cfg.jitter, kind=cfg.kernel)
        except OracleError:
            skipped[key] = CHOL_FAIL
            continue
        pts = rebuild_points(axis, xs, mu + mean_f)
        d2 = ((xs[:, None, :] - x[None, :, :]) ** 2).sum(axis=2)
        src = np.argmin(d2, axis=1)
        pred = {"key": key, "positions": pts, "colors": tc[src],
                "variances": np.clip(var, 0.0, None), "value_axis": axis,
                "color_src": src}
        cell.value_axis = axis
        omap.apply_prediction(key, pred)
        preds.append(pred)
    return preds, skipped


# ---------------------------------------------------------------------------
# S1–S5 — Gaussian initialisation (splat_init.py:70-148, camera.py:53-76)
# ---------------------------------------------------------------------------

@dataclass
class OracleCamera:
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int
    R: np.ndarray
    t: np.ndarray

    def project(self, p):
        cam = np.atleast_2d(p) @ self.R.T + self.t
        z = cam[:, 2]
        with np.errstate(divide="ignore", invalid="ignore"):
            u = self.fx * cam[:, 0] / z + self.cx
            v = self.fy * cam[:, 1] / z + self.cy
        return np.stack([u, v], axis=1), z


def subgrid_moments(points, weights):
    """(position, Phi) — Eq. 6/7: weighted mean and weighted second moment."""
    wsum = weights.sum()
    p = (points * weights[:, None]).sum(axis=0) / wsum
    Q = points - p
    phi = (Q * weights[:, None]).T @ Q / wsum
    return p, phi


def gaussians_for_prediction(pred, camera: OracleCamera, image, n_s=3, n_r=3,
                             weight_floor=1e-8, scale_floor=1e-4, opacity=0.5):
    """n_s² Gaussian records of one prediction; dict of arrays."""
    block = n_r * n_r
    if len(pred["positions"]) != n_s * n_s * block:
        raise OracleError("prediction size mismatch")
    w_all = 1.0 / np.maximum(pred["variances"], weight_floor)
    out = {k: [] for k in ("position", "scale", "rotation", "opacity", "color",
                           "phi", "source_key")}
    for b in range(n_s * n_s):
        sl = slice(b * block, (b + 1) * block)
        P, w, C = pred["positions"][sl], w_all[sl], pred["colors"][sl]
        p, phi = subgrid_moments(P, w)
        scale = np.maximum(np.sqrt(np.clip(np.diag(phi), 0.0, None)), scale_floor)
        fallback = (C * w[:, None]).sum(axis=0) / w.sum()
        rgb = fallback
        uv, z = camera.project(p.reshape(1, 3))
        if z[0] > 0 and np.all(np.isfinite(uv[0])):
            iu = int(np.floor(uv[0, 0] + 0.5))
            iv = int(np.floor(uv[0, 1] + 0.5))
            if 0 <= iu < camera.width and 0 <= iv < camera.height:
                rgb = np.asarray(image[iv, iu], dtype=np.float64)
        out["position"].append(p)
        out["scale"].append(scale)
        out["rotation"].append(IDENTITY_Q.copy())
        out["opacity"].append(opacity)
        out["color"].append((rgb - 0.5) / SH0)
        out["phi"].append(phi)
        out["source_key"].append(pred["key"])
    return {k: np.asarray(v) for k, v in out.items()}


def eigen_scale_rotation(phi, scale_floor=1e-4):
    """North-star extension (parity unpinned): Φ = R diag(s²) Rᵀ.

    Returns (scale (3,), quaternion w-first (4,)) from numpy.linalg.eigh with
    a right-handed eigenbasis; used only to check the device 3x3 eigensolver
    through the reconstruction R S² Rᵀ ≈ Φ.
    """
    w, V = np.linalg.eigh(phi)
    if np.linalg.det(V) < 0:
        V[:, 0] = -V[:, 0]
    s = np.maximum(np.sqrt(np.clip(w, 0.0, None)), scale_floor)
    return s, V


# ---------------------------------------------------------------------------
# Whole ingest (pipeline.py:139-187 restricted to the mapping hot path)
# ---------------------------------------------------------------------------

def ingest(omap: OracleMap, positions, colors, cfg: DensifyConfig,
           camera=None, image=None, splat=None):
    """store -> densify -> init for first solves; returns a summary dict."""
    update = omap.store_frame(positions, colors)
    first = {k for k in update if omap.cells[k].state == READY}
    preds, skipped = densify(update, omap, cfg)
    gauss = []
    if camera is not None:
        splat = splat or {}
        for p in preds:
            if p["key"] in first:
                gauss.append(gaussians_for_prediction(
                    omap.cells[p["key"]].pred, camera, image, cfg.n_s, cfg.n_r,
                    **splat))
    return {"update": update, "predictions": preds, "skipped": skipped,
            "gaussians": gauss}


class OraclePipeline:
    """pipeline.py:139-171 with the expansion threshold: first solves queue in
    `pending` (update order, pipeline.py:154-156) and are expanded — from their
    CURRENT prediction (`cell.last_prediction`, a re-fit may have replaced the
    first one) with the expanding frame's camera and image — once at least
    `threshold` voxels are pending (pipeline.py:157-171)."""

    def __init__(self, omap: OracleMap, cfg: DensifyConfig, threshold: int = 1):
        self.omap, self.cfg, self.threshold = omap, cfg, int(threshold)
        self.pending = []

    def ingest(self, positions, colors, camera, image):
        omap = self.omap
        update = omap.store_frame(positions, colors)
        first = {k for k in update if omap.cells[k].state == READY}
        preds, skipped = densify(update, omap, self.cfg)
        self.pending.extend(p["key"] for p in preds if p["key"] in first)
        gauss = []
        if self.pending and len(self.pending) >= self.threshold:
            for key in self.pending:
                gauss.append(gaussians_for_prediction(omap.cells[key].pred, camera, image,
                                                      self.cfg.n_s, self.cfg.n_r))
            self.pending = []
        return {"update": update, "predictions": preds, "skipped": skipped, "gaussians": gauss,
                "first": first}


# ---------------------------------------------------------------------------
# Forward splat renderer (renderer.py:90-207) — restated per primitive in a
# plain loop over pixels of its bbox rows (no patch broadcasting), checked
# against the reference's own outputs (tests/golden/render.npz).
# ---------------------------------------------------------------------------
R_ALPHA_CEILING, R_ALPHA_SKIP, R_T_EPS = 0.99, 1.0 / 255.0, 1e-4      # renderer.py:27-29
R_DILATION, R_SIGMAS = 0.3, 3.0                                       # renderer.py:30-31


def quat_rotation(q):
    """Rotation of a w-first quaternion, normalised first (geometry.py:34-48)."""
    w, x, y, z = np.asarray(q, dtype=float) / np.linalg.norm(q)
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                     [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                     [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])


def project_splats(pos, scl, rot, cam, near=0.01):
    """Per-primitive projection (renderer.py:90-137): mean2d, cov2d, depth,
    radius, valid, bbox — one primitive at a time."""
    fx, fy, cx, cy, W, H = cam["fx"], cam["fy"], cam["cx"], cam["cy"], cam["width"], cam["height"]
    Rc, t = np.asarray(cam["R"], dtype=float), np.asarray(cam["t"], dtype=float)
    n = len(pos)
    out = dict(mean2d=np.zeros((n, 2)), cov2d=np.zeros((n, 2, 2)), depth=np.zeros(n),
               radius=np.zeros(n), valid=np.zeros(n, dtype=bool), bbox=np.zeros((n, 4), np.int64))
    for i in range(n):
        pc = Rc @ np.asarray(pos[i], dtype=float) + t
        x, y, z = pc
        ok = z > near
        zs = z if ok else 1.0
        u, v = fx * x / zs + cx, fy * y / zs + cy
        G = quat_rotation(rot[i])
        phi = G @ np.diag(np.asarray(scl[i], dtype=float) ** 2) @ G.T
        M = Rc @ phi @ Rc.T
        J = np.array([[fx / zs, 0.0, -fx * x / zs ** 2], [0.0, fy / zs, -fy * y / zs ** 2]])
        c2 = J @ M @ J.T + R_DILATION * np.eye(2)
        c2 = 0.5 * (c2 + c2.T)
        a, b, c = c2[0, 0], c2[0, 1], c2[1, 1]
        lam = 0.5 * (a + c) + math.sqrt(max((0.5 * (a - c)) ** 2 + b * b, 0.0))
        rad = R_SIGMAS * math.sqrt(max(lam, 0.0))
        ok = ok and u + rad >= 0 and u - rad <= W - 1 and v + rad >= 0 and v - rad <= H - 1
        ok = ok and math.isfinite(u) and math.isfinite(v)
        x0 = int(min(max(math.ceil(u - rad), 0), W)) if math.isfinite(u) else 0
        x1 = int(min(max(math.floor(u + rad) + 1, 0), W)) if math.isfinite(u) else 0
        y0 = int(min(max(math.ceil(v - rad), 0), H)) if math.isfinite(v) else 0
        y1 = int(min(max(math.floor(v + rad) + 1, 0), H)) if math.isfinite(v) else 0
        ok = ok and x1 > x0 and y1 > y0
        out["mean2d"][i] = (u, v)
        out["cov2d"][i] = c2
        out["depth"][i] = z
        out["radius"][i] = rad
        out["valid"][i] = ok
        if ok:
            out["bbox"][i] = (x0, x1, y0, y1)
    return out


def render_splats(pos, scl, rot, opacity, sh0, cam, near=0.01):
    """Front-to-back blending (renderer.py:176-207): colour (H,W,3), depth, silhouette."""
    pr = project_splats(pos, scl, rot, cam, near)
    W, H = cam["width"], cam["height"]
    color, depth, sil = np.zeros((H, W, 3)), np.zeros((H, W)), np.zeros((H, W))
    T = np.ones((H, W))
    rgb = np.asarray(sh0, dtype=float) * 0.28209479177 + 0.5
    idx = np.flatnonzero(pr["valid"])
    for i in idx[np.argsort(pr["depth"][idx], kind="stable")]:
        x0, x1, y0, y1 = pr["bbox"][i]
        m0, m1 = pr["mean2d"][i]
        a, b, c = pr["cov2d"][i][0, 0], pr["cov2d"][i][0, 1], pr["cov2d"][i][1, 1]
        det = a * c - b * b
        dx = np.arange(x0, x1, dtype=float) - m0
        for py in range(y0, y1):
            dy = float(py) - m1
            power = -0.5 * (c * dx ** 2 - 2.0 * b * dx * dy + a * dy ** 2) / det
            al = np.minimum(opacity[i] * np.exp(power), R_ALPHA_CEILING)
            al[al < R_ALPHA_SKIP] = 0.0
            Tr = T[py, x0:x1]
            live = Tr >= R_T_EPS
            w = np.where(live, al * Tr, 0.0)
            color[py, x0:x1] += w[:, None] * rgb[i]
            depth[py, x0:x1] += w * pr["depth"][i]
            sil[py, x0:x1] += w
            T[py, x0:x1] = np.where(live, Tr * (1.0 - al), Tr)
    return color, depth, sil, pr
