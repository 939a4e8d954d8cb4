"""Deterministic synthetic LiDAR workloads for tests and the benchmark.

Bench/test tooling only — not on the product path.  A fresh NumPy generator
for the five BASELINE.json configurations as SURVEY.md §8(d) restates them:

  1. one 32-beam spinning scan of an outdoor scene (ground + boxes + spheres),
     ~60k rays, 0.5 m voxels;
  2. a trajectory of such scans, pose advancing 1 m per scan;
  3. a Livox-style rosette scan (uneven density, heavy-tailed voxel counts);
  4. a ~1M-voxel map of planar patches with a heavy-tailed points-per-voxel
     histogram, shuffled into scan order;
  5. the (n_s, n_r) sweep reuses config 1.

The surface/ray model follows the reference's scene module in spirit
(`/root/reference/pkg/src/voxsplat/scene.py:69-269`: analytic planes, boxes
and spheres, line-scan and rosette patterns, range noise along the ray) but
is written independently; exact reproduction of the reference scans is not
needed because every parity check feeds the SAME generated arrays to the
oracle and to the CUDA path (and the golden fixtures store their inputs).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np


# ---------------------------------------------------------------------------
# camera pose helpers
# ---------------------------------------------------------------------------

def look_at(eye, target, up=(0.0, 0.0, 1.0)):
    """Camera-from-world rotation: +z forward, +x right, +y down."""
    eye = np.asarray(eye, dtype=np.float64)
    fwd = np.asarray(target, dtype=np.float64) - eye
    fwd /= np.linalg.norm(fwd)
    right = np.cross(fwd, np.asarray(up, dtype=np.float64))
    right /= np.linalg.norm(right)
    down = np.cross(fwd, right)
    R = np.stack([right, down, fwd])          # rows = camera axes in world
    t = -R @ eye
    return R, t


@dataclass
class Pinhole:
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int
    R: np.ndarray
    t: np.ndarray

    @property
    def center(self):
        return -self.R.T @ self.t


# ---------------------------------------------------------------------------
# analytic surfaces (vectorised ray casting)
# ---------------------------------------------------------------------------

def _hit_plane(o, d, normal, offset):
    n = np.asarray(normal, dtype=np.float64)
    n = n / np.linalg.norm(n)
    den = d @ n
    with np.errstate(divide="ignore", invalid="ignore"):
        t = (offset - o @ n) / den
    t[np.abs(den) < 1e-15] = np.inf
    t[~(t > 1e-9)] = np.inf
    return t


def _hit_box(o, d, lo, hi):
    with np.errstate(divide="ignore", invalid="ignore"):
        inv = 1.0 / d
        a = (lo - o) * inv
        b = (hi - o) * inv
    tmin = np.nanmax(np.minimum(a, b), axis=1)
    tmax = np.nanmin(np.maximum(a, b), axis=1)
    t = np.where(tmin > 1e-9, tmin, tmax)
    ok = (tmin <= tmax) & (t > 1e-9)
    return np.where(ok, t, np.inf)


def _hit_sphere(o, d, c, r):
    oc = o - c
    b = 2.0 * np.einsum("ij,ij->i", oc, d)
    cc = np.einsum("ij,ij->i", oc, oc) - r * r
    disc = b * b - 4.0 * cc
    sq = np.sqrt(np.clip(disc, 0.0, None))
    t1 = (-b - sq) / 2.0
    t2 = (-b + sq) / 2.0
    t = np.where(t1 > 1e-9, t1, t2)
    return np.where((disc >= 0) & (t > 1e-9), t, np.inf)


@dataclass
class OutdoorScene:
    """Ground plane + box 'buildings' + sphere 'trees'."""

    boxes: np.ndarray     # (B, 2, 3) lo/hi
    spheres: np.ndarray   # (S, 4) cx cy cz r
    box_rgb: np.ndarray   # (B, 3)
    sphere_rgb: np.ndarray

    @classmethod
    def make(cls, seed=0, n_boxes=30, n_spheres=30, half=40.0):
        rng = np.random.default_rng(seed)
        boxes = []
        while len(boxes) < n_boxes:
            cxy = rng.uniform(-half, half, 2)
            if np.linalg.norm(cxy) < 6.0:
                continue
            fp = rng.uniform(3.0, 10.0, 2)
            h = rng.uniform(3.0, 15.0)
            lo = np.array([cxy[0] - fp[0] / 2, cxy[1] - fp[1] / 2, 0.0])
            hi = np.array([cxy[0] + fp[0] / 2, cxy[1] + fp[1] / 2, h])
            boxes.append(np.stack([lo, hi]))
        sph = []
        while len(sph) < n_spheres:
            cxy = rng.uniform(-half, half, 2)
            if np.linalg.norm(cxy) < 5.0:
                continue
            r = rng.uniform(1.0, 2.5)
            sph.append([cxy[0], cxy[1], 3.0, r])
        return cls(np.asarray(boxes), np.asarray(sph),
                   rng.uniform(0.2, 0.9, (n_boxes, 3)),
                   rng.uniform(0.1, 0.7, (n_spheres, 3)))

    def cast(self, o, d):
        """Nearest hit distance and RGB per ray (inf / 0 on miss)."""
        best = _hit_plane(o, d, (0.0, 0.0, 1.0), 0.0)
        rgb = np.zeros((len(d), 3))
        hitp = o + np.where(np.isfinite(best), best, 0.0)[:, None] * d
        chk = (np.floor(hitp[:, 0]) + np.floor(hitp[:, 1])).astype(np.int64) % 2 == 0
        rgb[:] = np.where(chk[:, None], 0.85, 0.15)
        for i, (lo, hi) in enumerate(self.boxes):
            t = _hit_box(o, d, lo, hi)
            c = t < best
            best[c] = t[c]
            rgb[c] = self.box_rgb[i]
        for i, s in enumerate(self.spheres):
            t = _hit_sphere(o, d, s[:3], s[3])
            c = t < best
            best[c] = t[c]
            rgb[c] = self.sphere_rgb[i]
        return best, rgb


def _dirs(az, el):
    ce = np.cos(el)
    return np.stack([ce * np.sin(az), np.sin(el), ce * np.cos(az)], axis=1)


def lidar_dirs(pattern, rays, rng, fov_az, fov_el, rows=32):
    if pattern == "line-scan":
        rows = max(2, rows)
        cols = max(2, rays // rows)
        el = np.linspace(-fov_el / 2, fov_el / 2, rows)
        az = np.linspace(-fov_az / 2, fov_az / 2, cols)
        A, E = np.meshgrid(az, el)
        A = A.ravel() + rng.uniform(-0.5, 0.5) * (az[1] - az[0])
        return _dirs(A, E.ravel())
    if pattern == "rosette":
        t = np.arange(rays) / rays
        ph = rng.uniform(0.0, 2 * np.pi)
        az = 0.5 * fov_az * np.sin(2 * np.pi * 13.0 * t + ph)
        el = 0.5 * fov_el * np.sin(2 * np.pi * 13.0 * (1 + math.sqrt(5)) / 2 * t)
        return _dirs(az, el)
    if pattern == "uniform":
        return _dirs(rng.uniform(-fov_az / 2, fov_az / 2, rays),
                     rng.uniform(-fov_el / 2, fov_el / 2, rays))
    raise ValueError(pattern)


def scan(scene: OutdoorScene, eye, target, seed, frame, pattern="line-scan",
         rays=60000, rows=32, fov_az=0.999 * 2 * math.pi,
         fov_el=math.radians(40.0), noise=0.01):
    """(positions (N,3) f64, colors (N,3) f64) of one simulated scan."""
    rng = np.random.default_rng([seed, frame])
    R, t = look_at(eye, target)
    d = lidar_dirs(pattern, rays, rng, fov_az, fov_el, rows) @ R
    o = np.broadcast_to(np.asarray(eye, dtype=np.float64), d.shape)
    dist, rgb = scene.cast(o, d)
    hit = np.isfinite(dist)
    dist, rgb, d = dist[hit], rgb[hit], d[hit]
    if noise > 0:
        dist = dist + rng.normal(0.0, noise, len(dist))
    pts = np.asarray(eye, dtype=np.float64) + dist[:, None] * d
    return np.ascontiguousarray(pts), np.ascontiguousarray(np.clip(rgb, 0, 1))


def config1_scan(seed=0, frame=0, rays=60000):
    """Config 1: 32-beam spinning scan, sensor at 1.8 m looking along +x."""
    sc = OutdoorScene.make(seed)
    x = float(frame)
    return scan(sc, (x, 0.0, 1.8), (x + 10.0, 0.0, 1.8), seed, frame, rays=rays)


def config3_scan(seed=0, frame=0, rays=60000):
    """Config 3: Livox-style rosette, 70.4° x 77.2° field of view."""
    sc = OutdoorScene.make(seed)
    x = float(frame)
    return scan(sc, (x, 0.0, 1.8), (x + 10.0, 0.0, 1.8), seed, frame,
                pattern="rosette", rays=rays, fov_az=math.radians(70.4),
                fov_el=math.radians(77.2))


def camera_for(frame=0, width=640, height=480, f=400.0):
    x = float(frame)
    R, t = look_at((x, 0.0, 1.8), (x + 10.0, 0.0, 1.8))
    return Pinhole(f, f, (width - 1) / 2, (height - 1) / 2, width, height, R, t)


def render_image(scene: OutdoorScene, cam: Pinhole):
    """Ray-cast ground-truth RGB image (H, W, 3) f64 for colour sampling."""
    uu, vv = np.meshgrid(np.arange(cam.width, dtype=np.float64),
                         np.arange(cam.height, dtype=np.float64))
    dc = np.stack([(uu - cam.cx) / cam.fx, (vv - cam.cy) / cam.fy,
                   np.ones_like(uu)], axis=-1).reshape(-1, 3)
    d = dc @ cam.R
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    o = np.broadcast_to(cam.center, d.shape)
    dist, rgb = scene.cast(o, d)
    rgb[~np.isfinite(dist)] = 0.0
    return np.ascontiguousarray(rgb.reshape(cam.height, cam.width, 3))


# ---------------------------------------------------------------------------
# config 4: ~1M-voxel planar map
# ---------------------------------------------------------------------------

# points-per-voxel histogram of the config-1 scan at 0.5 m
N_BINS = ((10, 16), (16, 32), (32, 64), (64, 128), (128, 160))
N_PROBS = (0.56, 0.29, 0.06, 0.085, 0.005)
# ... and of the Livox-style rosette scan (config 3, the tail variant of config
# 4): [10,16,32,64,128,256,512,743) = [144,170,85,39,26,10,12] of 486 solvable
# voxels, max n 742
TAIL_BINS = ((10, 16), (16, 32), (32, 64), (64, 128), (128, 256), (256, 512), (512, 743))
TAIL_PROBS = (144, 170, 85, 39, 26, 10, 12)


def planar_map(n_voxels=1_000_000, voxel_size=0.5, seed=0, shuffle=True,
               bins=N_BINS, probs=N_PROBS, noise=0.01, key_offset=(0, 0, 0)):
    """(positions, colors, counts, keys, owner) for a grid of planar voxel patches.

    Voxels are the first ``n_voxels`` cells of a square ground lattice (plus
    ``key_offset``); each holds n points (n from the histogram) on a gently
    tilted plane through the voxel centre with N(0, noise²) scatter, clipped
    inside the voxel.  Points are shuffled into a random scan order so the
    hashing stage sees no locality.
    """
    rng = np.random.default_rng(seed)
    side = int(math.ceil(math.sqrt(n_voxels)))
    v = np.arange(n_voxels)
    keys = np.stack([v % side, v // side, np.zeros_like(v)], axis=1).astype(np.int64)
    keys += np.asarray(key_offset, dtype=np.int64)
    b = rng.choice(len(bins), size=n_voxels, p=np.asarray(probs) / sum(probs))
    lo_n = np.asarray([x[0] for x in bins])[b]
    hi_n = np.asarray([x[1] for x in bins])[b]
    counts = rng.integers(lo_n, hi_n)
    owner = np.repeat(v, counts)
    total = len(owner)
    lo = keys[owner].astype(np.float64) * voxel_size
    m = 0.02 * voxel_size
    uv = rng.uniform(m, voxel_size - m, (total, 2))
    slope = rng.uniform(-0.3, 0.3, (n_voxels, 2))
    dz = (slope[owner, 0] * (uv[:, 0] - voxel_size / 2)
          + slope[owner, 1] * (uv[:, 1] - voxel_size / 2)
          + rng.normal(0.0, noise, total))
    z = np.clip(voxel_size / 2 + dz, m, voxel_size - m)
    pos = lo + np.column_stack([uv, z])
    col = rng.uniform(0.0, 1.0, (total, 3))
    if shuffle:
        perm = rng.permutation(total)
        pos, col, owner = pos[perm], col[perm], owner[perm]
    return (np.ascontiguousarray(pos), np.ascontiguousarray(col), counts, keys, owner)
