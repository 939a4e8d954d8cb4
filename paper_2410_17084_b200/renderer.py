"""Forward splat renderer (mirror of voxsplat/renderer.py).

Same names, constants and outputs as the reference: `project_points`
(renderer.py:90-137) and `render` (renderer.py:184-207) run on the device
through `vx_project_points` / `vx_render` (csrc/vx_render.cu: projection
kernel, depth-ordered tile binning, one CTA per 16x16 tile blending front to
back).  `render` also accepts the engine's device records
(`MappingEngine.gaussians_device()` or `splat_init.GaussianRecords`), which
never leave HBM.  The per-splat helpers
the reference exposes for its own tests (`gaussian_patch`, `alpha_patch`,
`depth_order`) stay small NumPy functions over caller-held arrays, like the
reference's; the device path does not call them.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .camera import Camera
from .splat_init import GaussianMap, GaussianPrimitive, GaussianRecords

ALPHA_CEILING = 0.99
ALPHA_SKIP = 1.0 / 255.0
TRANSMITTANCE_EPS = 1e-4
COV_DILATION = 0.3          # pixels^2, added to the 2D covariance diagonal
RADIUS_SIGMAS = 3.0
DEFAULT_NEAR = 0.01


@dataclass
class SplatProjection:
    """One primitive seen by one camera."""

    mean2d: np.ndarray
    cov2d: np.ndarray
    depth: float
    radius: float


@dataclass
class RenderBuffers:
    """Rasterization output: color C, depth D and silhouette S images."""

    color: np.ndarray       # (H, W, 3)
    depth: np.ndarray       # (H, W) meters
    silhouette: np.ndarray  # (H, W) in [0, 1]


@dataclass
class ProjectionSet:
    """Vectorized projections of a whole map for one camera."""

    mean2d: np.ndarray   # (n, 2)
    cov2d: np.ndarray    # (n, 2, 2)
    depth: np.ndarray    # (n,)
    radius: np.ndarray   # (n,)
    valid: np.ndarray    # (n,) bool
    bbox: np.ndarray     # (n, 4) int: x0, x1, y0, y1 half-open pixel ranges

    def projection(self, i: int) -> SplatProjection | None:
        if not self.valid[i]:
            return None
        return SplatProjection(mean2d=self.mean2d[i].copy(), cov2d=self.cov2d[i].copy(),
                               depth=float(self.depth[i]), radius=float(self.radius[i]))


def _device_arrays(primitives):
    """(positions, scales, rotations, opacities, sh0, n) as device tensors."""
    if isinstance(primitives, GaussianRecords):
        n = primitives.count
        return (primitives.position[:n], primitives.scale[:n], primitives.rotation[:n],
                primitives.opacity[:n], primitives.color[:n], n)
    if isinstance(primitives, dict):             # MappingEngine.gaussians_device()
        p = primitives
        return (p["position"].contiguous(), p["scale"].contiguous(), p["rotation"].contiguous(),
                p["opacity"].contiguous(), p["color"].contiguous(), int(p["position"].shape[0]))
    if isinstance(primitives, GaussianMap):
        arrs = (primitives.positions, primitives.scales, primitives.rotations,
                primitives.opacities, primitives.colors)
    else:
        prims = list(primitives)
        if prims and not all(isinstance(p, GaussianPrimitive) for p in prims):
            raise TypeError("render expects GaussianPrimitive objects, a GaussianMap or records")
        if not prims:
            z = np.empty((0, 3))
            arrs = (z, z.copy(), np.empty((0, 4)), np.empty(0), z.copy())
        else:
            arrs = (np.stack([p.position for p in prims]), np.stack([p.scale for p in prims]),
                    np.stack([p.rotation for p in prims]),
                    np.array([p.opacity for p in prims], dtype=float),
                    np.stack([p.color for p in prims]))
    n = len(arrs[0])
    return tuple(N.to_device(np.asarray(a, dtype=float)) for a in arrs) + (n,)


def project_points(positions, scales, rotations, cam: Camera,
                   near: float = DEFAULT_NEAR) -> ProjectionSet:
    """Project every primitive on the device (renderer.py:90-137)."""
    import torch
    n = len(positions)
    if n == 0:
        return ProjectionSet(np.empty((0, 2)), np.empty((0, 2, 2)), np.empty(0), np.empty(0),
                             np.zeros(0, dtype=bool), np.zeros((0, 4), dtype=np.int64))
    dp, ds, dr = (N.to_device(np.asarray(a, dtype=float)) for a in (positions, scales, rotations))
    dev = dp.device
    mean2d = torch.empty((n, 2), dtype=torch.float64, device=dev)
    cov2d = torch.empty((n, 2, 2), dtype=torch.float64, device=dev)
    depth = torch.empty((n,), dtype=torch.float64, device=dev)
    radius = torch.empty((n,), dtype=torch.float64, device=dev)
    valid = torch.empty((n,), dtype=torch.uint8, device=dev)
    bbox = torch.empty((n, 4), dtype=torch.int64, device=dev)
    camc = N.camera_struct(cam)
    N.check(N.lib().vx_project_points(N.ptr(dp), N.ptr(ds), N.ptr(dr), n, C.byref(camc),
                                      float(near), N.ptr(mean2d), N.ptr(cov2d), N.ptr(depth),
                                      N.ptr(radius), N.ptr(valid), N.ptr(bbox), N.stream_ptr()),
            "vx_project_points")
    return ProjectionSet(mean2d=mean2d.cpu().numpy(), cov2d=cov2d.cpu().numpy(),
                         depth=depth.cpu().numpy(), radius=radius.cpu().numpy(),
                         valid=valid.cpu().numpy().astype(bool), bbox=bbox.cpu().numpy())


def project_gaussian(g: GaussianPrimitive, cam: Camera,
                     near: float = DEFAULT_NEAR) -> SplatProjection | None:
    """Scalar projection of one primitive; None when culled."""
    ps = project_points(g.position[None, :], g.scale[None, :], g.rotation[None, :], cam, near)
    return ps.projection(0)


def render_device(primitives, cam: Camera, near: float = DEFAULT_NEAR):
    """Render into device tensors (color (H,W,3), depth (H,W), silhouette (H,W))."""
    import torch
    dp, ds, dr, do, dc, n = _device_arrays(primitives)
    dev = N.device()
    H, W = cam.height, cam.width
    color = torch.empty((H, W, 3), dtype=torch.float64, device=dev)
    depth = torch.empty((H, W), dtype=torch.float64, device=dev)
    sil = torch.empty((H, W), dtype=torch.float64, device=dev)
    camc = N.camera_struct(cam)
    N.check(N.lib().vx_render(N.ptr(dp), N.ptr(ds), N.ptr(dr), N.ptr(do), N.ptr(dc), n,
                              C.byref(camc), float(near), N.ptr(color), N.ptr(depth), N.ptr(sil),
                              N.stream_ptr()), "vx_render")
    return color, depth, sil


def render(primitives, cam: Camera, near: float = DEFAULT_NEAR) -> RenderBuffers:
    """Rasterize a whole map into color, depth and silhouette buffers (renderer.py:184-207)."""
    color, depth, sil = render_device(primitives, cam, near)
    return RenderBuffers(color=color.cpu().numpy(), depth=depth.cpu().numpy(),
                         silhouette=sil.cpu().numpy())


# ---------------------------------------------------------------------------
# host helpers over caller-held arrays (the reference exposes them for tests)
# ---------------------------------------------------------------------------
def gaussian_patch(mean2d, cov2d, x0, x1, y0, y1) -> np.ndarray:
    """Raw Gaussian density exp(-0.5 d^T cov^-1 d) over a pixel rectangle."""
    xs = np.arange(x0, x1, dtype=float) - mean2d[0]
    ys = np.arange(y0, y1, dtype=float) - mean2d[1]
    a, b, c = cov2d[0, 0], cov2d[0, 1], cov2d[1, 1]
    det = a * c - b * b
    dx = xs[None, :]
    dy = ys[:, None]
    return np.exp(-0.5 * (c * dx ** 2 - 2.0 * b * dx * dy + a * dy ** 2) / det)


def alpha_patch(mean2d, cov2d, opacity, x0, x1, y0, y1) -> np.ndarray:
    """Blending alpha of one splat over a pixel rectangle (skip / ceiling applied)."""
    alpha = np.minimum(opacity * gaussian_patch(mean2d, cov2d, x0, x1, y0, y1), ALPHA_CEILING)
    alpha[alpha < ALPHA_SKIP] = 0.0
    return alpha


def depth_order(depth: np.ndarray, valid: np.ndarray) -> np.ndarray:
    """Front-to-back ordering of the valid indices, ties broken by index."""
    idx = np.flatnonzero(valid)
    return idx[np.argsort(depth[idx], kind="stable")]
