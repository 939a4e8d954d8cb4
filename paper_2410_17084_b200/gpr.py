"""Per-voxel GP regression on the device (mirror of voxsplat/gpr.py).

Public names and signatures follow `/root/reference/pkg/src/voxsplat/gpr.py`.
All arithmetic runs in libvoxgpr's FP64 sm_100a kernels:

  select_value_axis   -> vx_select_axis_batch (closed 3x3 Jacobi eigen, gpr.py:57-78)
  make_mesh_grid      -> vx_mesh_grid (bit-exact, gpr.py:104-120)
  kernel_matrix       -> vx_kernel_matrix (gpr.py:123-130)
  gpr_solve(_batch)   -> vx_gpr_solve_batch (Cholesky + jitter retry, gpr.py:173-255)
  densify_frame       -> vx_map_densify (fused axis/grid/solve/colour/lifecycle,
                         gpr.py:269-311)

`split_by_axis`, `assemble_points` and `voxel_parameter_extent` are index
re-arrangements of host arrays the caller already holds; the fused densify
kernel performs the same rearrangement on the device.
"""

from __future__ import annotations

import ctypes as C
import logging
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .errors import (DegenerateGeometryError, InputDomainError, NumericalDegeneracyError)
from .voxel_map import (FrameUpdateSet, VoxelKey, VoxelMap, VoxelPrediction, voxel_bounds)

log = logging.getLogger(__name__)

DEFAULT_JITTER = 1e-10
PARAMETER_AXES = {0: (1, 2), 1: (2, 0), 2: (0, 1)}


@dataclass
class AxisSelection:
    value_axis: int
    f: np.ndarray
    x: np.ndarray


def _axes_batch(point_sets) -> np.ndarray:
    """Value axis (or -1 when degenerate) of each (n,3) point set, on the device."""
    import torch
    lib = N.lib()
    sets = [np.asarray(p, dtype=float).reshape(-1, 3) for p in point_sets]
    off = np.concatenate([[0], np.cumsum([len(s) for s in sets])]).astype(np.int64)
    pts = np.concatenate(sets) if off[-1] else np.zeros((1, 3))
    dp, do = N.to_device(pts), N.to_device(off, dtype=np.int64)
    out = torch.empty(len(sets), dtype=torch.int8, device=dp.device)
    N.check(lib.vx_select_axis_batch(N.ptr(dp), N.ptr(do), len(sets), N.ptr(out), N.stream_ptr()))
    return out.cpu().numpy()


def select_value_axis(points: np.ndarray) -> AxisSelection:
    """Coordinate axis closest to the PCA normal (ties prefer z, then y, then x)."""
    pts = np.asarray(points, dtype=float).reshape(-1, 3)
    if len(pts) < 3:
        raise DegenerateGeometryError(f"need at least 3 points, got {len(pts)}")
    axis = int(_axes_batch([pts])[0])
    if axis < 0:
        raise DegenerateGeometryError("points are coincident or collinear")
    return split_by_axis(pts, axis)


def split_by_axis(points: np.ndarray, value_axis: int) -> AxisSelection:
    pa, pb = PARAMETER_AXES[value_axis]
    pts = np.asarray(points, dtype=float).reshape(-1, 3)
    return AxisSelection(value_axis=value_axis, f=pts[:, value_axis].copy(),
                         x=np.stack([pts[:, pa], pts[:, pb]], axis=1))


def assemble_points(value_axis: int, x: np.ndarray, f: np.ndarray) -> np.ndarray:
    pa, pb = PARAMETER_AXES[value_axis]
    x = np.asarray(x, dtype=float).reshape(-1, 2)
    out = np.empty((len(x), 3))
    out[:, value_axis] = np.asarray(f, dtype=float).reshape(-1)
    out[:, pa] = x[:, 0]
    out[:, pb] = x[:, 1]
    return out


def make_mesh_grid(extent, n_s: int, n_r: int) -> np.ndarray:
    """((n_s n_r)^2, 2) cell-centre grid, (subgrid row, subgrid col, fine row, fine col)."""
    if n_s < 1 or n_r < 1:
        raise InputDomainError("n_s and n_r must be at least 1")
    import torch
    lib = N.lib()
    (lo0, hi0), (lo1, hi1) = extent
    e = N.to_device(np.array([lo0, hi0, lo1, hi1], dtype=np.float64))
    m = (n_s * n_r) ** 2
    out = torch.empty((m, 2), dtype=torch.float64, device=e.device)
    N.check(lib.vx_mesh_grid(N.ptr(e), 1, int(n_s), int(n_r), N.ptr(out), N.stream_ptr()))
    return out.cpu().numpy()


def kernel_matrix(xa: np.ndarray, xb: np.ndarray, lam: float, kernel: str = "se") -> np.ndarray:
    """Entry (i, j) = k(xa_i, xb_j); SE = exp(-lam ||xa_i - xb_j||^2)."""
    if lam <= 0:
        raise InputDomainError("kernel constant must be positive")
    import torch
    lib = N.lib()
    xa = np.asarray(xa, dtype=float).reshape(-1, 2)
    xb = np.asarray(xb, dtype=float).reshape(-1, 2)
    if len(xa) == 0 or len(xb) == 0:
        return np.empty((len(xa), len(xb)))
    da, db = N.to_device(xa), N.to_device(xb)
    out = torch.empty((len(xa), len(xb)), dtype=torch.float64, device=da.device)
    N.check(lib.vx_kernel_matrix(N.ptr(da), len(xa), N.ptr(db), len(xb), float(lam),
                                 N.KERNELS[kernel], N.ptr(out), N.stream_ptr()))
    return out.cpu().numpy()


# ---------------------------------------------------------------------------
# Posterior solve (gpr.py:137-255)
# ---------------------------------------------------------------------------

@dataclass
class GprProblem:
    x: np.ndarray
    f: np.ndarray
    noise_diag: np.ndarray
    x_star: np.ndarray
    lam: float = 1.0

    def __post_init__(self):
        self.x = np.asarray(self.x, dtype=float).reshape(-1, 2)
        self.f = np.asarray(self.f, dtype=float).reshape(-1)
        self.noise_diag = np.asarray(self.noise_diag, dtype=float).reshape(-1)
        self.x_star = np.asarray(self.x_star, dtype=float).reshape(-1, 2)
        n = len(self.x)
        if n < 1:
            raise InputDomainError("need at least one training point")
        if len(self.f) != n or len(self.noise_diag) != n:
            raise InputDomainError("x, f and noise_diag must agree in length")
        if np.any(self.noise_diag < 0):
            raise InputDomainError("noise variances must be nonnegative")
        if self.lam <= 0:
            raise InputDomainError("kernel constant must be positive")
        if not (np.all(np.isfinite(self.x)) and np.all(np.isfinite(self.f))
                and np.all(np.isfinite(self.x_star))):
            raise InputDomainError("problem data must be finite")


@dataclass
class GprResult:
    mu_star: np.ndarray
    sigma_star_diag: np.ndarray
    sigma_star_full: np.ndarray | None = None


@dataclass
class GprBatchResult:
    results: list
    errors: list

    @property
    def ok(self) -> bool:
        return not self.errors


def _solve_packed(problems, return_full, jitter, kernel="se"):
    """One vx_gpr_solve_batch launch over all problems; returns (mu, var, full, status, offs)."""
    import torch
    lib = N.lib()
    P = len(problems)
    n = np.array([len(p.x) for p in problems], dtype=np.int64)
    m = np.array([len(p.x_star) for p in problems], dtype=np.int64)
    x_off = np.concatenate([[0], np.cumsum(n)]).astype(np.int64)
    q_off = np.concatenate([[0], np.cumsum(m)]).astype(np.int64)
    dev = N.device()
    t = {k: N.to_device(v) for k, v in (
        ("x", np.concatenate([p.x for p in problems])),
        ("f", np.concatenate([p.f for p in problems])),
        ("noise", np.concatenate([p.noise_diag for p in problems])),
        ("xs", np.concatenate([p.x_star for p in problems]) if q_off[-1] else np.zeros((1, 2))),
        ("lam", np.array([float(p.lam) for p in problems])))}
    dxo, dqo = N.to_device(x_off, np.int64), N.to_device(q_off, np.int64)
    mu = torch.empty(max(int(q_off[-1]), 1), dtype=torch.float64, device=dev)
    var = torch.empty_like(mu)
    status = torch.full((P,), 255, dtype=torch.uint8, device=dev)
    full = dfo = None
    f_off = None
    if return_full:
        f_off = np.concatenate([[0], np.cumsum(m * m)]).astype(np.int64)
        full = torch.empty(max(int(f_off[-1]), 1), dtype=torch.float64, device=dev)
        dfo = N.to_device(f_off, np.int64)
    b = N.VxGprBatch()
    b.num_problems = P
    b.d_x_off, b.d_q_off = N.ptr(dxo), N.ptr(dqo)
    b.d_x, b.d_f, b.d_noise, b.d_xs, b.d_lam = (N.ptr(t[k]) for k in ("x", "f", "noise", "xs", "lam"))
    b.jitter, b.kernel = float(jitter), N.KERNELS[kernel]
    b.max_n, b.max_m = int(n.max()), int(m.max()) if P else 0
    b.d_mu, b.d_var, b.d_status = N.ptr(mu), N.ptr(var), N.ptr(status)
    b.d_full, b.d_full_off = (N.ptr(full), N.ptr(dfo)) if return_full else (None, None)
    N.check(lib.vx_gpr_solve_batch(C.byref(b), N.stream_ptr()))
    return (mu.cpu().numpy(), var.cpu().numpy(), full.cpu().numpy() if return_full else None,
            status.cpu().numpy(), q_off, f_off)


def _chol_error(jitter):
    return NumericalDegeneracyError(
        f"kernel matrix not positive definite even with jitter {jitter}")


def gpr_solve(problem: GprProblem, return_full: bool = False,
              jitter: float = DEFAULT_JITTER) -> GprResult:
    """Posterior mean and variance at the query grid (one device launch)."""
    batch = gpr_solve_batch([problem], return_full=return_full, jitter=jitter)
    if batch.errors:
        raise batch.errors[0][1]
    return batch.results[0]


def gpr_solve_batch(problems: list, workers: int = 0, return_full: bool = False,
                    jitter: float = DEFAULT_JITTER, kernel: str = "se") -> GprBatchResult:
    """All problems in one batched FP64 launch; order preserved, per-index errors.

    `workers` is accepted for signature compatibility (gpr.py:224); the device
    batch is already parallel and its result does not depend on it.
    """
    P = len(problems)
    if P == 0:
        return GprBatchResult(results=[], errors=[])
    mu, var, full, status, q_off, f_off = _solve_packed(problems, return_full, jitter, kernel)
    results, errs = [None] * P, []
    for i in range(P):
        if status[i] == N.ST_OK:
            a, b = q_off[i], q_off[i + 1]
            S = None
            if return_full:
                mm = b - a
                S = full[f_off[i]:f_off[i] + mm * mm].reshape(mm, mm).copy()
            results[i] = GprResult(mu_star=mu[a:b].copy(), sigma_star_diag=var[a:b].copy(),
                                   sigma_star_full=S)
        else:
            errs.append((i, _chol_error(jitter)))
    return GprBatchResult(results=results, errors=errs)


# ---------------------------------------------------------------------------
# Frame densification (gpr.py:262-311)
# ---------------------------------------------------------------------------

def voxel_parameter_extent(key: VoxelKey, voxel_size: float, value_axis: int):
    bounds = voxel_bounds(key, voxel_size)
    pa, pb = PARAMETER_AXES[value_axis]
    return (bounds[0, pa], bounds[1, pa]), (bounds[0, pb], bounds[1, pb])


class DensifyResult:
    """Device-side outcome of one densify call (batched SoA entry point).

    `solved_voxels` (int32, update order), and the store views; predictions of
    voxel v live at prediction slot `pred_slot[v]` of `pred_xyz/rgb/var`.
    Valid until the map's next mutation.
    """

    def __init__(self, vmap: VoxelMap, info: N.VxDensifyInfo):
        self.info = info
        v = vmap.device_view()
        S, K = int(v.solve_candidates), int(v.solved)
        self.candidates = N.view_tensor(v.solve_voxels, (S,), np.int32)
        self.status = N.view_tensor(v.solve_status, (S,), np.uint8)
        self.before = N.view_tensor(v.solve_state_before, (S,), np.uint8)
        self.after = N.view_tensor(v.solve_state_after, (S,), np.uint8)
        self.solved_voxels = N.view_tensor(v.solved_voxels, (K,), np.int32)
        V, M = int(v.num_voxels), int(v.pred_points)
        self.keys = N.view_tensor(v.keys, (V, 3), np.int64)
        self.pred_slot = N.view_tensor(v.pred_slot, (V,), np.int32)
        self.M = M
        self._v = v

    def predictions(self):
        """(keys, positions, colors, variances) of the solved voxels, device tensors."""
        import torch
        K = len(self.solved_voxels)
        slots = self.pred_slot.index_select(0, self.solved_voxels.long()).long()
        nslots = int(slots.max().item()) + 1 if K else 0
        px = N.view_tensor(self._v.pred_xyz, (nslots, self.M, 3), np.float64)
        pc = N.view_tensor(self._v.pred_rgb, (nslots, self.M, 3), np.float64)
        pv = N.view_tensor(self._v.pred_var, (nslots, self.M), np.float64)
        if K == 0:
            e = torch.empty((0, self.M, 3), dtype=torch.float64, device=self.keys.device)
            return self.keys[:0], e, e.clone(), e[..., 0]
        return (self.keys.index_select(0, self.solved_voxels.long()), px.index_select(0, slots),
                pc.index_select(0, slots), pv.index_select(0, slots))


def densify_device(update_set, vmap: VoxelMap, config) -> DensifyResult:
    """densify_frame without host materialisation (for >=1M-voxel frames)."""
    vmap._h()
    vmap._configure_solver(config)
    vmap._select_frame(update_set)
    info = vmap._densify()
    res = DensifyResult(vmap, info)
    if vmap.record_log and info.solved:
        st = res.status.cpu().numpy()
        ok = np.nonzero(st == N.ST_OK)[0]
        vids = res.candidates.cpu().numpy()[ok]
        vmap._record_solves(int(res._v.frame_index), vids,
                            res.before.cpu().numpy()[ok], res.after.cpu().numpy()[ok])
    return res


def densify_frame(update_set: FrameUpdateSet, vmap: VoxelMap, config) -> list[VoxelPrediction]:
    """Solve every READY or ACTIVE voxel of the update set (gpr.py:269-311).

    One fused device pass; skipped voxels are logged with the reference's
    warning text and stay unsolved.  Returns host VoxelPrediction objects in
    update order.
    """
    res = densify_device(update_set, vmap, config)
    info = res.info
    if info.degenerate or info.chol_failed:
        st = res.status.cpu().numpy()
        bad = np.nonzero(st != N.ST_OK)[0]
        keys = vmap._keys_of(res.candidates.cpu().numpy()[bad])
        for k, s in zip(keys.tolist(), st[bad]):
            key = VoxelKey(*k)
            if s == N.ST_DEGENERATE:
                log.warning("voxel %s skipped: %s", key, "points are coincident or collinear")
            else:
                exc = _chol_error(config.jitter)
                exc.key = key
                log.warning("voxel %s skipped: %s", key, exc)
    if info.solved == 0:
        return []
    keys, pos, col, var = res.predictions()
    keys, pos, col, var = (t.cpu().numpy() for t in (keys, pos, col, var))
    return [VoxelPrediction(VoxelKey(*k), pos[i], col[i], var[i])
            for i, k in enumerate(keys.tolist())]
