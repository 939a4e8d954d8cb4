"""Gaussian initialisation on the device (mirror of voxsplat/splat_init.py).

Public names follow `/root/reference/pkg/src/voxsplat/splat_init.py:22-217`.
The moments, colour sampling and full per-voxel initialisation run in
libvoxgpr (`vx_subgrid_moments`, `vx_init_color`,
`vx_gaussians_from_predictions`, and the map-resident `vx_map_init_gaussians`).
`GaussianMap` is the host SoA container the reference exposes, grown by
capacity doubling instead of re-concatenating on every `extend` (the
reference's `extend` is O(map) per call, splat_init.py:169-184).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .camera import Camera
from .errors import ContractViolationError, InputDomainError
from .voxel_map import VoxelKey, VoxelPrediction

SH0_BASIS = 0.28209479177
DEFAULT_SCALE_FLOOR = 1e-4
DEFAULT_WEIGHT_FLOOR = 1e-8
IDENTITY_QUATERNION = np.array([1.0, 0.0, 0.0, 0.0])


def rgb_to_sh0(color: np.ndarray) -> np.ndarray:
    """RGB in [0, 1] to zero-degree SH coefficients: (c - 0.5) / basis."""
    return (np.asarray(color, dtype=float) - 0.5) / SH0_BASIS


def sh0_to_rgb(coeff: np.ndarray) -> np.ndarray:
    return np.asarray(coeff, dtype=float) * SH0_BASIS + 0.5


@dataclass
class GaussianPrimitive:
    position: np.ndarray
    scale: np.ndarray
    rotation: np.ndarray
    opacity: float
    color: np.ndarray
    source_key: VoxelKey | None = None

    def __post_init__(self):
        self.position = np.asarray(self.position, dtype=float).reshape(3)
        self.scale = np.asarray(self.scale, dtype=float).reshape(3)
        self.rotation = np.asarray(self.rotation, dtype=float).reshape(4)
        self.color = np.asarray(self.color, dtype=float).reshape(3)
        if abs(np.linalg.norm(self.rotation) - 1.0) > 1e-9:
            raise InputDomainError("rotation quaternion must be normalized")
        if np.any(self.scale <= 0):
            raise InputDomainError("scale components must be positive")
        if not 0.0 < self.opacity <= 1.0:
            raise InputDomainError("opacity must lie in (0, 1]")


@dataclass
class Subgrid:
    points: np.ndarray
    weights: np.ndarray
    colors: np.ndarray


def partition_subgrids(prediction: VoxelPrediction, n_s: int, n_r: int,
                       weight_floor: float = DEFAULT_WEIGHT_FLOOR) -> list[Subgrid]:
    """n_s^2 contiguous blocks of n_r^2 points; weights 1/max(var, floor) on the device."""
    block = n_r * n_r
    expected = n_s * n_s * block
    if len(prediction) != expected:
        raise ContractViolationError(
            f"prediction has {len(prediction)} points, expected {expected}")
    import torch
    N.lib()
    v = N.to_device(prediction.variances)
    weights = torch.reciprocal(torch.clamp_min(v, float(weight_floor))).cpu().numpy()
    return [Subgrid(points=prediction.positions[b * block:(b + 1) * block],
                    weights=weights[b * block:(b + 1) * block],
                    colors=prediction.colors[b * block:(b + 1) * block])
            for b in range(n_s * n_s)]


def _moments(points, weights, center=None):
    import torch
    lib = N.lib()
    P = np.asarray(points, dtype=float).reshape(1, -1, 3)
    W = np.asarray(weights, dtype=float).reshape(1, -1)
    dp, dw = N.to_device(P), N.to_device(W)
    dc = N.to_device(np.asarray(center, dtype=float).reshape(1, 3)) if center is not None else None
    pos = torch.empty((1, 3), dtype=torch.float64, device=dp.device)
    phi = torch.empty((1, 9), dtype=torch.float64, device=dp.device)
    N.check(lib.vx_subgrid_moments(N.ptr(dp), N.ptr(dw), 1, P.shape[1], N.ptr(dc), N.ptr(pos),
                                   N.ptr(phi), N.stream_ptr()))
    return pos.cpu().numpy()[0], phi.cpu().numpy()[0].reshape(3, 3)


def init_position(grid: Subgrid) -> np.ndarray:
    """Weighted mean of the subgrid points (Eq. 6)."""
    if np.asarray(grid.weights, dtype=float).sum() <= 0:
        raise InputDomainError("subgrid weights must sum to a positive value")
    return _moments(grid.points, grid.weights)[0]


def init_covariance(grid: Subgrid, position: np.ndarray,
                    scale_floor: float = DEFAULT_SCALE_FLOOR):
    """(Phi, scale, quaternion): weighted second moment about `position` (Eq. 7)."""
    _, phi = _moments(grid.points, grid.weights, center=position)
    scale = np.maximum(np.sqrt(np.clip(np.diag(phi), 0.0, None)), scale_floor)
    return phi, scale, IDENTITY_QUATERNION.copy()


def init_color(position: np.ndarray, camera: Camera, image: np.ndarray,
               fallback_rgb: np.ndarray) -> np.ndarray:
    """SH0 colour of the nearest pixel of the projected position, else the fallback."""
    import torch
    lib = N.lib()
    dp = N.to_device(np.asarray(position, dtype=float).reshape(1, 3))
    df = N.to_device(np.asarray(fallback_rgb, dtype=float).reshape(1, 3))
    di = N.to_device(image_for_camera(camera, np.asarray(image, dtype=float)))
    out = torch.empty((1, 3), dtype=torch.float64, device=dp.device)
    cam = N.camera_struct(camera)
    N.check(lib.vx_init_color(N.ptr(dp), N.ptr(df), 1, C.byref(cam), N.ptr(di), N.ptr(out),
                              N.stream_ptr()))
    return out.cpu().numpy()[0]


def _splat_cfg(config):
    return N.splat_struct(config.n_s, config.n_r, config.weight_floor, config.scale_floor,
                          config.initial_opacity, getattr(config, "rotation", "identity"))


class GaussianRecords:
    """Device SoA of Gaussian records (the VXSPLAT1 record split by field)."""

    def __init__(self, count: int):
        import torch
        dev = N.device()
        self.count = count
        self.position = torch.empty((count, 3), dtype=torch.float64, device=dev)
        self.scale = torch.empty((count, 3), dtype=torch.float64, device=dev)
        self.rotation = torch.empty((count, 4), dtype=torch.float64, device=dev)
        self.opacity = torch.empty((count,), dtype=torch.float64, device=dev)
        self.color = torch.empty((count, 3), dtype=torch.float64, device=dev)
        self.source_key = torch.empty((count, 3), dtype=torch.int64, device=dev)

    def out_struct(self, offset: int = 0) -> N.VxGaussianOut:
        o = N.VxGaussianOut()
        o.position = self.position.data_ptr() + offset * 24
        o.scale = self.scale.data_ptr() + offset * 24
        o.rotation = self.rotation.data_ptr() + offset * 32
        o.opacity = self.opacity.data_ptr() + offset * 8
        o.color = self.color.data_ptr() + offset * 24
        o.source_key = self.source_key.data_ptr() + offset * 24
        return o

    def to_host(self, count=None):
        n = self.count if count is None else count
        return {k: getattr(self, k)[:n].cpu().numpy() for k in
                ("position", "scale", "rotation", "opacity", "color", "source_key")}


def image_for_camera(camera, image):
    """The (height, width, 3) pixel block the device samples (init_color,
    splat_init.py:124-130 indexes image[iv, iu] for iv < height, iu < width).

    A larger image is cropped to that block (the same pixels the reference
    reads); one that does not cover the camera raises IndexError up front (the
    reference would raise it when a Gaussian projects onto a missing pixel),
    since the device reads the block without per-pixel bounds.  numpy arrays
    come back as contiguous float64, torch tensors as contiguous tensors."""
    H, W = int(camera.height), int(camera.width)
    shape = tuple(image.shape)
    if len(shape) != 3 or shape[0] < H or shape[1] < W or shape[2] < 3:
        raise IndexError(f"image of shape {shape} does not cover the camera's {H}x{W} pixels "
                         f"(expected ({H}, {W}, 3))")
    if shape != (H, W, 3):
        image = image[:H, :W, :3]
    if hasattr(image, "contiguous"):
        return image.contiguous()
    return np.ascontiguousarray(image, dtype=np.float64)


def init_gaussians_batch(predictions, camera: Camera, image: np.ndarray, config) -> dict:
    """Gaussian records of many predictions in one launch (host SoA dict)."""
    lib = N.lib()
    preds = list(predictions)
    if not preds:
        return {"position": np.empty((0, 3)), "scale": np.empty((0, 3)),
                "rotation": np.empty((0, 4)), "opacity": np.empty(0), "color": np.empty((0, 3)),
                "source_key": np.empty((0, 3), dtype=np.int64)}
    m = len(preds[0])
    expected = config.n_s * config.n_s * config.n_r * config.n_r
    for p in preds:
        if len(p) != expected:
            raise ContractViolationError(f"prediction has {len(p)} points, expected {expected}")
    dx = N.to_device(np.stack([p.positions for p in preds]))
    dc = N.to_device(np.stack([p.colors for p in preds]))
    dv = N.to_device(np.stack([p.variances for p in preds]))
    dk = N.to_device(np.array([tuple(p.key) for p in preds], dtype=np.int64), np.int64)
    di = N.to_device(image_for_camera(camera, np.asarray(image, dtype=float)))
    recs = GaussianRecords(len(preds) * config.n_s * config.n_s)
    cam, sc, out = N.camera_struct(camera), _splat_cfg(config), recs.out_struct()
    N.check(lib.vx_gaussians_from_predictions(N.ptr(dx), N.ptr(dc), N.ptr(dv), N.ptr(dk),
                                              len(preds), m, C.byref(cam), N.ptr(di),
                                              C.byref(sc), C.byref(out), N.stream_ptr()))
    return recs.to_host()


class _InitQueue:
    """Per-voxel `init_gaussians_for_voxel` calls, coalesced into one launch.

    The reference's callers initialise voxel by voxel inside a Python loop
    (pipeline.py:160-171) and only use the primitives through `len()` and
    `GaussianMap.extend`.  Each call therefore validates its prediction at once
    (same exception as the reference) but only queues it; the queue is solved
    in ONE `vx_gaussians_from_predictions` launch (one H2D of the stacked
    predictions and of the image, one D2H) when any primitive is read, when
    the camera / image / config of the calls changes, or when a GaussianMap
    holding them is read.
    """

    def __init__(self):
        self.ctx = None
        self.items = []          # (prediction, _LazyPrimitives)

    def add(self, prediction, camera, image, config):
        ctx = (id(camera), id(image), id(config))
        if self.ctx is not None and ctx != self.ctx:
            self.flush()
        if not self.items:
            self.ctx, self.refs = ctx, (camera, image, config)
        lazy = _LazyPrimitives(self, config.n_s * config.n_s)
        self.items.append((prediction, lazy))
        return lazy

    def flush(self):
        if not self.items:
            return
        items, (camera, image, config) = self.items, self.refs
        self.items, self.ctx, self.refs = [], None, None
        h = init_gaussians_batch([p for p, _ in items], camera, image, config)
        for i, (pred, lazy) in enumerate(items):
            lazy._batch = (h, i)          # records = rows [i k, (i + 1) k) of the batch
            lazy._key = pred.key


_QUEUE = _InitQueue()


class _LazyPrimitives(list):
    """The n_s^2 primitives of one queued voxel: a list that fills itself from
    the coalesced launch on first read (length known up front)."""

    __slots__ = ("_queue", "_n", "_batch", "_key")

    def __init__(self, queue, n):
        super().__init__()
        self._queue, self._n, self._batch, self._key = queue, n, None, None

    @property
    def _records(self):
        if self._batch is None:
            return None
        h, i = self._batch
        k = self._n
        return {name: v[i * k:(i + 1) * k] for name, v in h.items()}

    def _fill(self):
        if self._batch is None:
            self._queue.flush()
        if list.__len__(self) == 0 and self._n:
            h, key = self._records, VoxelKey(*(int(v) for v in self._key))
            list.extend(self, [GaussianPrimitive(position=h["position"][i], scale=h["scale"][i],
                                                 rotation=h["rotation"][i],
                                                 opacity=float(h["opacity"][i]),
                                                 color=h["color"][i], source_key=key)
                               for i in range(self._n)])

    def records(self) -> dict:
        if self._batch is None:
            self._queue.flush()
        return self._records

    def __len__(self):
        return self._n

    def __iter__(self):
        self._fill()
        return list.__iter__(self)

    def __getitem__(self, i):
        self._fill()
        return list.__getitem__(self, i)

    def __repr__(self):
        self._fill()
        return list.__repr__(self)

    def __eq__(self, other):
        self._fill()
        return list.__eq__(self, other)

    def __bool__(self):
        return self._n > 0


def init_gaussians_for_voxel(prediction: VoxelPrediction, camera: Camera, image: np.ndarray,
                             config) -> list[GaussianPrimitive]:
    """All n_s^2 primitives of a solved voxel (splat_init.py:134-148).

    Validated now; computed with every other queued voxel in one device
    launch when first read (`_InitQueue`)."""
    expected = config.n_s * config.n_s * config.n_r * config.n_r
    if len(prediction) != expected:
        raise ContractViolationError(
            f"prediction has {len(prediction)} points, expected {expected}")
    return _QUEUE.add(prediction, camera, image, config)


class GaussianMap:
    """Struct-of-arrays splat map with amortised O(1) appends."""

    _FIELDS = (("positions", 3, np.float64), ("scales", 3, np.float64),
               ("rotations", 4, np.float64), ("opacities", 0, np.float64),
               ("colors", 3, np.float64), ("source_keys", 3, np.int64))

    def __init__(self):
        self._n = 0
        self._buf = {name: np.empty((0, w) if w else (0,), dtype=dt)
                     for name, w, dt in self._FIELDS}
        self._lazy = []          # queued _LazyPrimitives (init_gaussians_for_voxel)

    def _settle(self):
        """Append the queued voxels' records (one launch for all of them); runs
        of voxels that are consecutive rows of one launch's batch are appended
        with one copy per field."""
        if self._lazy:
            pend, self._lazy = self._lazy, []
            for lz in pend:
                if lz._batch is None:
                    lz.records()                 # flushes the queue: every batch is set
            j = 0
            while j < len(pend):
                h, i0 = pend[j]._batch
                k = pend[j]._n
                e = j + 1
                while e < len(pend) and pend[e]._batch[0] is h and pend[e]._batch[1] == i0 + (e - j) \
                        and pend[e]._n == k:
                    e += 1
                r0, r1 = i0 * k, (i0 + e - j) * k
                self.extend_records({name: v[r0:r1] for name, v in h.items()})
                j = e

    def _reserve(self, extra: int):
        need = self._n + extra
        cap = len(self._buf["opacities"])
        if need <= cap:
            return
        new_cap = max(need, 2 * cap, 64)
        for name, w, dt in self._FIELDS:
            nb = np.empty((new_cap, w) if w else (new_cap,), dtype=dt)
            nb[:self._n] = self._buf[name][:self._n]
            self._buf[name] = nb

    def __len__(self) -> int:
        return self._n + sum(len(lz) for lz in self._lazy)

    def _get(self, name):
        self._settle()
        return self._buf[name][:self._n]

    def _set(self, name, value):
        self._settle()
        w = dict((f, wd) for f, wd, _ in self._FIELDS)[name]
        dt = dict((f, d) for f, _, d in self._FIELDS)[name]
        v = np.asarray(value, dtype=dt)
        v = v.reshape(-1, w) if w else v.reshape(-1)
        self._buf[name] = v.copy()
        self._n = len(v)

    positions = property(lambda s: s._get("positions"), lambda s, v: s._set("positions", v))
    scales = property(lambda s: s._get("scales"), lambda s, v: s._set("scales", v))
    rotations = property(lambda s: s._get("rotations"), lambda s, v: s._set("rotations", v))
    opacities = property(lambda s: s._get("opacities"), lambda s, v: s._set("opacities", v))
    colors = property(lambda s: s._get("colors"), lambda s, v: s._set("colors", v))
    source_keys = property(lambda s: s._get("source_keys"), lambda s, v: s._set("source_keys", v))

    def extend(self, primitives: list[GaussianPrimitive]) -> None:
        if isinstance(primitives, _LazyPrimitives) and primitives._batch is None:
            if self._lazy and self._lazy[-1]._batch is not None:
                # the queue was flushed since (a new frame's first voxel): settle
                # the computed voxels now so the queue of lazy objects stays short
                self._settle()
            self._lazy.append(primitives)        # materialised on the next read
            return
        if not primitives:
            return
        self._settle()
        self.extend_arrays(
            np.stack([p.position for p in primitives]), np.stack([p.scale for p in primitives]),
            np.stack([p.rotation for p in primitives]),
            np.array([p.opacity for p in primitives]), np.stack([p.color for p in primitives]),
            np.array([p.source_key if p.source_key is not None else (0, 0, 0)
                      for p in primitives], dtype=np.int64).reshape(-1, 3))

    def extend_arrays(self, positions, scales, rotations, opacities, colors, source_keys):
        if self._lazy:
            self._settle()
        k = len(opacities)
        self._reserve(k)
        for name, arr in (("positions", positions), ("scales", scales), ("rotations", rotations),
                          ("opacities", opacities), ("colors", colors),
                          ("source_keys", source_keys)):
            self._buf[name][self._n:self._n + k] = arr
        self._n += k

    def extend_records(self, rec: dict) -> None:
        self.extend_arrays(rec["position"], rec["scale"], rec["rotation"], rec["opacity"],
                           rec["color"], rec["source_key"])

    def primitive(self, i: int) -> GaussianPrimitive:
        return GaussianPrimitive(
            position=self.positions[i].copy(), scale=self.scales[i].copy(),
            rotation=self.rotations[i].copy(), opacity=float(self.opacities[i]),
            color=self.colors[i].copy(),
            source_key=VoxelKey(*(int(v) for v in self.source_keys[i])))

    def copy(self) -> "GaussianMap":
        out = GaussianMap()
        out.extend_arrays(self.positions, self.scales, self.rotations, self.opacities,
                          self.colors, self.source_keys)
        return out

    @classmethod
    def from_arrays(cls, positions, scales, rotations, opacities, colors,
                    source_keys=None) -> "GaussianMap":
        positions = np.asarray(positions, dtype=float).reshape(-1, 3)
        n = len(positions)
        if source_keys is None:
            source_keys = np.zeros((n, 3), dtype=np.int64)
        out = cls()
        out.extend_arrays(positions, np.asarray(scales, dtype=float).reshape(n, 3),
                          np.asarray(rotations, dtype=float).reshape(n, 4),
                          np.asarray(opacities, dtype=float).reshape(n),
                          np.asarray(colors, dtype=float).reshape(n, 3),
                          np.asarray(source_keys, dtype=np.int64).reshape(n, 3))
        return out
