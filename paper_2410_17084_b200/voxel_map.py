"""Voxel map with a device-resident store (mirror of voxsplat/voxel_map.py).

Same public names, signatures and mutation semantics as the reference
(`/root/reference/pkg/src/voxsplat/voxel_map.py:35-399`).  The difference is
where the cells live: `VoxelMap` owns a `VxMap` handle of libvoxgpr whose
hash table, point arena, prediction store and lifecycle states are in HBM.
`store_frame` (voxel_map.py:313-342) and the solves run as CUDA kernels;
`cells`, `transitions` and `solve_log` are host views materialised from the
device on access.  Host-only objects (`PointCloud`, `VoxelCell` built by the
caller, `classify_voxel`, `update_voxel_variances`) keep the reference's
pure-Python semantics because they operate on host data the caller owns.
"""

from __future__ import annotations

import ctypes as C
import logging
from collections.abc import Mapping, Sequence
from dataclasses import dataclass, field
from enum import IntEnum
from typing import Iterable, NamedTuple

import numpy as np

from . import _native as N
from .errors import ContractViolationError, InputDomainError

log = logging.getLogger(__name__)


# ---------------------------------------------------------------------------
# Point containers (voxel_map.py:35-105)
# ---------------------------------------------------------------------------

@dataclass
class ColoredPoint:
    """A single LiDAR return: world position, RGB in [0, 1], noise variance m^2."""

    position: np.ndarray
    color: np.ndarray
    noise_var: float

    def __post_init__(self):
        self.position = np.asarray(self.position, dtype=float).reshape(3)
        self.color = np.asarray(self.color, dtype=float).reshape(3)
        if not np.all(np.isfinite(self.position)):
            raise InputDomainError("point position must be finite")
        if np.any(self.color < 0) or np.any(self.color > 1):
            raise InputDomainError("color components must lie in [0, 1]")
        if self.noise_var < 0:
            raise InputDomainError("noise_var must be nonnegative")


@dataclass(slots=True)
class PointCloud:
    """Struct-of-arrays batch of colored points (host arrays, validated)."""

    positions: np.ndarray
    colors: np.ndarray
    noise_var: np.ndarray

    def __post_init__(self):
        self.positions = np.asarray(self.positions, dtype=float).reshape(-1, 3)
        self.colors = np.asarray(self.colors, dtype=float).reshape(-1, 3)
        self.noise_var = np.asarray(self.noise_var, dtype=float).reshape(-1)
        n = len(self.positions)
        if len(self.colors) != n or len(self.noise_var) != n:
            raise InputDomainError("positions, colors and noise_var must agree in length")
        if n and not np.all(np.isfinite(self.positions)):
            raise InputDomainError("point positions must be finite")
        if n and (self.colors.min() < 0 or self.colors.max() > 1):
            raise InputDomainError("color components must lie in [0, 1]")
        if n and self.noise_var.min() < 0:
            raise InputDomainError("noise variances must be nonnegative")

    @classmethod
    def empty(cls) -> "PointCloud":
        return cls(np.empty((0, 3)), np.empty((0, 3)), np.empty(0))

    @classmethod
    def from_points(cls, points: Iterable[ColoredPoint]) -> "PointCloud":
        pts = list(points)
        if not pts:
            return cls.empty()
        return cls(np.stack([p.position for p in pts]), np.stack([p.color for p in pts]),
                   np.array([p.noise_var for p in pts]))

    @staticmethod
    def concat(*clouds: "PointCloud") -> "PointCloud":
        parts = [c for c in clouds if c is not None and len(c)]
        if not parts:
            return PointCloud.empty()
        return PointCloud(np.concatenate([c.positions for c in parts]),
                          np.concatenate([c.colors for c in parts]),
                          np.concatenate([c.noise_var for c in parts]))

    def subset(self, index) -> "PointCloud":
        return PointCloud(self.positions[index], self.colors[index], self.noise_var[index])

    def point(self, i: int) -> ColoredPoint:
        return ColoredPoint(self.positions[i], self.colors[i], float(self.noise_var[i]))

    def __len__(self) -> int:
        return len(self.positions)


# ---------------------------------------------------------------------------
# Keys and states (voxel_map.py:112-149)
# ---------------------------------------------------------------------------

class VoxelKey(NamedTuple):
    ix: int
    iy: int
    iz: int


class VoxelState(IntEnum):
    UNREADY = 0
    READY = 1
    ACTIVE = 2
    CONVERGED = 3


_STATES = tuple(VoxelState)          # int -> member without the enum call


def voxel_keys(positions: np.ndarray, voxel_size: float) -> np.ndarray:
    """floor(p / voxel_size) as (n, 3) int64, computed by `vx_voxel_keys`."""
    if voxel_size <= 0:
        raise InputDomainError("voxel_size must be positive")
    pts = np.asarray(positions, dtype=float).reshape(-1, 3)
    if len(pts) == 0:
        return np.empty((0, 3), dtype=np.int64)
    lib = N.lib()
    import torch
    d = N.to_device(pts)
    out = torch.empty((len(pts), 3), dtype=torch.int64, device=d.device)
    N.check(lib.vx_voxel_keys(N.ptr(d), len(pts), float(voxel_size), N.ptr(out), N.stream_ptr()))
    return out.cpu().numpy()


def voxel_key(position, voxel_size: float) -> VoxelKey:
    """Lattice cell of a position (voxel_map.py:125-133)."""
    if voxel_size <= 0:
        raise InputDomainError("voxel_size must be positive")
    p = np.asarray(position, dtype=float).reshape(3)
    if not np.all(np.isfinite(p)):
        raise InputDomainError("cannot hash a non-finite position")
    k = voxel_keys(p.reshape(1, 3), voxel_size)[0]
    return VoxelKey(int(k[0]), int(k[1]), int(k[2]))


def voxel_bounds(key, voxel_size: float) -> np.ndarray:
    """Axis-aligned bounds (2, 3) rows (lo, hi): lo = key * size, hi = lo + size."""
    lo = np.array(key, dtype=float) * voxel_size
    return np.stack([lo, lo + voxel_size])


# ---------------------------------------------------------------------------
# Cells, predictions, frame bookkeeping (voxel_map.py:156-221)
# ---------------------------------------------------------------------------

@dataclass(slots=True)
class VoxelPrediction:
    key: VoxelKey
    positions: np.ndarray
    colors: np.ndarray
    variances: np.ndarray

    def __len__(self) -> int:
        return len(self.positions)

    @property
    def mean_variance(self) -> float:
        return float(self.variances.mean())


@dataclass(slots=True)
class VoxelCell:
    key: VoxelKey
    raw: PointCloud = field(default_factory=PointCloud.empty)
    pseudo: PointCloud | None = None
    state: VoxelState = VoxelState.UNREADY
    value_axis: int | None = None
    last_prediction: VoxelPrediction | None = None

    @property
    def solved(self) -> bool:
        return self.last_prediction is not None

    @property
    def point_count(self) -> int:
        return len(self.raw)

    @property
    def mean_posterior_variance(self) -> float | None:
        if self.last_prediction is None:
            return None
        return self.last_prediction.mean_variance

    def training_cloud(self) -> PointCloud:
        if self.pseudo is None:
            return self.raw
        return PointCloud.concat(self.raw, self.pseudo)


class FrameUpdateSet:
    """Voxel keys touched by one frame, in first-touch order, no duplicates.

    Backed by an (n, 3) int64 array; `keys` materialises VoxelKey tuples on
    first use.  `_source` identifies the device frame list it mirrors, so
    `densify_frame` can reuse it without re-uploading the keys.
    """

    def __init__(self, keys=None, *, array=None, source=None):
        if array is None:
            keys = list(keys or [])
            array = np.array([tuple(k) for k in keys], dtype=np.int64).reshape(-1, 3)
            self._keys = [VoxelKey(*(int(v) for v in k)) for k in keys]
        else:
            self._keys = None
        self.array = np.asarray(array, dtype=np.int64).reshape(-1, 3)
        self._source = source

    @property
    def keys(self) -> list[VoxelKey]:
        if self._keys is None:
            self._keys = [VoxelKey(a, b, c) for a, b, c in self.array.tolist()]
        return self._keys

    def __len__(self) -> int:
        return len(self.array)

    def __iter__(self):
        return iter(self.keys)

    def __eq__(self, other):
        if isinstance(other, FrameUpdateSet):
            return np.array_equal(self.array, other.array)
        return NotImplemented

    def __repr__(self):
        return f"FrameUpdateSet({len(self)} keys)"


@dataclass(slots=True)
class StateTransition:
    frame: int
    key: VoxelKey
    old: VoxelState
    new: VoxelState


# ---------------------------------------------------------------------------
# Pure lifecycle functions on host cells (voxel_map.py:228-261)
# ---------------------------------------------------------------------------

def classify_voxel(cell: VoxelCell, tau: int, eta: float) -> VoxelState:
    """UNREADY/READY by point count until solved, then ACTIVE/CONVERGED by eta."""
    if not cell.solved:
        return VoxelState.READY if cell.point_count >= tau else VoxelState.UNREADY
    return VoxelState.CONVERGED if cell.mean_posterior_variance <= eta else VoxelState.ACTIVE


def update_voxel_variances(cell: VoxelCell, prediction: VoxelPrediction, tau: int,
                           eta: float) -> VoxelCell:
    """Fold a solve result back into a host cell and reclassify it."""
    if prediction.key != cell.key:
        raise ContractViolationError(
            f"prediction for voxel {prediction.key} applied to cell {cell.key}")
    if cell.state not in (VoxelState.READY, VoxelState.ACTIVE):
        raise ContractViolationError(
            f"cell {cell.key} in state {cell.state.name} cannot accept a solve")
    cell.pseudo = PointCloud(prediction.positions, prediction.colors,
                             np.clip(prediction.variances, 0.0, None))
    cell.last_prediction = prediction
    cell.state = classify_voxel(cell, tau, eta)
    return cell


# ---------------------------------------------------------------------------
# The device-backed map
# ---------------------------------------------------------------------------

class _Snapshot:
    """Host copy of the whole device store at one mutation epoch."""

    def __init__(self, vmap: "VoxelMap"):
        v = vmap._view()
        V = int(v.num_voxels)
        M = int(v.pred_points)
        self.V = V
        self.M = M
        self.keys = N.view_tensor(v.keys, (V, 3), np.int64).cpu().numpy()
        self.state = N.view_tensor(v.state, (V,), np.uint8).cpu().numpy()
        self.axis = N.view_tensor(v.value_axis, (V,), np.int8).cpu().numpy()
        self.count = N.view_tensor(v.raw_count, (V,), np.int32).cpu().numpy()
        self.off = N.view_tensor(v.raw_offset, (V,), np.int64).cpu().numpy()
        self.slot = N.view_tensor(v.pred_slot, (V,), np.int32).cpu().numpy()
        self.has = N.view_tensor(v.has_pred, (V,), np.uint8).cpu().numpy()
        top = int((self.off + self.count).max()) if V else 0
        self.xyz = N.view_tensor(v.raw_xyz, (top, 3), np.float64).cpu().numpy()
        self.rgb = N.view_tensor(v.raw_rgb, (top, 3), np.float64).cpu().numpy()
        slots = int(self.slot.max()) + 1 if V and self.slot.max() >= 0 else 0
        self.pxyz = N.view_tensor(v.pred_xyz, (slots, M, 3), np.float64).cpu().numpy()
        self.prgb = N.view_tensor(v.pred_rgb, (slots, M, 3), np.float64).cpu().numpy()
        self.pvar = N.view_tensor(v.pred_var, (slots, M), np.float64).cpu().numpy()
        self.index = {tuple(k): i for i, k in enumerate(self.keys.tolist())}
        self.sensor_var = vmap.sensor_var

    def cell(self, vid: int) -> VoxelCell:
        key = VoxelKey(*(int(x) for x in self.keys[vid]))
        o, c = int(self.off[vid]), int(self.count[vid])
        raw = PointCloud(self.xyz[o:o + c].copy(), self.rgb[o:o + c].copy(),
                         np.full(c, self.sensor_var))
        cell = VoxelCell(key=key, raw=raw, state=VoxelState(int(self.state[vid])),
                         value_axis=None if self.axis[vid] < 0 else int(self.axis[vid]))
        if self.has[vid]:
            s = int(self.slot[vid])
            pred = VoxelPrediction(key, self.pxyz[s].copy(), self.prgb[s].copy(),
                                   self.pvar[s].copy())
            cell.last_prediction = pred
            cell.pseudo = PointCloud(pred.positions, pred.colors, pred.variances)
        return cell


FRAME_CACHE_MAX = 1 << 17


class _EventLog(Sequence):
    """`VoxelMap.transitions` / `solve_log`: a read-only list whose rows live in
    numpy chunks (frame, key, old, new) and become `StateTransition` objects
    (or `(frame, key)` tuples) only when read.  A long-running map therefore
    holds O(1) Python objects per frame instead of one per transition, which
    keeps the caller's garbage-collector passes short."""

    def __init__(self, solves: bool = False):
        self._solves = solves
        self._chunks = []
        self._flat = None
        self._n = 0

    def add(self, frames, keys, old=None, new=None):
        k = len(frames)
        if k:
            self._chunks.append((np.asarray(frames, np.int64), np.asarray(keys, np.int64).reshape(-1, 3),
                                 None if old is None else np.asarray(old, np.int64),
                                 None if new is None else np.asarray(new, np.int64)))
            self._n += k
            self._flat = None

    def _arrays(self):
        if self._flat is None:
            if len(self._chunks) > 1:
                fr = np.concatenate([c[0] for c in self._chunks])
                ky = np.concatenate([c[1] for c in self._chunks])
                od = None if self._solves else np.concatenate([c[2] for c in self._chunks])
                nw = None if self._solves else np.concatenate([c[3] for c in self._chunks])
                self._chunks = [(fr, ky, od, nw)]
            self._flat = self._chunks[0] if self._chunks else \
                (np.empty(0, np.int64), np.empty((0, 3), np.int64), np.empty(0, np.int64),
                 np.empty(0, np.int64))
        return self._flat

    def _rows(self, lo, hi, step=1):
        fr, ky, od, nw = self._arrays()
        fr, ky = fr[lo:hi:step].tolist(), ky[lo:hi:step].tolist()
        if self._solves:
            return [(f, VoxelKey(*k)) for f, k in zip(fr, ky)]
        od, nw = od[lo:hi:step].tolist(), nw[lo:hi:step].tolist()
        return [StateTransition(f, VoxelKey(*k), _STATES[a], _STATES[b])
                for f, k, a, b in zip(fr, ky, od, nw)]

    def __len__(self):
        return self._n

    def __getitem__(self, i):
        if isinstance(i, slice):
            return self._rows(*i.indices(self._n))
        if i < 0:
            i += self._n
        if not 0 <= i < self._n:
            raise IndexError(i)
        return self._rows(i, i + 1)[0]

    def __iter__(self):
        for lo in range(0, self._n, 4096):
            yield from self._rows(lo, min(lo + 4096, self._n))

    def __eq__(self, other):
        return list(self) == list(other)

    def __repr__(self):
        return f"[{len(self)} {'solves' if self._solves else 'transitions'}]"


class _DeviceCell(VoxelCell):
    """A `VoxelCell` backed by the device store.

    `key`, `state` and `value_axis` are fetched with the cell; `raw`, `pseudo`
    and `last_prediction` are copied from HBM on first access (only this
    voxel's rows), or come from the batch the map prefetched for the last
    frame's solved voxels.  Like the reference's cells (which the map mutates in
    place) the lazy fields reflect the store when they are first read.  Slotted,
    with the lazy-field dict made on first use: a frame's thousands of cells
    are one tracked object each for the caller's garbage collector.
    """

    __slots__ = ("_vmap", "_vid", "_pred", "_epoch", "_lazy")

    def __init__(self, vmap, key, vid, state, axis, pred=None, epoch=None):
        self._vmap, self._vid = vmap, vid
        self.key = key
        self.state = _STATES[state]
        self.value_axis = None if axis < 0 else axis
        self._pred = pred            # (positions, colors, variances) or None
        self._epoch = epoch          # set: the map's frame batch may hold the prediction
        self._lazy = None

    def _lz(self) -> dict:
        if self._lazy is None:
            self._lazy = {}
        return self._lazy

    def _fetch(self, name):
        lz = self._lz()
        if name not in lz:
            lz.update(self._vmap._cell_payload(self._vid, want_pred=self._pred is None))
            if self._pred is not None:
                lz["pred"] = self._pred
        return lz[name]

    @property
    def raw(self):
        return self._fetch("raw")

    @raw.setter
    def raw(self, v):
        self._lz()["raw"] = v

    @property
    def last_prediction(self):
        pr = self._pred
        if pr is None and self._epoch is not None:
            # one batched copy serves every touched voxel of the frame
            found, pr = self._vmap._frame_pred(self._vid, self._epoch)
            self._epoch = None
            if found:
                self._pred = pr
                self._lz()["pred"] = pr
        if pr is None:
            lz = self._lz()
            pr = lz["pred"] if "pred" in lz else self._fetch("pred")
        if pr is None:
            return None
        if not isinstance(pr, VoxelPrediction):
            pr = VoxelPrediction(self.key, *pr)
            self._pred = pr
            self._lz()["pred"] = pr
        return pr

    @last_prediction.setter
    def last_prediction(self, v):
        self._pred = v
        self._lz()["pred"] = v

    @property
    def pseudo(self):
        lz = self._lz()
        if "pseudo" in lz:
            return lz["pseudo"]
        pr = self.last_prediction
        return None if pr is None else PointCloud(pr.positions, pr.colors, pr.variances)

    @pseudo.setter
    def pseudo(self, v):
        self._lz()["pseudo"] = v


class _CellsView(Mapping):
    """`VoxelMap.cells`: dict-like, insertion (= creation) ordered, read-only.

    `cells[key]` / `key in cells` cost O(1) device traffic: the map keeps a
    per-mutation cache of the last frame's touched voxels (metadata, and the
    predictions of its solved voxels, each fetched in ONE copy of O(touched)
    bytes) and resolves any other key with one `vx_map_lookup`.  Iteration
    (`values()`, `items()`, `iter`) is the only whole-map operation.
    """

    def __init__(self, vmap: "VoxelMap"):
        self._m = vmap

    def __getitem__(self, key):
        m = self._m
        fc = m._fc
        if fc is not None and fc[0] == m._epoch and type(key) in (VoxelKey, tuple):
            hit = fc[1].get(key)           # a touched voxel of the cached frame
            if hit is not None:
                c = m._fcells.get(hit[0])
                if c is None:
                    c = _DeviceCell(m, key if type(key) is VoxelKey else VoxelKey(*key), hit[0],
                                    hit[1], hit[2], None, fc[0])
                    m._fcells[hit[0]] = c
                return c
        c = m._cell_for(key)
        if c is None:
            raise KeyError(key)
        return c

    def get(self, key, default=None):
        try:
            return self[key]
        except KeyError:
            return default

    def __contains__(self, key):
        try:
            return self._m._cell_for(key) is not None
        except (TypeError, ValueError):
            return False

    def __iter__(self):
        s = self._m._snapshot()
        return (VoxelKey(*(int(x) for x in k)) for k in s.keys.tolist())

    def __len__(self):
        return len(self._m)

    def values(self):
        s = self._m._snapshot()
        return [s.cell(i) for i in range(s.V)]

    def items(self):
        s = self._m._snapshot()
        return [(VoxelKey(*(int(x) for x in s.keys[i])), s.cell(i)) for i in range(s.V)]


class VoxelMap:
    """Hash map from lattice keys to cells, resident in HBM (voxel_map.py:268-399).

    Single writer: every mutation is a call into libvoxgpr on the current
    CUDA stream.  `shard_rank`/`shard_world` (B200 extension) keep only the
    keys whose hash falls on this rank.
    """

    def __init__(self, voxel_size: float, sensor_var: float, tau: int, eta: float, *,
                 shard_rank: int = 0, shard_world: int = 1, voxel_capacity: int = 0,
                 point_capacity: int = 0, record_log: bool = True):
        if voxel_size <= 0:
            raise InputDomainError("voxel_size must be positive")
        if sensor_var < 0:
            raise InputDomainError("sensor_var must be nonnegative")
        self.voxel_size = float(voxel_size)
        self.sensor_var = float(sensor_var)
        self.tau = int(tau)
        self.eta = float(eta)
        self.shard_rank, self.shard_world = int(shard_rank), int(shard_world)
        self._capacity = (int(voxel_capacity), int(point_capacity))
        self.record_log = record_log
        self._handle = None
        self._epoch = 0              # bumps on every mutation
        self._frame_serial = 0       # bumps when the device frame list changes
        self._snap = None
        self._events = []            # ("t", frame, keys, old, new) / ("s", frame, keys)
        self._transitions = _EventLog()
        self._solve_log = _EventLog(solves=True)
        self._consumed = 0
        self._solver = None
        self._fc = None              # frame cache (epoch, {key: entry})
        self._fp = None              # its batched predictions {vid: tuple}
        self._fp_rest = True         # touched voxels not yet in _fp may still be fetched
        self._fcells = {}            # cells built from it {vid: _DeviceCell}
        self.cells = _CellsView(self)

    @classmethod
    def from_config(cls, config, **kw) -> "VoxelMap":
        return cls(config.voxel_size, config.sensor_var, config.tau, config.eta, **kw)

    # -- native handle ------------------------------------------------------
    def _h(self):
        if self._handle is None:
            lib = N.lib()
            cfg = N.VxMapConfig()
            cfg.voxel_size, cfg.sensor_var, cfg.tau = self.voxel_size, self.sensor_var, self.tau
            cfg.n_s, cfg.n_r, cfg.kernel = 3, 3, 0
            cfg.eta, cfg.kernel_lambda, cfg.jitter = self.eta, 1.0, 1e-10
            cfg.shard_rank, cfg.shard_world = self.shard_rank, self.shard_world
            cfg.voxel_capacity, cfg.point_capacity = self._capacity
            h = N.vp()
            N.check(lib.vx_map_create(C.byref(cfg), C.byref(h)))
            self._handle = h
            self._lib = lib
        return self._handle

    def __del__(self):
        h = getattr(self, "_handle", None)
        if h is not None:
            try:
                self._lib.vx_map_destroy(h)
            except Exception:
                pass

    def _view(self) -> N.VxMapView:
        v = N.VxMapView()
        N.check(self._lib.vx_map_view(self._h(), C.byref(v)))
        return v

    def _mutated(self):
        self._epoch += 1
        self._snap = None

    def _snapshot(self) -> _Snapshot:
        if self._handle is None:
            self._h()
        if self._snap is None or self._snap[0] != self._epoch:
            import torch
            torch.cuda.current_stream().synchronize()
            self._snap = (self._epoch, _Snapshot(self))
        return self._snap[1]

    # -- per-key cell access (O(touched) traffic) ------------------------------
    def _frame_cache(self):
        """{key tuple: [vid, state, axis, has_pred, cell|None]} of the last frame's
        touched voxels at the current mutation epoch, in one batched device
        gather (keys and metadata; the predictions follow on first use, see
        `_frame_pred`)."""
        fc = self._fc
        if fc is not None and fc[0] == self._epoch:
            return fc[1]
        import torch
        cache = {}
        if self._handle is not None:
            v = self._view()
            U, V = int(v.frame_touched), int(v.num_voxels)
            # frames of up to FRAME_CACHE_MAX voxels are prefetched in one batch;
            # larger ones (config-4 scale) resolve keys one lookup at a time
            if U and V and U <= FRAME_CACHE_MAX:
                vids = N.view_tensor(v.frame_voxels, (U,), np.int32).long()
                keys = N.view_tensor(v.keys, (V, 3), np.int64).index_select(0, vids)
                st = N.view_tensor(v.state, (V,), np.uint8).index_select(0, vids).long()
                ax = N.view_tensor(v.value_axis, (V,), np.int8).index_select(0, vids).long()
                hp = N.view_tensor(v.has_pred, (V,), np.uint8).index_select(0, vids).long()
                meta = torch.cat([torch.stack([vids, st, ax, hp], 1), keys], 1).cpu().tolist()
                # keyed by plain tuples: equal (and equally hashed) to VoxelKey;
                # int-only tuple values (the collector untracks them)
                cache = {(r[4], r[5], r[6]): (r[0], r[1], r[2], r[3]) for r in meta}
        self._fc = (self._epoch, cache)
        self._fp = None
        self._fcells = {}
        return cache

    def _frame_pred(self, vid: int, epoch: int):
        """(found, prediction tuple | None) of a voxel of the cached frame.

        Predictions arrive in batched gathers (O(touched) bytes): the first
        request at an epoch fetches the last densify's first solves among the
        touched voxels (what the pipeline's expansion loop reads,
        pipeline.py:160-165); a request outside that batch fetches every other
        touched voxel that has a prediction."""
        fc = self._fc
        if fc is None or fc[0] != epoch or epoch != self._epoch:
            return False, None
        if self._fp is None:
            self._fp, self._fp_rest = {}, True
            first = self._last_first_solves()
            if first:
                self._fetch_preds([e[0] for e in fc[1].values() if e[3] and e[0] in first])
        if vid not in self._fp and self._fp_rest:
            self._fp_rest = False
            self._fetch_preds([e[0] for e in fc[1].values() if e[3] and e[0] not in self._fp])
        return True, self._fp.get(vid)

    def _last_first_solves(self) -> set:
        """Voxel ids the last densify solved for the first time (READY before)."""
        v = self._view()
        S = int(v.solve_candidates)
        if not S:
            return set()
        st = N.view_tensor(v.solve_status, (S,), np.uint8)
        bf = N.view_tensor(v.solve_state_before, (S,), np.uint8)
        vids = N.view_tensor(v.solve_voxels, (S,), np.int32)
        return set(vids[(st == N.ST_OK) & (bf == int(VoxelState.READY))].cpu().tolist())

    def _fetch_preds(self, vids: list):
        if not vids:
            return
        import torch
        v = self._view()
        V, M = int(v.num_voxels), int(v.pred_points)
        hv = torch.as_tensor(vids, dtype=torch.long, device=N.device())
        slot = N.view_tensor(v.pred_slot, (V,), np.int32).index_select(0, hv).long()
        ns = int(slot.max().item()) + 1
        px = N.view_tensor(v.pred_xyz, (ns, M, 3), np.float64).index_select(0, slot).cpu().numpy()
        pc = N.view_tensor(v.pred_rgb, (ns, M, 3), np.float64).index_select(0, slot).cpu().numpy()
        pv = N.view_tensor(v.pred_var, (ns, M), np.float64).index_select(0, slot).cpu().numpy()
        self._fp.update({h: (px[r], pc[r], pv[r]) for r, h in enumerate(vids)})

    def _cell_for(self, key):
        cache = self._frame_cache()
        hit = cache.get(key) if type(key) in (VoxelKey, tuple) else None
        if hit is None:
            k = tuple(int(x) for x in key)
            if len(k) != 3:
                raise ValueError("voxel keys have three components")
            key = VoxelKey(*k)
            hit = cache.get(k)
        if hit is not None:
            c = self._fcells.get(hit[0])
            if c is None:
                if type(key) is not VoxelKey:
                    key = VoxelKey(*key)
                c = _DeviceCell(self, key, hit[0], hit[1], hit[2], None, self._epoch)
                self._fcells[hit[0]] = c
            return c
        if self._handle is None:
            return None
        import torch
        d = torch.tensor([tuple(key)], dtype=torch.int64, device=N.device())
        out = torch.empty(1, dtype=torch.int32, device=d.device)
        N.check(self._lib.vx_map_lookup(self._h(), N.ptr(d), 1, N.ptr(out), N.stream_ptr()))
        vid = int(out.item())
        if vid < 0:
            return None
        v = self._view()
        V = int(v.num_voxels)
        st = int(N.view_tensor(v.state, (V,), np.uint8)[vid].item())
        ax = int(N.view_tensor(v.value_axis, (V,), np.int8)[vid].item())
        return _DeviceCell(self, key, vid, st, ax)

    def _cell_payload(self, vid: int, want_pred: bool = True) -> dict:
        """raw points (and the prediction) of one voxel: O(voxel) bytes."""
        v = self._view()
        V = int(v.num_voxels)
        cnt = int(N.view_tensor(v.raw_count, (V,), np.int32)[vid].item())
        off = int(N.view_tensor(v.raw_offset, (V,), np.int64)[vid].item())
        xyz = N.view_tensor(v.raw_xyz, (off + cnt, 3), np.float64)[off:off + cnt].cpu().numpy()
        rgb = N.view_tensor(v.raw_rgb, (off + cnt, 3), np.float64)[off:off + cnt].cpu().numpy()
        out = {"raw": PointCloud(xyz, rgb, np.full(cnt, self.sensor_var))}
        if want_pred:
            pred = None
            if int(N.view_tensor(v.has_pred, (V,), np.uint8)[vid].item()):
                M = int(v.pred_points)
                sl = int(N.view_tensor(v.pred_slot, (V,), np.int32)[vid].item())
                pred = (N.view_tensor(v.pred_xyz, (sl + 1, M, 3), np.float64)[sl].cpu().numpy(),
                        N.view_tensor(v.pred_rgb, (sl + 1, M, 3), np.float64)[sl].cpu().numpy(),
                        N.view_tensor(v.pred_var, (sl + 1, M), np.float64)[sl].cpu().numpy())
            out["pred"] = pred
        return out

    # -- accessors ----------------------------------------------------------
    @property
    def frame_index(self) -> int:
        if self._handle is None:
            return -1
        return int(self._view().frame_index)

    def __len__(self) -> int:
        if self._handle is None:
            return 0
        return int(self._view().num_voxels)

    def __contains__(self, key) -> bool:
        return key in self.cells

    def cell(self, key) -> VoxelCell:
        return self.cells[key]

    def cells_in_state(self, state: VoxelState) -> list[VoxelCell]:
        s = self._snapshot()
        return [s.cell(i) for i in np.nonzero(s.state == int(state))[0]]

    def all_raw_points(self) -> PointCloud:
        return PointCloud.concat(*(c.raw for c in self.cells.values()))

    def device_view(self) -> N.VxMapView:
        """Raw device pointers of the store (valid until the next mutation)."""
        return self._view()

    # -- event log (lazy) ---------------------------------------------------
    def _record_transitions(self, frame, vids, old, new):
        if not self.record_log or len(vids) == 0:
            return
        self._events.append(("t", frame, self._keys_of(vids), old, new))

    def _record_solves(self, frame, vids, before, after):
        if not self.record_log or len(vids) == 0:
            return
        self._events.append(("s", frame, self._keys_of(vids), before, after))

    def _keys_of(self, vids: np.ndarray) -> np.ndarray:
        import torch
        v = self._view()
        keys = N.view_tensor(v.keys, (int(v.num_voxels), 3), np.int64)
        idx = torch.as_tensor(np.asarray(vids, dtype=np.int64), device=keys.device)
        return keys.index_select(0, idx).cpu().numpy()

    def _log_from_view(self, frame: int, ready_transitions: int, solved: int):
        """Event log of a store + densify that ran as one library call
        (MappingEngine / vx_map_ingest): the frame's UNREADY->READY
        transitions, then its solves, from the device view."""
        if not self.record_log:
            return
        v = self._view()
        U = int(v.frame_touched)
        if ready_transitions and U:
            vids = N.view_tensor(v.frame_voxels, (U,), np.int32).cpu().numpy()
            fb = N.view_tensor(v.frame_state_before, (U,), np.uint8).cpu().numpy()
            fa = N.view_tensor(v.frame_state_after, (U,), np.uint8).cpu().numpy()
            ch = np.nonzero(fa != fb)[0]
            self._record_transitions(frame, vids[ch], fb[ch], fa[ch])
        S = int(v.solve_candidates)
        if solved and S:
            st = N.view_tensor(v.solve_status, (S,), np.uint8).cpu().numpy()
            ok = np.nonzero(st == N.ST_OK)[0]
            vids = N.view_tensor(v.solve_voxels, (S,), np.int32).cpu().numpy()[ok]
            bf = N.view_tensor(v.solve_state_before, (S,), np.uint8).cpu().numpy()[ok]
            af = N.view_tensor(v.solve_state_after, (S,), np.uint8).cpu().numpy()[ok]
            self._record_solves(frame, vids, bf, af)

    def _drain_events(self):
        for kind, frame, keys, a, b in self._events[self._consumed:]:
            keys = np.asarray(keys, np.int64).reshape(-1, 3)
            a, b = np.asarray(a, np.int64), np.asarray(b, np.int64)
            k = len(keys)
            if kind == "t":
                self._transitions.add(np.full(k, frame), keys, a, b)
            else:
                self._solve_log.add(np.full(k, frame), keys)
                # a first solve that converges passes through ACTIVE: solve i adds
                # the transitions a_i -> a_i + 1 -> ... -> b_i, in solve order
                cnt = np.maximum(b - a, 0)
                tot = int(cnt.sum())
                if tot:
                    idx = np.repeat(np.arange(k), cnt)
                    step = np.arange(tot) - np.repeat(np.cumsum(cnt) - cnt, cnt)
                    old = a[idx] + step
                    self._transitions.add(np.full(tot, frame), keys[idx], old, old + 1)
        self._consumed = len(self._events)
        if self._consumed > 64:
            self._events, self._consumed = [], 0

    @property
    def transitions(self) -> list[StateTransition]:
        self._drain_events()
        return self._transitions

    @property
    def solve_log(self) -> list[tuple[int, VoxelKey]]:
        self._drain_events()
        return self._solve_log

    # -- mutation -----------------------------------------------------------
    def store_frame(self, cloud: PointCloud) -> FrameUpdateSet:
        """Append one frame of points to their cells (voxel_map.py:313-342)."""
        pos = np.ascontiguousarray(cloud.positions, dtype=np.float64)
        col = np.ascontiguousarray(cloud.colors, dtype=np.float64)
        dpos, dcol = (N.to_device(pos), N.to_device(col)) if len(pos) else (None, None)
        return self.store_frame_device(dpos, dcol, len(pos))

    def store_frame_device(self, d_xyz, d_rgb, n: int) -> FrameUpdateSet:
        """store_frame on device-resident (n,3) float64 tensors."""
        h = self._h()
        info = N.VxFrameInfo()
        rc = self._lib.vx_map_store_frame(h, N.ptr(d_xyz), N.ptr(d_rgb), int(n), C.byref(info),
                                          N.stream_ptr())
        self._mutated()
        self._frame_serial += 1
        N.check(rc)
        U = int(info.touched)
        if U == 0:
            return FrameUpdateSet(array=np.empty((0, 3), np.int64),
                                  source=(id(self), self._frame_serial))
        v = self._view()
        vids = N.view_tensor(v.frame_voxels, (U,), np.int32)
        keys_dev = N.view_tensor(v.keys, (int(v.num_voxels), 3), np.int64)
        keys = keys_dev.index_select(0, vids.long()).cpu().numpy()
        if self.record_log and info.ready_transitions:
            fb = N.view_tensor(v.frame_state_before, (U,), np.uint8).cpu().numpy()
            fa = N.view_tensor(v.frame_state_after, (U,), np.uint8).cpu().numpy()
            ch = np.nonzero(fa != fb)[0]
            self._events.append(("t", int(info.frame_index), keys[ch], fb[ch], fa[ch]))
        return FrameUpdateSet(array=keys, source=(id(self), self._frame_serial))

    def _configure_solver(self, config):
        want = (int(config.n_s), int(config.n_r), float(config.kernel_lambda),
                float(config.jitter), N.KERNELS[getattr(config, "kernel", "se")])
        if want != self._solver:
            N.check(self._lib.vx_map_configure_solver(self._h(), *want))
            self._solver = want

    def _select_frame(self, update_set):
        """Make `update_set` the device frame list for the next densify."""
        src = getattr(update_set, "_source", None)
        if src == (id(self), self._frame_serial):
            return
        arr = update_set.array if isinstance(update_set, FrameUpdateSet) else \
            np.array([tuple(k) for k in update_set], dtype=np.int64).reshape(-1, 3)
        d = N.to_device(arr, dtype=np.int64) if len(arr) else None
        rc = self._lib.vx_map_set_frame_keys(self._h(), N.ptr(d), len(arr), N.stream_ptr())
        self._frame_serial += 1
        if rc == N.VX_E_CONTRACT:
            raise KeyError(N.last_error())
        N.check(rc)
        if isinstance(update_set, FrameUpdateSet):
            update_set._source = (id(self), self._frame_serial)

    def _densify(self) -> N.VxDensifyInfo:
        info = N.VxDensifyInfo()
        rc = self._lib.vx_map_densify(self._h(), C.byref(info), N.stream_ptr())
        self._mutated()
        N.check(rc)
        return info

    def apply_prediction(self, prediction: VoxelPrediction):
        """Fold a host prediction into its device cell (voxel_map.py:344-355)."""
        key = np.asarray(tuple(prediction.key), dtype=np.int64)
        m = len(prediction.positions)
        dx = N.to_device(prediction.positions)
        dc = N.to_device(prediction.colors)
        dv = N.to_device(prediction.variances)
        ba = (C.c_uint8 * 2)()
        rc = self._lib.vx_map_apply_prediction(self._h(), key.ctypes.data_as(N.c_i64p), N.ptr(dx),
                                               N.ptr(dc), N.ptr(dv), m, ba, N.stream_ptr())
        if rc == N.VX_E_INPUT:
            raise KeyError(prediction.key)
        N.check(rc)
        self._mutated()
        frame = self.frame_index
        self._events.append(("s", frame, key.reshape(1, 3), np.array([ba[0]]), np.array([ba[1]])))
        return self.cells[prediction.key]

    def clear(self):
        """Drop every voxel (B200 extension; keeps device allocations)."""
        if self._handle is not None:
            N.check(self._lib.vx_map_clear(self._handle, N.stream_ptr()))
        self._mutated()
        self._frame_serial += 1
        self._events, self._consumed = [], 0
        self._transitions, self._solve_log = _EventLog(), _EventLog(solves=True)

    # -- audits (voxel_map.py:364-399) --------------------------------------
    def audit_transitions(self) -> list[str]:
        issues = []
        seq: dict = {}
        for tr in self.transitions:
            cur = seq.get(tr.key, int(VoxelState.UNREADY))
            if int(tr.old) != cur or int(tr.new) != cur + 1:
                issues.append(f"voxel {tr.key}: illegal transition "
                              f"{tr.old.name} -> {tr.new.name} at frame {tr.frame}")
            seq[tr.key] = int(tr.new)
        return issues

    def audit_converged_resolves(self) -> list[str]:
        conv = {tr.key: tr.frame for tr in self.transitions if tr.new == VoxelState.CONVERGED}
        issues = []
        for key, fc in conv.items():
            late = [f for f, k in self.solve_log if k == key and f > fc]
            if late:
                issues.append(f"voxel {key} re-solved after convergence at frames {late}")
        return issues

    def audit_hash_consistency(self) -> list[str]:
        """Raw points whose lattice key disagrees with their cell (device check)."""
        import torch
        if self._handle is None:
            return []
        v = self._view()
        V = int(v.num_voxels)
        if V == 0:
            return []
        count = N.view_tensor(v.raw_count, (V,), np.int32).long()
        off = N.view_tensor(v.raw_offset, (V,), np.int64)
        top = int((off + count).max().item())
        xyz = N.view_tensor(v.raw_xyz, (top, 3), np.float64)
        keys = N.view_tensor(v.keys, (V, 3), np.int64)
        owner = torch.repeat_interleave(torch.arange(V, device=keys.device), count)
        rows = torch.repeat_interleave(off, count) + (
            torch.arange(int(count.sum().item()), device=keys.device)
            - torch.repeat_interleave(torch.cumsum(count, 0) - count, count))
        # keys of the stored points by the hashing kernel's own arithmetic (IEEE
        # division + floor, vx_voxel_keys); torch's `xyz / scalar` on CUDA is a
        # multiply by the reciprocal and can misplace points on a lattice face
        pts = xyz[rows].contiguous()
        pk = torch.empty((len(pts), 3), dtype=torch.int64, device=keys.device)
        if len(pts):
            N.check(self._lib.vx_voxel_keys(N.ptr(pts), len(pts), float(self.voxel_size),
                                            N.ptr(pk), N.stream_ptr()))
        bad = (pk != keys[owner]).any(dim=1)
        per = torch.zeros(V, dtype=torch.int64, device=keys.device).index_add_(0, owner, bad.long())
        idx = torch.nonzero(per).flatten().cpu().numpy()
        kh = keys.cpu().numpy()
        perh = per.cpu().numpy()
        return [f"voxel {VoxelKey(*kh[i].tolist())}: {int(perh[i])} raw points hash elsewhere"
                for i in idx]
