"""Device-resident ingest: the batched public entry point of the hot path.

`MappingEngine.ingest` is `MappingPipeline.ingest_frame` (pipeline.py:139-187)
restricted to the mapping hot path — store the scan, densify the touched
READY/ACTIVE voxels, initialise Gaussians for first solves once
`expansion_threshold` of them are pending — executed as one
`vx_map_ingest` call (expansion_threshold == 1) with every intermediate in
HBM.  Inputs may be host arrays (copied H2D from pinned staging) or device
tensors; Gaussian records accumulate in a device SoA.
"""

from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .config import PipelineConfig
from .formats import PlyPayload
from .splat_init import GaussianMap, GaussianRecords, image_for_camera
from .voxel_map import VoxelMap


@dataclass
class IngestReport:
    """Same fields as pipeline.IngestReport (pipeline.py:77-95)."""

    frame_index: int
    points_stored: int
    voxels_touched: int
    voxels_solved: int
    newly_active: int
    newly_converged: int
    primitives_added: int
    duration_s: float
    errors: list = field(default_factory=list)

    def to_dict(self) -> dict:
        return {"frame": self.frame_index, "points": self.points_stored,
                "touched": self.voxels_touched, "solved": self.voxels_solved,
                "newly_active": self.newly_active, "newly_converged": self.newly_converged,
                "primitives_added": self.primitives_added,
                "ingest_s": round(self.duration_s, 6), "errors": self.errors}


class MappingEngine:
    def __init__(self, config: PipelineConfig, *, shard_rank: int = 0, shard_world: int = 1,
                 voxel_capacity: int = 0, point_capacity: int = 0, gaussian_capacity: int = 0,
                 record_log: bool = False, track_order: bool = False):
        self.config = config
        self.vmap = VoxelMap.from_config(config, shard_rank=shard_rank, shard_world=shard_world,
                                         voxel_capacity=voxel_capacity,
                                         point_capacity=point_capacity, record_log=record_log)
        self._gcap = int(gaussian_capacity)
        self.records = None
        self.num_gaussians = 0
        self.pending = []        # device int32 tensors of first-solved voxel ids
        self._pending_n = 0
        self._pinned = {}
        # track_order: a global order key per record, (frame << 32) | index of the
        # voxel's first point in the frame that first-solved it, taken when the
        # voxel is solved (not when its records are emitted), so sharded outputs
        # can be merged back into the single-GPU order (sharding.py)
        self.track_order = bool(track_order)
        self._orders = []        # device int64 tensors, one per record batch
        self._pending_keys = []  # order keys of the pending voxels (threshold > 1)

    # -- buffers ------------------------------------------------------------
    def _ensure_records(self, need: int):
        import torch
        if self.records is not None and self.records.count >= need:
            return
        cap = max(need, 2 * (self.records.count if self.records else 0), self._gcap, 1024)
        new = GaussianRecords(cap)
        if self.records is not None and self.num_gaussians:
            n = self.num_gaussians
            for k in ("position", "scale", "rotation", "opacity", "color", "source_key"):
                getattr(new, k)[:n].copy_(getattr(self.records, k)[:n])
        self.records = new
        # device-wide: the old buffer may still be read by a D2H on another stream
        torch.cuda.synchronize()

    def _stage_host(self, name, arr):
        """Copy a host array into a reusable pinned buffer (no device work)."""
        import torch
        a = np.ascontiguousarray(arr, dtype=np.float64)
        buf = self._pinned.get(name)
        if buf is None or buf.numel() < a.size:
            buf = torch.empty(a.size, dtype=torch.float64).pin_memory()
            self._pinned[name] = buf
        host = buf[:a.size]
        host.numpy()[:] = a.reshape(-1)
        return host.view(*a.shape)

    def _stage(self, name, arr):
        """Copy a host array into a reusable pinned buffer, then H2D (async)."""
        return self._stage_host(name, arr).to(N.device(), non_blocking=True)

    def _first_solves(self, frame_index: int):
        """(voxel ids, order keys) of the last densify's first solves, update order."""
        v = self.vmap.device_view()
        S = int(v.solve_candidates)
        st = N.view_tensor(v.solve_status, (S,), np.uint8)
        bf = N.view_tensor(v.solve_state_before, (S,), np.uint8)
        vids = N.view_tensor(v.solve_voxels, (S,), np.int32)
        first = vids[(st == N.ST_OK) & (bf == 1)].clone()
        keys = None
        if self.track_order:
            lf = N.view_tensor(v.last_first, (int(v.num_voxels),), np.int32)
            keys = (int(frame_index) << 32) | self._global_point(lf.index_select(0, first.long()).long())
        return first, keys

    def _global_point(self, idx):
        """Frame point numbers -> the scan's global row numbers (sliced ingest)."""
        pi = getattr(self, "_point_index", None)
        return idx if pi is None else pi.index_select(0, idx)

    def _append_orders(self, keys):
        import torch
        if keys is not None and keys.numel():
            self._orders.append(torch.repeat_interleave(keys, self.config.n_s * self.config.n_s))

    def record_order(self):
        """Order keys of the records `gaussians_device()` returns (track_order)."""
        import torch
        if not self.track_order:
            raise RuntimeError("MappingEngine(track_order=True) is required")
        if not self._orders:
            return torch.empty(0, dtype=torch.int64, device=N.device())
        if len(self._orders) > 1:
            self._orders = [torch.cat(self._orders)]
        return self._orders[0]

    def frame_predictions(self) -> dict:
        """The last densify's predictions as device tensors, in update order.

        `densify_frame`'s `list[VoxelPrediction]` (gpr.py:269-311) without the
        host objects: keys (S,3) int64, order (S,) int64 ((frame << 32) | first
        point index, the global merge key of sharded outputs), positions (S,M,3),
        colors (S,M,3), variances (S,M) of the S voxels solved in the frame.
        """
        import torch
        v = self.vmap.device_view()
        S, M = int(v.solved), int(v.pred_points)
        V = int(v.num_voxels)
        dev = N.device()
        if S == 0:
            return {"keys": torch.empty((0, 3), dtype=torch.int64, device=dev),
                    "order": torch.empty(0, dtype=torch.int64, device=dev),
                    "positions": torch.empty((0, M, 3), dtype=torch.float64, device=dev),
                    "colors": torch.empty((0, M, 3), dtype=torch.float64, device=dev),
                    "variances": torch.empty((0, M), dtype=torch.float64, device=dev)}
        vids = N.view_tensor(v.solved_voxels, (S,), np.int32).long()
        slot = N.view_tensor(v.pred_slot, (V,), np.int32).index_select(0, vids).long()
        nslot = int(slot.max().item()) + 1
        lf = N.view_tensor(v.last_first, (V,), np.int32).index_select(0, vids).long()
        return {"keys": N.view_tensor(v.keys, (V, 3), np.int64).index_select(0, vids),
                "order": (int(v.frame_index) << 32) | self._global_point(lf),
                "positions": N.view_tensor(v.pred_xyz, (nslot, M, 3), np.float64).index_select(0, slot),
                "colors": N.view_tensor(v.pred_rgb, (nslot, M, 3), np.float64).index_select(0, slot),
                "variances": N.view_tensor(v.pred_var, (nslot, M), np.float64).index_select(0, slot)}

    # -- ingest -------------------------------------------------------------
    def ingest(self, positions, colors, camera=None, image=None) -> IngestReport:
        """Host-array ingest: H2D of the scan (and image), then `ingest_device`.

        The image (7 MB for a 640x480 float64 frame) is copied into its pinned
        buffer on a helper thread while the device stores and solves the scan;
        its H2D is issued, and the Gaussians emitted, once the copy is done."""
        t0 = time.perf_counter()
        if image is not None and camera is not None:
            image = image_for_camera(camera, image)
        deferred = image is not None and camera is not None and self.config.expansion_threshold <= 1
        fut = None
        if deferred:
            if getattr(self, "_stager", None) is None:
                from concurrent.futures import ThreadPoolExecutor
                self._stager = ThreadPoolExecutor(max_workers=1, thread_name_prefix="vx-stage")
            ev = getattr(self, "_img_ev", None)
            if ev is not None:
                ev.synchronize()            # the last frame's image H2D has left the pinned buffer
            fut = self._stager.submit(self._stage_host, "img", image)
        dx = self._stage("xyz", positions) if len(positions) else None
        dc = self._stage("rgb", colors) if len(positions) else None
        if deferred:
            rep = self.ingest_device(dx, dc, len(positions), camera, None, image_future=fut)
        else:
            di = self._stage("img", image) if image is not None else None
            rep = self.ingest_device(dx, dc, len(positions), camera, di)
        rep.duration_s = time.perf_counter() - t0
        return rep

    def ingest_stream(self, frames, reset_each: bool = False, on_frame=None,
                      fetch_records: bool = False, on_records=None, ingest_fn=None) -> list:
        """Ingest a sequence of host frames with H2D double-buffering.

        `frames` yields (positions, colors, camera, image) with positions /
        colors as (n, 3) float64 host tensors (pinned for true overlap) and
        image an (H, W, 3) float64 host tensor or None.  The copy of frame k+1
        runs on a side stream while frame k is processed, so a steady stream
        costs max(H2D, device work) per frame instead of their sum.

        `on_frame(report)` runs after each frame's ingest (e.g. the sharded
        gather).  `fetch_records`: the Gaussian records each frame adds (the
        GaussianMap the reference's ingest_frame produces on the host,
        pipeline.py:161-171) are copied D2H into pinned host memory on a third
        stream, overlapped with the next frame's device work;
        `on_records(report, host_fields)` receives them once they have landed
        (the dict's tensors are reused two frames later: copy what you keep).
        `ingest_fn(d_xyz, d_rgb, n, camera, d_image)` replaces `ingest_device`
        for each frame (e.g. `ShardedEngine.ingest_sliced` of this rank's slice).
        """
        import torch
        dev = N.device()
        compute = torch.cuda.current_stream()
        if getattr(self, "_copier", None) is None:
            # persistent side streams + double buffers (allocated once, reused)
            self._copier = torch.cuda.Stream(device=dev)
            self._d2h = torch.cuda.Stream(device=dev)
            self._bufs = [dict(), dict()]
            self._free = [None, None]
            self._hrec = [dict(), dict()]
            self._drec = [None, None]
            self._drec_free = [None, None]
        copier, bufs, free = self._copier, self._bufs, self._free
        reports = []
        waiting = []            # (report, d2h-done event, host fields)
        it = iter(frames)

        def issue(frame, slot):
            pos, col, cam, img = frame
            with torch.cuda.stream(copier):
                if free[slot] is not None:
                    copier.wait_event(free[slot])
                b = bufs[slot]
                decoded = isinstance(pos, PlyPayload)
                if decoded:
                    # raw 15-byte PLY vertex records: H2D, then widened to f64
                    # xyz / rgb by vx_decode_ply on this copy stream
                    n = pos.count
                    rec = b.get("ply")
                    if rec is None or rec.numel() < pos.records.numel():
                        rec = torch.empty(pos.records.numel(), dtype=torch.uint8, device=dev)
                        b["ply"] = rec
                    for name in ("xyz", "rgb"):
                        cur = b.get(name)
                        if cur is None or cur.shape != (n, 3):
                            b[name] = torch.empty((n, 3), dtype=torch.float64, device=dev)
                    if n:
                        rec[:pos.records.numel()].copy_(pos.records, non_blocking=True)
                        N.check(N.lib().vx_decode_ply(N.ptr(rec), n, N.ptr(b["xyz"]),
                                                      N.ptr(b["rgb"]), N.vp(copier.cuda_stream)),
                                f"vx_decode_ply {pos.path}")
                    pos = b["xyz"]
                if img is not None and cam is not None:
                    img = image_for_camera(cam, img)
                for name, t in (("xyz", pos), ("rgb", col), ("img", img)):
                    if decoded and name != "img":
                        continue          # decoded in place above
                    if t is None:
                        b[name] = None
                        continue
                    t = t if isinstance(t, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(t))
                    cur = b.get(name)
                    if cur is None or cur.shape != t.shape:
                        cur = torch.empty(t.shape, dtype=t.dtype, device=dev)
                        b[name] = cur
                    if cur.numel():
                        cur.copy_(t, non_blocking=True)
                ready = torch.cuda.Event()
                ready.record(copier)
            return (b["xyz"], b["rgb"], int(pos.shape[0]), cam, b["img"], ready)

        def fetch(rep, first, slot):
            n = self.num_gaussians - first
            done = torch.cuda.Event()
            host = self._hrec[slot]
            src = {k: v[first:first + n] for k, v in self.gaussians_device().items()} if n else {}
            ev = torch.cuda.Event()
            ev.record(compute)
            with torch.cuda.stream(self._d2h):
                self._d2h.wait_event(ev)
                out = {}
                for k, t in src.items():
                    h = host.get(k)
                    if h is None or h.shape[0] < n:
                        h = torch.empty((max(n, 1024),) + tuple(t.shape[1:]), dtype=t.dtype).pin_memory()
                        host[k] = h
                    out[k] = h[:n]
                    out[k].copy_(t, non_blocking=True)
                done.record(self._d2h)
            if reset_each:
                self._drec_free[slot] = done   # the device records may be rewritten after this
            waiting.append((rep, done, out))

        def drain(keep: int):
            while len(waiting) > keep:
                rep, done, out = waiting.pop(0)
                done.synchronize()
                if on_records is not None:
                    on_records(rep, out)

        nxt = next(it, None)
        pending = issue(nxt, 0) if nxt is not None else None
        k = 0
        while pending is not None:
            dx, dc, n, cam, di, ready = pending
            nxt = next(it, None)
            pending = issue(nxt, (k + 1) & 1) if nxt is not None else None
            compute.wait_event(ready)
            if reset_each:
                self.reset()
                if fetch_records:
                    # double-buffered device records: frame k writes one buffer while
                    # the D2H of frame k-1 reads the other
                    self.records = self._drec[k & 1]
                    if self._drec_free[k & 1] is not None:
                        compute.wait_event(self._drec_free[k & 1])
            first = self.num_gaussians
            rep = (ingest_fn or self.ingest_device)(dx, dc, n, cam, di)
            if reset_each and fetch_records:
                self._drec[k & 1] = self.records
            reports.append(rep)
            if on_frame is not None:
                on_frame(rep)
            if fetch_records:
                fetch(rep, first, k & 1)
                drain(1)
            done = torch.cuda.Event()
            done.record(compute)
            free[k & 1] = done
            k += 1
        drain(0)
        return reports

    def ingest_device(self, d_xyz, d_rgb, n: int, camera=None, d_image=None,
                      image_future=None, point_index=None) -> IngestReport:
        """One frame of device-resident points.  `point_index` (int64, n): the
        scan row number of each point when the frame is this rank's share of a
        sliced scan (`ShardedEngine.ingest_sliced`); order keys then use it."""
        t0 = time.perf_counter()
        self._point_index = point_index
        if d_image is not None and camera is not None:
            d_image = image_for_camera(camera, d_image)
        cfg = self.config
        vm = self.vmap
        vm._h()
        vm._configure_solver(cfg)
        lib = vm._lib
        nsub = cfg.n_s * cfg.n_s
        fi, di = N.VxFrameInfo(), N.VxDensifyInfo()
        added = 0
        if cfg.expansion_threshold <= 1 and camera is not None:
            # first guess for the record buffer: every touched voxel of this frame
            # can be a first solve (voxels left at tau-1 points by earlier
            # frames, or READY after a failed solve, need one new point each), so
            # the guess is only a guess; a shortfall is reported after the frame
            # has committed and the records are emitted into a grown buffer below
            guess = nsub * (n // max(cfg.tau, 1) + 1)
            self._ensure_records(self.num_gaussians + guess)
            out = self.records.out_struct(self.num_gaussians)
            cam, sc = N.camera_struct(camera), N.splat_struct(
                cfg.n_s, cfg.n_r, cfg.weight_floor, cfg.scale_floor, cfg.initial_opacity,
                cfg.rotation)
            written = C.c_int64(0)
            if image_future is not None:
                # records deferred until the image (staged on the helper thread
                # meanwhile) is on the device
                rc = lib.vx_map_ingest(vm._h(), N.ptr(d_xyz), N.ptr(d_rgb), int(n), C.byref(cam),
                                       N.ptr(None), C.byref(sc), None, 0, C.byref(written),
                                       C.byref(fi), C.byref(di), N.stream_ptr())
                vm._mutated()
                vm._frame_serial += 1
                import torch
                d_image = image_future.result().to(N.device(), non_blocking=True)
                self._img_ev = torch.cuda.Event()
                self._img_ev.record()
                if rc == N.VX_OK and written.value:
                    rc = N.VX_E_CAPACITY           # emit below (grows the buffer if needed)
            else:
                rc = lib.vx_map_ingest(vm._h(), N.ptr(d_xyz), N.ptr(d_rgb), int(n), C.byref(cam),
                                       N.ptr(d_image), C.byref(sc), C.byref(out),
                                       self.records.count - self.num_gaussians, C.byref(written),
                                       C.byref(fi), C.byref(di), N.stream_ptr())
                vm._mutated()
                vm._frame_serial += 1
            if rc == N.VX_E_CAPACITY:
                # the frame is stored and densified; its first-solve list is kept
                # by the library until the next mutating call
                self._ensure_records(self.num_gaussians + int(written.value))
                out = self.records.out_struct(self.num_gaussians)
                rc = lib.vx_map_emit_first_gaussians(
                    vm._h(), C.byref(cam), N.ptr(d_image), C.byref(sc), C.byref(out),
                    self.records.count - self.num_gaussians, C.byref(written), N.stream_ptr())
            N.check(rc)
            vm._log_from_view(int(fi.frame_index), int(fi.ready_transitions), int(di.solved))
            added = int(written.value)
            self.num_gaussians += added
            if self.track_order and added:
                self._append_orders(self._first_solves(fi.frame_index)[1])
        else:
            rc = lib.vx_map_store_frame(vm._h(), N.ptr(d_xyz), N.ptr(d_rgb), int(n), C.byref(fi),
                                        N.stream_ptr())
            vm._mutated()
            vm._frame_serial += 1
            N.check(rc)
            rc = lib.vx_map_densify(vm._h(), C.byref(di), N.stream_ptr())
            vm._mutated()
            N.check(rc)
            vm._log_from_view(int(fi.frame_index), int(fi.ready_transitions), int(di.solved))
            if di.first_solves:
                first, keys = self._first_solves(fi.frame_index)
                self.pending.append(first)
                if keys is not None:
                    self._pending_keys.append(keys)
                self._pending_n += len(first)
            if camera is not None and self._expand_now(self._pending_n):
                added = self._expand(camera, d_image)
        return IngestReport(frame_index=int(fi.frame_index), points_stored=int(n),
                            voxels_touched=int(fi.touched), voxels_solved=int(di.solved),
                            newly_active=int(di.first_solves), newly_converged=int(di.converged),
                            primitives_added=added, duration_s=time.perf_counter() - t0)

    def _expand_now(self, pending: int) -> bool:
        """pipeline.py:158-159: expand once `expansion_threshold` voxels are pending
        (ShardedEngine replaces this with the count over all shards)."""
        return pending > 0 and pending >= self.config.expansion_threshold

    def _expand(self, camera, d_image) -> int:
        if not self._pending_n:
            return 0
        import torch
        cfg = self.config
        vids = torch.cat(self.pending).contiguous()
        keys = torch.cat(self._pending_keys) if self._pending_keys else None
        self.pending, self._pending_n, self._pending_keys = [], 0, []
        recs = len(vids) * cfg.n_s * cfg.n_s
        self._ensure_records(self.num_gaussians + recs)
        out = self.records.out_struct(self.num_gaussians)
        cam, sc = N.camera_struct(camera), N.splat_struct(
            cfg.n_s, cfg.n_r, cfg.weight_floor, cfg.scale_floor, cfg.initial_opacity, cfg.rotation)
        N.check(self.vmap._lib.vx_map_init_gaussians(self.vmap._h(), N.ptr(vids), len(vids),
                                                     C.byref(cam), N.ptr(d_image), C.byref(sc),
                                                     C.byref(out), N.stream_ptr()))
        self.num_gaussians += recs
        self._append_orders(keys)
        return recs

    # -- outputs ------------------------------------------------------------
    def gaussians_device(self) -> dict:
        """The records so far as device tensors (empty tensors before the first)."""
        import torch
        n = self.num_gaussians
        if self.records is None:
            dev = N.device()
            return {k: torch.empty((0,) + s, dtype=dt, device=dev) for k, s, dt in (
                ("position", (3,), torch.float64), ("scale", (3,), torch.float64),
                ("rotation", (4,), torch.float64), ("opacity", (), torch.float64),
                ("color", (3,), torch.float64), ("source_key", (3,), torch.int64))}
        return {k: getattr(self.records, k)[:n] for k in
                ("position", "scale", "rotation", "opacity", "color", "source_key")}

    def gaussian_map(self) -> GaussianMap:
        g = GaussianMap()
        if self.num_gaussians:
            g.extend_records(self.records.to_host(self.num_gaussians))
        return g

    def reset(self):
        self.vmap.clear()
        self.num_gaussians = 0
        self.pending, self._pending_n, self._pending_keys = [], 0, []
        self._orders = []
