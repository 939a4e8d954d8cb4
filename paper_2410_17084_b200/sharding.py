"""Multi-GPU voxel hash-sharding.

The mapping path shards by voxel: a voxel's solve and Gaussian init touch only
that voxel (gpr.py:281-310, SPEC "embarrassingly parallel over problems").
Ownership is `mix64(packed_key ^ 0x9e3779b97f4a7c15) % world` — the same
function the hashing kernel applies (`shard_of` in csrc/vx_map.cu) — so every
rank receives the whole scan by H2D from pinned host memory, keeps only its
keys in its own device map and never exchanges data on the hot path (no
data-path collective; weak scaling).

The only collective is the hand-off of the outputs to a consumer rank
(SURVEY §8(e)): the frame's predictions (81 points x (xyz, rgb, variance) per
solved voxel) and its Gaussian records.  `gather_v` is a gather-v: an
all-gather of the per-rank counts, then ONE grouped batch of point-to-point
transfers (`dist.batch_isend_irecv` = ncclGroupStart / ncclSend x fields /
ncclRecv x (ranks x fields) / ncclGroupEnd over NVLink) straight into the
consumer's output slices — no padding, no intermediate copies.  The consumer
then restores the single-GPU order with one stable sort by the order key
((frame << 32) | index of the voxel's first point in the frame, taken when the
voxel is solved).  Single-GPU outputs are in update order = ascending first
point index within a frame (voxel_map.py:324-326, gpr.py:281-310,
pipeline.py:154-171), so the gathered predictions and records are identical,
bit for bit and in order, to an unsharded run.
"""

from __future__ import annotations

import numpy as np

from .engine import MappingEngine
from .errors import InputDomainError

KEY_BITS = 21
KEY_BIAS = 1 << (KEY_BITS - 1)
_M64 = (1 << 64) - 1
SHARD_SALT = 0x9E3779B97F4A7C15


def pack_keys(keys) -> np.ndarray:
    """Host replica of csrc/vx_common.cuh pack_key (3 x 21-bit offset binary)."""
    k = np.asarray(keys, dtype=np.int64).reshape(-1, 3) + KEY_BIAS
    if k.size and (k.min() < 0 or k.max() >= (1 << KEY_BITS)):
        raise ValueError("key outside the packed lattice")
    k = k.astype(np.uint64)
    return (k[:, 0] << np.uint64(2 * KEY_BITS)) | (k[:, 1] << np.uint64(KEY_BITS)) | k[:, 2]


def mix64(x: np.ndarray) -> np.ndarray:
    """murmur3 finaliser, vectorised (host replica of csrc mix64)."""
    x = np.asarray(x, dtype=np.uint64).copy()
    with np.errstate(over="ignore"):
        x ^= x >> np.uint64(33)
        x *= np.uint64(0xFF51AFD7ED558CCD)
        x ^= x >> np.uint64(33)
        x *= np.uint64(0xC4CEB9FE1A85EC53)
        x ^= x >> np.uint64(33)
    return x


def owner_of(keys, world: int) -> np.ndarray:
    """Rank that owns each voxel key (identical to the device's shard_of)."""
    if world <= 1:
        return np.zeros(len(np.asarray(keys).reshape(-1, 3)), dtype=np.int64)
    h = mix64(pack_keys(keys) ^ np.uint64(SHARD_SALT))
    return (h % np.uint64(world)).astype(np.int64)


def _staged(t, backend: str):
    """gloo moves host tensors only: stage device tensors through the host."""
    return t.cpu() if backend == "gloo" and t.is_cuda else t


def gather_v(fields: dict, order, dst: int = 0, group=None):
    """Gather per-rank row sets to `dst` and merge them into global order.

    `fields` maps name -> tensor whose leading dimension is this rank's row
    count; `order` (int64, same rows) is the merge key.  Returns the merged
    dict (rows sorted stably by `order`; the key itself under "order") on
    `dst`, None elsewhere.  NCCL moves device tensors rank to rank over NVLink;
    under gloo (CPU tests) the same calls move host tensors.
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    backend = dist.get_backend(group)
    dev = order.device
    cdev = torch.device("cpu") if backend == "gloo" else dev
    n = torch.tensor([order.numel()], dtype=torch.int64, device=cdev)
    counts = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(counts, n, group=group)
    counts = [int(c.item()) for c in counts]
    names = sorted(fields) + ["order"]
    src = dict(fields, order=order)
    ops = []
    out = None
    if rank == dst:
        total = sum(counts)
        offs = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
        out = {}
        for nm in names:
            t = src[nm]
            out[nm] = torch.empty((total,) + tuple(t.shape[1:]), dtype=t.dtype, device=cdev)
            out[nm][offs[rank]:offs[rank + 1]] = _staged(t, backend)
        for r in range(world):
            if r == rank or counts[r] == 0:
                continue
            for nm in names:
                ops.append(dist.P2POp(dist.irecv, out[nm][offs[r]:offs[r + 1]],
                                      dist.get_global_rank(group, r) if group else r, group))
    elif counts[rank]:
        keep = []
        for nm in names:
            t = _staged(src[nm].contiguous(), backend)
            keep.append(t)
            ops.append(dist.P2POp(dist.isend, t,
                                  dist.get_global_rank(group, dst) if group else dst, group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    if rank != dst:
        return None
    key = out.pop("order")
    perm = torch.sort(key, stable=True).indices
    res = {k: v.index_select(0, perm) for k, v in out.items()}
    res["order"] = key.index_select(0, perm)
    if backend == "gloo" and dev.type == "cuda":
        res = {k: v.to(dev) for k, v in res.items()}
    return res


def gather_records(rec: dict, order, dst: int = 0, group=None):
    """Gaussian record SoA fields of every rank -> `dst`, in global order."""
    out = gather_v(rec, order, dst=dst, group=group)
    if out is not None:
        out.pop("order")
    return out


class ShardedEngine:
    """MappingEngine on rank `rank` of `world`: owns mix64(key) % world == rank.

    Every rank ingests the whole scan (its hashing kernel keeps only owned
    keys); `gather_frame` hands the frame's predictions and new Gaussian
    records to the consumer rank, `gather` the whole Gaussian map.
    """

    def __init__(self, config, rank: int, world: int, group=None, **kw):
        self.rank, self.world = rank, world
        self.engine = MappingEngine(config, shard_rank=rank, shard_world=world,
                                    track_order=True, **kw)
        self._frame_first_record = 0
        self.group = group
        if world > 1:
            # expansion_threshold counts pending voxels over the WHOLE map
            # (pipeline.py:157-159): every shard expands when the global count
            # reaches it, so the records match an unsharded run
            self.engine._expand_now = self._expand_now

    def _expand_now(self, pending: int) -> bool:
        import torch
        import torch.distributed as dist
        from . import _native as N
        dev = torch.device("cpu") if dist.get_backend(self.group) == "gloo" else N.device()
        t = torch.tensor([pending], dtype=torch.int64, device=dev)
        dist.all_reduce(t, group=self.group)
        total = int(t.item())
        return total > 0 and total >= self.engine.config.expansion_threshold

    def ingest(self, positions, colors, camera=None, image=None):
        self._frame_first_record = self.engine.num_gaussians
        return self.engine.ingest(positions, colors, camera, image)

    def ingest_device(self, d_xyz, d_rgb, n, camera=None, d_image=None):
        self._frame_first_record = self.engine.num_gaussians
        return self.engine.ingest_device(d_xyz, d_rgb, n, camera, d_image)

    def ingest_sliced(self, d_xyz, d_rgb, n: int, global_base: int, camera=None, d_image=None):
        """Ingest this rank's slice (rows [global_base, global_base + n)) of a
        scan that is split over the ranks.

        The slice's points are grouped by the rank owning their voxel
        (`vx_map_partition_by_owner`), exchanged with one all-to-all (NCCL over
        NVLink; under gloo through the host), and the points this rank receives
        — its voxels' points of the whole scan, in global frame order since the
        slices are contiguous and each group keeps frame order — are ingested
        with their global row numbers as the order-key source.  Outputs equal
        `ingest` of the whole scan on every rank (bit for bit after
        `gather_frame`); each rank moves 1/world of the scan over PCIe.
        """
        import ctypes as C
        import torch
        import torch.distributed as dist
        from . import _native as N
        eng = self.engine
        world = self.world
        dev = N.device()
        ox = torch.empty((max(n, 0), 3), dtype=torch.float64, device=dev)
        oc = torch.empty_like(ox)
        og = torch.empty(max(n, 0), dtype=torch.int64, device=dev)
        counts = (C.c_int64 * (world + 1))()
        vm = eng.vmap
        h = vm._h()
        N.check(vm._lib.vx_map_partition_by_owner(h, N.ptr(d_xyz), N.ptr(d_rgb), int(n),
                                                   int(global_base), N.ptr(ox), N.ptr(oc),
                                                   N.ptr(og), counts, N.stream_ptr()))
        backend = dist.get_backend(self.group)
        cdev = torch.device("cpu") if backend == "gloo" else dev
        # rows without a voxel key fail the frame on EVERY rank (the reference
        # rejects the frame; no rank may go on to the next collective alone)
        bad = torch.tensor([int(counts[world])], dtype=torch.int64, device=cdev)
        dist.all_reduce(bad, group=self.group)
        if int(bad.item()):
            raise InputDomainError(f"{int(bad.item())} scan points have no voxel key "
                                   "(non-finite, or outside the lattice |k| < 2^20)")
        send = torch.tensor(list(counts)[:world], dtype=torch.int64, device=cdev)
        recv = torch.empty_like(send)
        dist.all_to_all_single(recv, send, group=self.group)
        ss, rs = [int(x) for x in send.tolist()], [int(x) for x in recv.tolist()]
        tot = sum(rs)

        def exchange(t, shape):
            out = torch.empty((tot,) + shape, dtype=t.dtype, device=cdev)
            dist.all_to_all_single(out, _staged(t, backend), output_split_sizes=rs,
                                   input_split_sizes=ss, group=self.group)
            return out.to(dev) if out.device != dev else out

        rx, rc, rg = exchange(ox, (3,)), exchange(oc, (3,)), exchange(og, ())
        self._frame_first_record = eng.num_gaussians
        return eng.ingest_device(rx, rc, tot, camera, d_image, point_index=rg)

    def reset(self):
        self.engine.reset()
        self._frame_first_record = 0

    def _records(self, lo: int = 0):
        recs = self.engine.gaussians_device()
        order = self.engine.record_order()
        return {k: v[lo:] for k, v in recs.items()}, order[lo:]

    def gather_frame(self, dst: int = 0, group=None) -> dict | None:
        """The last frame's outputs on `dst`, identical to an unsharded run.

        {"predictions": {keys, order, positions, colors, variances} of every
        voxel solved in the frame (update order), "gaussians": the records the
        frame added (position, scale, rotation, opacity, color, source_key)}.
        """
        pred = self.engine.frame_predictions()
        order = pred.pop("order")
        p = gather_v(pred, order, dst=dst, group=group)
        recs, rorder = self._records(self._frame_first_record)
        g = gather_records(recs, rorder, dst=dst, group=group)
        if p is None:
            return None
        return {"predictions": p, "gaussians": g}

    def gather(self, dst: int = 0, group=None):
        """Every Gaussian record of the sharded map on `dst`, in global order."""
        recs, order = self._records(0)
        return gather_records(recs, order, dst=dst, group=group)
