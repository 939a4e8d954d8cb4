"""Multi-GPU voxel hash-sharding.

The mapping path shards by voxel: a voxel's solve and Gaussian init touch only
that voxel (gpr.py:281-310, SPEC "embarrassingly parallel over problems").
Ownership is `mix64(packed_key ^ 0x9e3779b97f4a7c15) % world` — the same
function the hashing kernel applies (`shard_of` in csrc/vx_map.cu) — so every
rank receives the whole scan by H2D from pinned host memory, keeps only its
keys in its own device map and never exchanges data on the hot path (no
data-path collective; weak scaling).

The only collective is the optional hand-off of the Gaussian records to a
consumer rank (`gather_records`): an all-gather of per-rank counts, a padded
gather of the SoA fields over NCCL (gloo on CPU for the tests), and a stable
sort by the record order key (frame << 32 | first point index of the voxel in
that frame).  Because single-GPU records are emitted in first-solve update
order — i.e. ascending first-touch point index within a frame
(voxel_map.py:324-326, pipeline.py:154-171) — the gathered map is identical,
record for record, to the single-GPU map.
"""

from __future__ import annotations

import numpy as np

from .engine import MappingEngine

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


def gather_records(rec: dict, order, dst: int = 0, group=None):
    """Gather per-rank Gaussian record SoA tensors to `dst`, in global order.

    `rec` maps field name -> tensor with the record count as leading dim;
    `order` is an int64 tensor of record order keys.  Returns the merged dict
    on `dst` (None elsewhere).  Works with NCCL (device tensors) and gloo
    (host tensors).
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    dev = order.device
    n = torch.tensor([order.numel()], dtype=torch.int64, device=dev)
    counts = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(counts, n, group=group)
    counts = [int(c.item()) for c in counts]
    cap = max(counts) if counts else 0
    out = {}
    for name in sorted(rec) + ["__order__"]:
        t = order if name == "__order__" else rec[name]
        pad = torch.zeros((cap,) + tuple(t.shape[1:]), dtype=t.dtype, device=dev)
        pad[: t.shape[0]] = t
        bufs = [torch.empty_like(pad) for _ in range(world)] if rank == dst else None
        dist.gather(pad, bufs, dst=dst, group=group)
        if rank == dst:
            out[name] = torch.cat([b[:c] for b, c in zip(bufs, counts)])
    if rank != dst:
        return None
    perm = torch.sort(out.pop("__order__"), stable=True).indices
    return {k: v.index_select(0, perm) for k, v in out.items()}


class ShardedEngine:
    """MappingEngine on rank `rank` of `world`: owns mix64(key) % world == rank."""

    def __init__(self, config, rank: int, world: int, **kw):
        self.rank, self.world = rank, world
        self.engine = MappingEngine(config, shard_rank=rank, shard_world=world, **kw)
        self.orders = []

    def ingest(self, positions, colors, camera=None, image=None):
        before = self.engine.num_gaussians
        rep = self.engine.ingest(positions, colors, camera, image)
        self._record_order(before, rep)
        return rep

    def _record_order(self, before: int, rep):
        import torch
        from . import _native as N
        added = self.engine.num_gaussians - before
        if added == 0:
            return
        v = self.engine.vmap.device_view()
        S = int(v.solve_candidates)
        st = N.view_tensor(v.solve_status, (S,), np.uint8)
        bf = N.view_tensor(v.solve_state_before, (S,), np.uint8)
        vids = N.view_tensor(v.solve_voxels, (S,), np.int32)
        first = vids[(st == N.ST_OK) & (bf == 1)].long()
        lf = N.view_tensor(v.last_first, (int(v.num_voxels),), np.int32)
        key = (int(rep.frame_index) << 32) | lf.index_select(0, first).long()
        nsub = self.engine.config.n_s ** 2
        self.orders.append(torch.repeat_interleave(key, nsub))

    def gather(self, dst: int = 0, group=None):
        import torch
        dev = self.engine.records.position.device if self.engine.records is not None else None
        recs = self.engine.gaussians_device()
        order = torch.cat(self.orders) if self.orders else torch.empty(0, dtype=torch.int64,
                                                                        device=dev)
        if not recs:
            recs = {k: torch.empty((0,) + s, dtype=dt, device=dev) for k, s, dt in (
                ("position", (3,), torch.float64), ("scale", (3,), torch.float64),
                ("rotation", (4,), torch.float64), ("opacity", (), torch.float64),
                ("color", (3,), torch.float64), ("source_key", (3,), torch.int64))}
        return gather_records(recs, order, dst=dst, group=group)
