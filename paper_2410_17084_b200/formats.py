"""PLY scan ingest and VXSPLAT1 map files on the device.

`read_ply_device` parses the PLY header on the host, stages the raw 15-byte
binary vertex records in pinned memory, copies them H2D (15 B/point instead of
the 48 B/point of f64 positions + colours) and widens them on the device
(`vx_decode_ply`); `read_ply` returns the reference's host `PointCloud`.

Same byte format as the reference writer/reader (formats.py:23-32, 154-198):
8-byte magic `VXSPLAT1`, `<IQI` (version 1, record count, echo length), the
UTF-8 config echo (`PipelineConfig.to_lines()`), then packed 136-byte records
(position 3 f8, scale 3 f8, rotation 4 f8 w-first, opacity f8, SH0 color 3 f8,
source_key 3 i8).  `write_map` packs the records on the device
(`vx_pack_map_records`) and does one D2H copy.
"""

from __future__ import annotations

import ctypes as C
import struct
from pathlib import Path

import numpy as np

from . import _native as N
from .errors import ContractViolationError, InputDomainError
from .splat_init import GaussianMap

PLY_VERTEX = np.dtype([("x", "<f4"), ("y", "<f4"), ("z", "<f4"),
                       ("red", "u1"), ("green", "u1"), ("blue", "u1")])
_PLY_PROPS = [("float", "x"), ("float", "y"), ("float", "z"),
              ("uchar", "red"), ("uchar", "green"), ("uchar", "blue")]


def _ply_header(data: bytes, path):
    if data[:3] != b"ply":
        raise InputDomainError(f"{path}: missing ply magic")
    off, fmt, count, props = 0, None, None, []
    for _ in range(101):
        end = data.find(b"\n", off)
        if end < 0:
            raise InputDomainError(f"{path}: header never ends")
        line = data[off:end].decode("ascii", "replace").strip()
        off = end + 1
        tok = line.split()
        if line == "end_header":
            break
        if not tok or tok[0] in ("comment", "ply"):
            continue
        if tok[0] == "format":
            if len(tok) < 2 or tok[1] not in ("ascii", "binary_little_endian"):
                raise InputDomainError(f"{path}: unsupported format {line!r}")
            fmt = tok[1]
        elif tok[0] == "element":
            if len(tok) != 3 or tok[1] != "vertex":
                raise InputDomainError(f"{path}: unsupported element {line!r}")
            count = int(tok[2])
        elif tok[0] == "property":
            props.append(tuple(tok[1:]))
    else:
        raise InputDomainError(f"{path}: header too long")
    if fmt is None or count is None or props != _PLY_PROPS:
        raise InputDomainError(f"{path}: unsupported PLY layout {props!r}")
    return fmt, count, off


def read_ply_device(path):
    """(d_xyz (n,3) f64, d_rgb (n,3) f64, n) on the device from a PLY file."""
    import torch
    lib = N.lib()
    data = Path(path).read_bytes()
    fmt, count, off = _ply_header(data, path)
    dev = N.device()
    xyz = torch.empty((count, 3), dtype=torch.float64, device=dev)
    rgb = torch.empty((count, 3), dtype=torch.float64, device=dev)
    if fmt == "binary_little_endian":
        need = count * PLY_VERTEX.itemsize
        if len(data) - off < need:
            raise InputDomainError(f"{path}: payload truncated")
        host = torch.frombuffer(bytearray(data[off:off + need]), dtype=torch.uint8).pin_memory()
        rec = host.to(dev, non_blocking=True)
        N.check(lib.vx_decode_ply(N.ptr(rec), count, N.ptr(xyz), N.ptr(rgb), N.stream_ptr()))
    else:
        # ascii rows hold decimal text: the reference parses them straight to
        # float64 (formats.py:140-141), so positions are not narrowed to f32
        rows = np.loadtxt(data[off:].decode("ascii").splitlines()[:count], ndmin=2)
        if len(rows) < count or rows.shape[1] != 6:
            raise InputDomainError(f"{path}: bad ascii payload")
        r = np.zeros(count, dtype=PLY_VERTEX)
        r["red"], r["green"], r["blue"] = rows[:, 3], rows[:, 4], rows[:, 5]
        rec = torch.from_numpy(r.view(np.uint8).copy()).to(dev)
        N.check(lib.vx_decode_ply(N.ptr(rec), count, N.ptr(xyz), N.ptr(rgb), N.stream_ptr()))
        xyz.copy_(torch.from_numpy(np.ascontiguousarray(rows[:, :3])))   # u8/255 colours kept
    return xyz, rgb, count


def read_ply(path, noise_var: float = 0.0):
    """PointCloud of a PLY scan (formats.py:66-147): positions widened from f32,
    colours u8 / 255, noise column = noise_var."""
    from .voxel_map import PointCloud
    xyz, rgb, n = read_ply_device(path)
    return PointCloud(xyz.cpu().numpy(), rgb.cpu().numpy(), np.full(n, float(noise_var)))


MAP_MAGIC = b"VXSPLAT1"
MAP_VERSION = 1
MAP_RECORD = np.dtype([("position", "<f8", (3,)), ("scale", "<f8", (3,)),
                       ("rotation", "<f8", (4,)), ("opacity", "<f8"), ("color", "<f8", (3,)),
                       ("source_key", "<i8", (3,))])
assert MAP_RECORD.itemsize == 136


def _device_records(src):
    """Device SoA dict from a MappingEngine, a records dict of tensors, or a GaussianMap."""
    import torch
    if hasattr(src, "gaussians_device"):
        return src.gaussians_device()
    if isinstance(src, GaussianMap):
        dev = N.device()
        f = lambda a, dt=torch.float64: torch.as_tensor(np.ascontiguousarray(a), dtype=dt, device=dev)
        return {"position": f(src.positions), "scale": f(src.scales), "rotation": f(src.rotations),
                "opacity": f(src.opacities), "color": f(src.colors),
                "source_key": f(src.source_keys, torch.int64)}
    return src


def write_map(path, source, config=None) -> int:
    """Write a VXSPLAT1 file; returns the record count."""
    import torch
    rec = _device_records(source)
    n = int(rec["opacity"].shape[0]) if rec else 0
    echo = "\n".join(config.to_lines()).encode("utf-8") if config is not None else b""
    payload = b""
    if n:
        lib = N.lib()
        fields = {k: rec[k].contiguous() for k in rec}
        o = N.VxGaussianOut()
        o.position, o.scale, o.rotation = (fields[k].data_ptr() for k in ("position", "scale", "rotation"))
        o.opacity, o.color, o.source_key = (fields[k].data_ptr() for k in ("opacity", "color", "source_key"))
        out = torch.empty(n * 136, dtype=torch.uint8, device=fields["opacity"].device)
        N.check(lib.vx_pack_map_records(C.byref(o), n, N.ptr(out), N.stream_ptr()))
        payload = out.cpu().numpy().tobytes()
    with open(Path(path), "wb") as fh:
        fh.write(MAP_MAGIC)
        fh.write(struct.pack("<IQI", MAP_VERSION, n, len(echo)))
        fh.write(echo)
        fh.write(payload)
    return n


def read_map(path):
    """(GaussianMap, config-echo dict) — mirror of the reference read_map."""
    data = Path(path).read_bytes()
    if data[:8] != MAP_MAGIC:
        raise ContractViolationError(f"{path}: bad magic, not a map file")
    version, count, echo_len = struct.unpack_from("<IQI", data, 8)
    if version != MAP_VERSION:
        raise ContractViolationError(f"{path}: unsupported version {version}")
    body = 8 + 16
    echo = data[body:body + echo_len].decode("utf-8")
    need = count * MAP_RECORD.itemsize
    payload = data[body + echo_len:body + echo_len + need]
    if len(payload) < need:
        raise ContractViolationError(f"{path}: payload truncated")
    rec = np.frombuffer(payload, dtype=MAP_RECORD)
    gmap = GaussianMap.from_arrays(rec["position"], rec["scale"], rec["rotation"], rec["opacity"],
                                   rec["color"], rec["source_key"])
    pairs = dict(line.split("=", 1) for line in echo.splitlines() if "=" in line)
    return gmap, {k.strip(): v.strip() for k, v in pairs.items()}
