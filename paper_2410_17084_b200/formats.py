"""VXSPLAT1 map files straight from device Gaussian records.

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
from .errors import ContractViolationError
from .splat_init import GaussianMap

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
