"""PLY scan ingest and VXSPLAT1 map files on the device.

`read_ply_device` parses the PLY header on the host, stages the raw 15-byte
binary vertex records in pinned memory, copies them H2D (15 B/point instead of
the 48 B/point of f64 positions + colours) and widens them on the device
(`vx_decode_ply`); `read_ply` returns the reference's host `PointCloud`;
`read_ply_payload` stops at the pinned records (`PlyPayload`), which
`MappingEngine.ingest_stream` copies and decodes on its copy stream
(`stream.stream_frames`).  Every format failure raises `ParseError(path,
location, reason)` as the reference does (errors.py:39-46).

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
from .errors import ParseError
from .splat_init import GaussianMap

PLY_VERTEX = np.dtype([("x", "<f4"), ("y", "<f4"), ("z", "<f4"),
                       ("red", "u1"), ("green", "u1"), ("blue", "u1")])
_PLY_PROPS = [("float", "x"), ("float", "y"), ("float", "z"),
              ("uchar", "red"), ("uchar", "green"), ("uchar", "blue")]


def _ply_header(data: bytes, path):
    """(format, vertex count, payload offset); ParseError with the reference's
    locations (formats.py:66-118)."""
    if data[:3] != b"ply":
        raise ParseError(path, "byte 0", "missing ply magic")
    # collect the header lines first, then interpret them: a malformed line in a
    # header that never ends reports the missing end, as the reference does
    lines, off = [], 0
    while True:
        end = data.find(b"\n", off)
        if end < 0:
            raise ParseError(path, f"byte {off}", "header never ends")
        lines.append((off, data[off:end].decode("ascii", "replace").strip()))
        off = end + 1
        if lines[-1][1] == "end_header":
            break
        if len(lines) > 100:
            raise ParseError(path, f"byte {off}", "header too long")
    if lines[0][1] != "ply":
        raise ParseError(path, "byte 0", "missing ply magic")
    fmt, count, props = None, None, []
    for line_off, line in lines[1:-1]:
        tok = line.split()
        if not tok or tok[0] == "comment":
            continue
        if tok[0] == "format":
            if len(tok) < 2 or tok[1] not in ("ascii", "binary_little_endian"):
                raise ParseError(path, f"byte {line_off}", f"unsupported format {line!r}")
            fmt = tok[1]
        elif tok[0] == "element":
            if len(tok) != 3 or tok[1] != "vertex":
                raise ParseError(path, f"byte {line_off}", f"unsupported element {line!r}")
            try:
                count = int(tok[2])
            except ValueError as exc:
                raise ParseError(path, f"byte {line_off}", "bad vertex count") from exc
        elif tok[0] == "property":
            props.append(tuple(tok[1:]))
    nlines = len(lines)
    if fmt is None or count is None:
        raise ParseError(path, "header", "format or element vertex line missing")
    if props != _PLY_PROPS:
        raise ParseError(path, "header", f"unsupported property layout {props!r}")
    return fmt, count, off, nlines


class PlyPayload:
    """Binary PLY vertex records staged in pinned host memory (15 B/point).

    `MappingEngine.ingest_stream` copies them H2D and widens them on the device
    (`vx_decode_ply`): the scan crosses PCIe at 15 B/point instead of 48.
    """

    def __init__(self, records, count: int, path=""):
        self.records, self.count, self.path = records, int(count), str(path)
        self.shape = (self.count, 3)


def read_ply_payload(path) -> PlyPayload:
    """Header parse on the host + the raw records in pinned memory (binary PLY);
    ascii files are parsed to float64 rows and re-packed (no narrowing)."""
    import torch
    data = Path(path).read_bytes()
    fmt, count, off, nlines = _ply_header(data, path)
    if fmt == "binary_little_endian":
        need = count * PLY_VERTEX.itemsize
        if len(data) - off < need:
            raise ParseError(path, f"byte {len(data)}",
                             f"payload truncated: need {need} bytes, have {len(data) - off}")
        host = torch.frombuffer(bytearray(data[off:off + need]), dtype=torch.uint8).pin_memory()
        return PlyPayload(host, count, path)
    raise ParseError(path, "header", "stream ingest expects binary_little_endian PLY frames")


def _ascii_rows(data: bytes, off: int, count: int, nlines: int, path) -> np.ndarray:
    rows = data[off:].decode("ascii", "replace").splitlines()
    if len(rows) < count:
        raise ParseError(path, f"line {nlines + len(rows)}",
                         f"payload truncated: need {count} rows, have {len(rows)}")
    out = np.empty((count, 6))
    for i in range(count):
        tok = rows[i].split()
        if len(tok) != 6:
            raise ParseError(path, f"line {nlines + i + 1}", f"expected 6 fields, got {len(tok)}")
        try:
            out[i, :3] = [float(v) for v in tok[:3]]
            out[i, 3:] = [int(v) for v in tok[3:]]
        except ValueError as exc:
            raise ParseError(path, f"line {nlines + i + 1}", f"bad vertex row: {exc}") from exc
    return out


def read_ply_device(path):
    """(d_xyz (n,3) f64, d_rgb (n,3) f64, n) on the device from a PLY file."""
    import torch
    lib = N.lib()
    data = Path(path).read_bytes()
    fmt, count, off, nlines = _ply_header(data, path)
    dev = N.device()
    xyz = torch.empty((count, 3), dtype=torch.float64, device=dev)
    rgb = torch.empty((count, 3), dtype=torch.float64, device=dev)
    if fmt == "binary_little_endian":
        need = count * PLY_VERTEX.itemsize
        if len(data) - off < need:
            raise ParseError(path, f"byte {len(data)}",
                             f"payload truncated: need {need} bytes, have {len(data) - off}")
        host = torch.frombuffer(bytearray(data[off:off + need]), dtype=torch.uint8).pin_memory()
        rec = host.to(dev, non_blocking=True)
        N.check(lib.vx_decode_ply(N.ptr(rec), count, N.ptr(xyz), N.ptr(rgb), N.stream_ptr()))
    else:
        # ascii rows hold decimal text: the reference parses them straight to
        # float64 (formats.py:140-141), so positions are not narrowed to f32
        rows = _ascii_rows(data, off, count, nlines, path)
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
    """(GaussianMap, config-echo dict) — mirror of the reference read_map
    (formats.py:172-198), ParseError locations included."""
    data = Path(path).read_bytes()
    if data[:8] != MAP_MAGIC:
        raise ParseError(path, "byte 0", "bad magic, not a map file")
    if len(data) < 8 + 16:
        raise ParseError(path, f"byte {len(data)}", "truncated header")
    version, count, echo_len = struct.unpack_from("<IQI", data, 8)
    if version != MAP_VERSION:
        raise ParseError(path, "byte 8", f"unsupported version {version}")
    body = 8 + 16
    echo = data[body:body + echo_len].decode("utf-8")
    need = count * MAP_RECORD.itemsize
    payload = data[body + echo_len:body + echo_len + need]
    if len(payload) < need:
        raise ParseError(path, f"byte {len(data)}",
                         f"payload truncated: need {need} bytes, have {len(data) - body - echo_len}")
    rec = np.frombuffer(payload, dtype=MAP_RECORD)
    gmap = GaussianMap.from_arrays(rec["position"], rec["scale"], rec["rotation"], rec["opacity"],
                                   rec["color"], rec["source_key"])
    pairs = dict(line.split("=", 1) for line in echo.splitlines() if "=" in line)
    return gmap, {k.strip(): v.strip() for k, v in pairs.items()}
