"""Frame-stream directories: NNNNNN.ply + NNNNNN.png +
trajectory.txt + scene.cfg, the container the reference writes with
`write_stream` and loads with `read_stream` (formats.py:357-409).

`read_stream(directory)` is the drop-in: a list of `FrameSample` (host
`PointCloud`, float image, `Camera`) with the reference's values and its
`ParseError`s.  `stream_frames(directory)` is the ingest path: it yields
frames for `MappingEngine.ingest_stream` whose points are the PLY's raw 15-byte
vertex records in pinned host memory (`formats.PlyPayload`); the engine copies
them H2D on its copy stream and widens them on the device (`vx_decode_ply`),
overlapped with the previous frame's mapping work.  Only the header, the
trajectory line and the PNG are parsed on the host.
"""

from __future__ import annotations

from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .camera import Camera
from .errors import ParseError
from .formats import read_ply, read_ply_payload


@dataclass
class FrameSample:
    """One input frame (pipeline.py:31-43): points, observed image, pose."""

    timestamp: float
    points: object
    image: np.ndarray
    camera: Camera

    def __post_init__(self):
        if np.shape(self.image) != (self.camera.height, self.camera.width, 3):
            from .errors import VoxsplatError
            raise VoxsplatError("frame image does not match camera dimensions")


def read_config_pairs(path):
    """(lineno, key, value) of a key=value file with # comments (formats.py:303-318)."""
    path = Path(path)
    out = []
    for lineno, raw in enumerate(path.read_text().splitlines(), start=1):
        body = raw.split("#", 1)[0].strip()
        if not body:
            continue
        key, sep, value = body.partition("=")
        if not sep:
            raise ParseError(path, f"line {lineno}", "expected key=value")
        out.append((lineno, key.strip(), value.strip()))
    return out


def read_trajectory(path):
    """(timestamp, translation (3,), unit quaternion xyzw (4,)) rows of
    "t tx ty tz qx qy qz qw" (formats.py:243-268); |q| must be within 1e-3 of 1."""
    path = Path(path)
    rows = []
    for lineno, raw in enumerate(path.read_text().splitlines(), start=1):
        line = raw.strip()
        if not line or line.startswith("#"):
            continue
        tok = line.split()
        if len(tok) != 8:
            raise ParseError(path, f"line {lineno}", f"expected 8 fields, got {len(tok)}")
        try:
            vals = np.array([float(v) for v in tok])
        except ValueError as exc:
            raise ParseError(path, f"line {lineno}", f"bad number: {exc}") from exc
        q = vals[4:8]
        qn = np.linalg.norm(q)
        if abs(qn - 1.0) > 1e-3:
            raise ParseError(path, f"line {lineno}", f"quaternion norm {qn:.3f} too far from 1")
        rows.append((float(vals[0]), vals[1:4].copy(), q / qn))
    return rows


def _rotation_of(q_wxyz) -> np.ndarray:
    """Rotation of a w-first quaternion, normalised first (geometry.py:13-29)."""
    q = np.asarray(q_wxyz, dtype=float)
    w, x, y, z = q / np.linalg.norm(q, axis=-1, keepdims=True)
    R = np.empty((3, 3))
    R[0] = (1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y))
    R[1] = (2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x))
    R[2] = (2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y))
    return R


def camera_from_pose(intrinsics: dict, translation, quaternion_xyzw, path="<pose>") -> Camera:
    """Camera of a world-from-camera pose row (formats.py:278-289)."""
    q = np.asarray(quaternion_xyzw, dtype=float)
    qn = np.linalg.norm(q)
    if abs(qn - 1.0) > 1e-3:
        raise ParseError(path, "pose", f"quaternion norm {qn:.3f} too far from 1")
    q = q / qn
    r_wc = _rotation_of(np.array([q[3], q[0], q[1], q[2]]))
    return Camera(rotation=r_wc.T, translation=-r_wc.T @ np.asarray(translation, dtype=float),
                  **intrinsics)


def read_image(path) -> np.ndarray:
    """(H, W, 3) float image in [0, 1] from an 8-bit PNG or P6 PPM (formats.py:213-240)."""
    path = Path(path)
    if path.suffix.lower() == ".ppm":
        data = path.read_bytes()
        try:
            magic, dims, maxval, payload = data.split(b"\n", 3)
            if magic != b"P6":
                raise ParseError(path, "byte 0", "not a P6 ppm")
            w, h = (int(v) for v in dims.split())
            if int(maxval) != 255:
                raise ParseError(path, "header", "only maxval 255 supported")
        except (ValueError, IndexError) as exc:
            raise ParseError(path, "header", f"bad ppm header: {exc}") from exc
        if len(payload) < w * h * 3:
            raise ParseError(path, f"byte {len(data)}", "ppm payload truncated")
        return np.frombuffer(payload[:w * h * 3], dtype=np.uint8).reshape(h, w, 3) / 255.0
    from PIL import Image
    with Image.open(path) as im:
        return np.asarray(im.convert("RGB"), dtype=np.uint8) / 255.0


def _scene(directory: Path):
    cfg = directory / "scene.cfg"
    if not cfg.exists():
        raise ParseError(cfg, "file", "stream directory lacks scene.cfg")
    intr = None
    for lineno, key, value in read_config_pairs(cfg):
        if key != "camera":
            continue
        tok = value.split()
        if len(tok) != 6:
            raise ParseError(cfg, f"line {lineno}", "camera needs fx fy cx cy width height")
        intr = dict(fx=float(tok[0]), fy=float(tok[1]), cx=float(tok[2]), cy=float(tok[3]),
                    width=int(tok[4]), height=int(tok[5]))
    if intr is None:
        raise ParseError(cfg, "end of file", "scene.cfg lacks a camera line")
    return intr


def _frame_files(directory: Path, i: int):
    ply, png = directory / f"{i:06d}.ply", directory / f"{i:06d}.png"
    if not ply.exists():
        raise ParseError(ply, "file", "stream frame missing its point cloud")
    if not png.exists():
        raise ParseError(png, "file", "stream frame missing its image")
    return ply, png


def read_stream(directory) -> list:
    """FrameSamples of a stream directory (formats.py:378-409), PLYs decoded on
    the device (`formats.read_ply`)."""
    directory = Path(directory)
    intr = _scene(directory)
    traj = directory / "trajectory.txt"
    frames = []
    for i, (ts, t, q) in enumerate(read_trajectory(traj)):
        ply, png = _frame_files(directory, i)
        cam = camera_from_pose(intr, t, q, path=traj)
        frames.append(FrameSample(timestamp=ts, points=read_ply(ply), image=read_image(png),
                                  camera=cam))
    return frames


def stream_frames(directory):
    """Frames of a stream directory for `MappingEngine.ingest_stream`: (PLY
    records in pinned memory, None, Camera, pinned float64 image), lazily, so
    the host parses frame k+1 while the device maps frame k."""
    import torch
    directory = Path(directory)
    intr = _scene(directory)
    traj = directory / "trajectory.txt"
    for i, (ts, t, q) in enumerate(read_trajectory(traj)):
        ply, png = _frame_files(directory, i)
        cam = camera_from_pose(intr, t, q, path=traj)
        img = read_image(png)
        if img.shape != (cam.height, cam.width, 3):
            from .errors import VoxsplatError
            raise VoxsplatError("frame image does not match camera dimensions")
        yield (read_ply_payload(ply), None, cam, torch.from_numpy(img).pin_memory())
