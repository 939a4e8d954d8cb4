"""ctypes binding of libvoxgpr.so (include/voxgpr.h).

This is the reference-facing plugin boundary: every compute call of the
package goes through these C entry points into sm_100a kernels.  There is no
CPU fallback: importing the package works without a GPU (so host-side logic
can be tested), but the first call that needs the library raises
`NativeUnavailable` when the library or a CUDA device is missing.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import errors

_HERE = os.path.dirname(os.path.abspath(__file__))
# VX_LIB_PATH selects another in-tree build of the same library (A/B experiments)
LIB_PATH = os.environ.get("VX_LIB_PATH") or os.path.join(_HERE, "_lib", "libvoxgpr.so")

VX_OK, VX_E_INPUT, VX_E_CONTRACT, VX_E_CUDA, VX_E_NOMEM, VX_E_RANGE = 0, -1, -2, -3, -4, -5
VX_E_CAPACITY = -6
ST_OK, ST_DEGENERATE, ST_CHOL_FAIL = 0, 1, 2
KERNELS = {"se": 0, "matern32": 1, "matern52": 2}
ROT_IDENTITY, ROT_EIGEN = 0, 1


class NativeUnavailable(RuntimeError):
    """libvoxgpr.so or a CUDA device is missing; there is no CPU path."""


c_i64p = C.POINTER(C.c_int64)
vp = C.c_void_p


class VxGprBatch(C.Structure):
    _fields_ = [("num_problems", C.c_int64), ("d_x_off", vp), ("d_q_off", vp), ("d_x", vp),
                ("d_f", vp), ("d_noise", vp), ("d_xs", vp), ("d_lam", vp), ("jitter", C.c_double),
                ("kernel", C.c_int32), ("max_n", C.c_int32), ("max_m", C.c_int32),
                ("reserved", C.c_int32), ("d_mu", vp), ("d_var", vp), ("d_full", vp),
                ("d_full_off", vp), ("d_status", vp)]


class VxCamera(C.Structure):
    _fields_ = [("fx", C.c_double), ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("width", C.c_int32), ("height", C.c_int32), ("R", C.c_double * 9),
                ("t", C.c_double * 3)]


class VxSplatConfig(C.Structure):
    _fields_ = [("n_s", C.c_int32), ("n_r", C.c_int32), ("weight_floor", C.c_double),
                ("scale_floor", C.c_double), ("initial_opacity", C.c_double),
                ("rotation_mode", C.c_int32), ("reserved", C.c_int32)]


class VxGaussianOut(C.Structure):
    _fields_ = [("position", vp), ("scale", vp), ("rotation", vp), ("opacity", vp),
                ("color", vp), ("source_key", vp)]


class VxMapConfig(C.Structure):
    _fields_ = [("voxel_size", C.c_double), ("sensor_var", C.c_double), ("tau", C.c_int32),
                ("n_s", C.c_int32), ("n_r", C.c_int32), ("kernel", C.c_int32),
                ("eta", C.c_double), ("kernel_lambda", C.c_double), ("jitter", C.c_double),
                ("shard_rank", C.c_int32), ("shard_world", C.c_int32),
                ("voxel_capacity", C.c_int64), ("point_capacity", C.c_int64)]


class VxFrameInfo(C.Structure):
    _fields_ = [("frame_index", C.c_int64), ("points_in", C.c_int64),
                ("points_stored", C.c_int64), ("touched", C.c_int64),
                ("new_voxels", C.c_int64), ("ready_transitions", C.c_int64)]


class VxDensifyInfo(C.Structure):
    _fields_ = [("candidates", C.c_int64), ("solved", C.c_int64), ("degenerate", C.c_int64),
                ("chol_failed", C.c_int64), ("first_solves", C.c_int64),
                ("converged", C.c_int64), ("max_train", C.c_int64)]


class VxMapView(C.Structure):
    _fields_ = [("num_voxels", C.c_int64), ("keys", vp), ("state", vp), ("value_axis", vp),
                ("raw_count", vp), ("raw_offset", vp), ("pred_slot", vp), ("has_pred", vp),
                ("last_first", vp),
                ("raw_xyz", vp), ("raw_rgb", vp), ("pred_points", C.c_int64), ("pred_xyz", vp),
                ("pred_rgb", vp), ("pred_var", vp), ("frame_touched", C.c_int64),
                ("frame_voxels", vp), ("frame_state_before", vp), ("frame_state_after", vp),
                ("solve_candidates", C.c_int64), ("solve_voxels", vp), ("solve_status", vp),
                ("solve_state_before", vp), ("solve_state_after", vp), ("solved", C.c_int64),
                ("solved_voxels", vp), ("frame_index", C.c_int64)]


_SIGS = {
    "vx_abi_version": ([], C.c_int),
    "vx_last_error": ([], C.c_char_p),
    "vx_launch_count": ([], C.c_int64),
    "vx_voxel_keys": ([vp, C.c_int64, C.c_double, vp, vp], C.c_int),
    "vx_kernel_matrix": ([vp, C.c_int64, vp, C.c_int64, C.c_double, C.c_int32, vp, vp], C.c_int),
    "vx_mesh_grid": ([vp, C.c_int64, C.c_int32, C.c_int32, vp, vp], C.c_int),
    "vx_select_axis_batch": ([vp, vp, C.c_int64, vp, vp], C.c_int),
    "vx_gpr_solve_batch": ([C.POINTER(VxGprBatch), vp], C.c_int),
    "vx_subgrid_moments": ([vp, vp, C.c_int64, C.c_int32, vp, vp, vp, vp], C.c_int),
    "vx_gaussians_from_predictions": ([vp, vp, vp, vp, C.c_int64, C.c_int64,
                                       C.POINTER(VxCamera), vp, C.POINTER(VxSplatConfig),
                                       C.POINTER(VxGaussianOut), vp], C.c_int),
    "vx_init_color": ([vp, vp, C.c_int64, C.POINTER(VxCamera), vp, vp, vp], C.c_int),
    "vx_map_create": ([C.POINTER(VxMapConfig), C.POINTER(vp)], C.c_int),
    "vx_map_destroy": ([vp], C.c_int),
    "vx_map_clear": ([vp, vp], C.c_int),
    "vx_map_view": ([vp, C.POINTER(VxMapView)], C.c_int),
    "vx_map_store_frame": ([vp, vp, vp, C.c_int64, C.POINTER(VxFrameInfo), vp], C.c_int),
    "vx_map_densify": ([vp, C.POINTER(VxDensifyInfo), vp], C.c_int),
    "vx_map_init_gaussians": ([vp, vp, C.c_int64, C.POINTER(VxCamera), vp,
                               C.POINTER(VxSplatConfig), C.POINTER(VxGaussianOut), vp], C.c_int),
    "vx_map_ingest": ([vp, vp, vp, C.c_int64, C.POINTER(VxCamera), vp, C.POINTER(VxSplatConfig),
                       C.POINTER(VxGaussianOut), C.c_int64, c_i64p, C.POINTER(VxFrameInfo),
                       C.POINTER(VxDensifyInfo), vp], C.c_int),
    "vx_map_emit_first_gaussians": ([vp, C.POINTER(VxCamera), vp, C.POINTER(VxSplatConfig),
                                     C.POINTER(VxGaussianOut), C.c_int64, c_i64p, vp], C.c_int),
    "vx_map_lookup": ([vp, vp, C.c_int64, vp, vp], C.c_int),
    "vx_map_partition_by_owner": ([vp, vp, vp, C.c_int64, C.c_int64, vp, vp, vp, c_i64p, vp], C.c_int),
    "vx_map_set_frame_keys": ([vp, vp, C.c_int64, vp], C.c_int),
    "vx_map_apply_prediction": ([vp, c_i64p, vp, vp, vp, C.c_int64, C.POINTER(C.c_uint8), vp],
                                C.c_int),
    "vx_map_configure_solver": ([vp, C.c_int32, C.c_int32, C.c_double, C.c_double, C.c_int32],
                                C.c_int),
    "vx_fp64_peak": ([C.POINTER(C.c_double), vp], C.c_int),
    "vx_pack_map_records": ([C.POINTER(VxGaussianOut), C.c_int64, vp, vp], C.c_int),
    "vx_decode_ply": ([vp, C.c_int64, vp, vp, vp], C.c_int),
    "vx_project_points": ([vp, vp, vp, C.c_int64, C.POINTER(VxCamera), C.c_double, vp, vp, vp, vp,
                           vp, vp, vp], C.c_int),
    "vx_render": ([vp, vp, vp, vp, vp, C.c_int64, C.POINTER(VxCamera), C.c_double, vp, vp, vp, vp],
                  C.c_int),
    "vx_profile": ([C.c_int], C.c_int),
    "vx_profile_read": ([C.POINTER(C.c_double), C.POINTER(C.c_int64), C.c_int32], C.c_int),
}

EXPORTED = tuple(_SIGS)

_lib = None


def load_library(path: str = LIB_PATH):
    """Load libvoxgpr.so (no CUDA device needed) and bind every export."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise NativeUnavailable(
            f"{path} is missing: build it with `python -m paper_2410_17084_b200.build` "
            "(there is no CPU fallback)")
    lib = C.CDLL(path)
    for name, (args, res) in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    if lib.vx_abi_version() != 1:
        raise NativeUnavailable("libvoxgpr ABI mismatch")
    _lib = lib
    return lib


def lib():
    """The library, with a CUDA device verified; raises NativeUnavailable."""
    import torch
    if not torch.cuda.is_available():
        raise NativeUnavailable("no CUDA device: the voxel-GPR path runs only on the GPU")
    return load_library()


def last_error() -> str:
    return (_lib.vx_last_error() or b"").decode(errors="replace") if _lib else ""


def check(rc: int, what: str = "") -> None:
    """Translate a VX_E_* code into the reference exception classes."""
    if rc == VX_OK:
        return
    msg = last_error() or what
    if rc == VX_E_INPUT or rc == VX_E_RANGE:
        raise errors.InputDomainError(msg)
    if rc == VX_E_CONTRACT:
        raise errors.ContractViolationError(msg)
    if rc == VX_E_NOMEM:
        raise MemoryError(msg)
    if rc == VX_E_CAPACITY:
        raise BufferError(msg)
    raise RuntimeError(f"voxgpr CUDA failure: {msg}")


# ---------------------------------------------------------------------------
# device-memory helpers (torch owns the memory; the library sees raw pointers)
# ---------------------------------------------------------------------------

def device():
    import torch
    if not torch.cuda.is_available():
        raise NativeUnavailable("no CUDA device: the voxel-GPR path runs only on the GPU")
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr():
    import torch
    return vp(torch.cuda.current_stream().cuda_stream)


def to_device(arr, dtype=np.float64):
    """Contiguous device tensor from a host array (one H2D copy)."""
    import torch
    a = np.ascontiguousarray(np.asarray(arr, dtype=dtype))
    t = torch.from_numpy(a)
    return t.to(device(), non_blocking=False)


def empty(shape, dtype):
    import torch
    return torch.empty(shape, dtype=dtype, device=device())


def ptr(t):
    return vp(0) if t is None else vp(t.data_ptr())


class _CAI:
    """__cuda_array_interface__ wrapper to view library-owned device memory."""

    def __init__(self, p, shape, typestr):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                         "data": (int(p or 0), False), "version": 2,
                                         "strides": None}


_TYPESTR = {np.float64: "<f8", np.int64: "<i8", np.int32: "<i4", np.uint8: "|u1",
            np.int8: "|i1"}


def view_tensor(p, shape, dtype):
    """Zero-copy torch tensor over library-owned device memory (read-only use)."""
    import torch
    n = int(np.prod(shape)) if len(shape) else 1
    if n == 0 or not p:
        return torch.empty(shape, dtype=_torch_dtype(dtype), device=device())
    return torch.as_tensor(_CAI(p, shape, _TYPESTR[dtype]), device=device())


def _torch_dtype(dtype):
    import torch
    return {np.float64: torch.float64, np.int64: torch.int64, np.int32: torch.int32,
            np.uint8: torch.uint8, np.int8: torch.int8}[dtype]


def camera_struct(camera) -> VxCamera:
    c = VxCamera()
    c.fx, c.fy, c.cx, c.cy = float(camera.fx), float(camera.fy), float(camera.cx), float(camera.cy)
    c.width, c.height = int(camera.width), int(camera.height)
    R = np.asarray(camera.rotation, dtype=np.float64).reshape(9)
    t = np.asarray(camera.translation, dtype=np.float64).reshape(3)
    for i in range(9):
        c.R[i] = float(R[i])
    for i in range(3):
        c.t[i] = float(t[i])
    return c


def splat_struct(n_s, n_r, weight_floor, scale_floor, opacity, rotation="identity") -> VxSplatConfig:
    s = VxSplatConfig()
    s.n_s, s.n_r = int(n_s), int(n_r)
    s.weight_floor, s.scale_floor, s.initial_opacity = float(weight_floor), float(scale_floor), float(opacity)
    s.rotation_mode = ROT_EIGEN if rotation == "eigen" else ROT_IDENTITY
    return s


PROFILE_STAGES = ("hash", "gpr_n16", "gpr_n24", "gpr_n64", "gpr_n128", "gpr_n_large",
                  "gpr_n32", "gpr_n96", "gpr_n160", "splat", "densify", "pca")


def profile(enable: bool) -> None:
    lib().vx_profile(1 if enable else 0)


def profile_read() -> dict:
    ms = (C.c_double * 16)()
    n = (C.c_int64 * 16)()
    k = lib().vx_profile_read(ms, n, 16)
    return {PROFILE_STAGES[i]: (float(ms[i]), int(n[i])) for i in range(k)}


def fp64_peak_tflops() -> float:
    t = C.c_double(0)
    check(lib().vx_fp64_peak(C.byref(t), stream_ptr()))
    return float(t.value)


def launch_count() -> int:
    return int(_lib.vx_launch_count()) if _lib else 0
