"""B200-native voxel-GPR mapping hot path of GS-LIVM (arXiv 2410.17084).

Drop-in for the reference package `voxsplat`'s mapping path
(`voxel_map`, `gpr`, `splat_init`, plus `PipelineConfig`, `Camera` and the
error types) and its consumer `renderer`: same names and signatures, with the arithmetic in hand-written
FP64 sm_100a CUDA kernels behind the C ABI of `include/voxgpr.h`
(`_lib/libvoxgpr.so`, loaded through `_native`).  There is no CPU path.
"""

from .camera import Camera, relative_transform, same_view
from .config import PipelineConfig
from .engine import IngestReport, MappingEngine
from .errors import (ContractViolationError, DegenerateGeometryError, InputDomainError,
                     NumericalDegeneracyError, ParseError, VoxsplatError)
from .gpr import (AxisSelection, GprBatchResult, GprProblem, GprResult, densify_device,
                  densify_frame, gpr_solve, gpr_solve_batch, kernel_matrix, make_mesh_grid,
                  select_value_axis)
from .splat_init import (GaussianMap, GaussianPrimitive, Subgrid, init_color, init_covariance,
                         init_gaussians_batch, init_gaussians_for_voxel, init_position,
                         partition_subgrids)
from . import formats, renderer, stream
from .renderer import RenderBuffers, SplatProjection, project_gaussian, project_points, render
from .voxel_map import (ColoredPoint, FrameUpdateSet, PointCloud, VoxelCell, VoxelKey, VoxelMap,
                        VoxelPrediction, VoxelState, classify_voxel, update_voxel_variances,
                        voxel_key)

__version__ = "0.1.0"

__all__ = [
    "Camera", "same_view", "relative_transform", "PipelineConfig", "MappingEngine",
    "IngestReport", "VoxsplatError", "InputDomainError", "DegenerateGeometryError",
    "NumericalDegeneracyError", "ContractViolationError", "ParseError",
    "AxisSelection", "GprBatchResult", "GprProblem", "GprResult", "densify_frame",
    "densify_device", "gpr_solve", "gpr_solve_batch", "kernel_matrix", "make_mesh_grid",
    "select_value_axis",
    "GaussianMap", "GaussianPrimitive", "Subgrid", "init_color", "init_covariance",
    "init_gaussians_batch", "init_gaussians_for_voxel", "init_position", "partition_subgrids",
    "ColoredPoint", "FrameUpdateSet", "PointCloud", "VoxelCell", "VoxelKey", "VoxelMap",
    "VoxelPrediction", "VoxelState", "classify_voxel", "update_voxel_variances", "voxel_key",
    "formats", "stream", "renderer", "render", "project_points", "project_gaussian", "SplatProjection",
    "RenderBuffers",
]
