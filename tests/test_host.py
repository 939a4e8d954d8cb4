"""CPU-only checks: the C-ABI library loads and exports every declared
symbol, the package imports without a GPU, compute refuses to run on the CPU
(no fallback), and the host-side mirrors behave like the reference."""

import os
import re

import numpy as np
import pytest

import paper_2410_17084_b200 as vx
from paper_2410_17084_b200 import _native as N

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def _declared():
    txt = open(os.path.join(ROOT, "include", "voxgpr.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|const char\*)\s+(vx_\w+)\(", txt, re.M)))


def test_library_exports_every_declared_symbol():
    lib = N.load_library()
    names = _declared()
    assert len(names) >= 20
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(N.EXPORTED)
    assert lib.vx_abi_version() == 1


def test_library_built_for_sm100a():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", N.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(N.NativeUnavailable):
        vx.gpr_solve(vx.GprProblem(x=[[0, 0]], f=[1.0], noise_diag=[0.1], x_star=[[0, 0]]))
    with pytest.raises(N.NativeUnavailable):
        vx.VoxelMap(0.2, 1e-4, 10, 0.3).store_frame(
            vx.PointCloud(np.zeros((1, 3)), np.zeros((1, 3)), np.zeros(1)))


def test_error_code_mapping():
    N.load_library()
    with pytest.raises(vx.InputDomainError):
        N.check(N.VX_E_INPUT)
    with pytest.raises(vx.ContractViolationError):
        N.check(N.VX_E_CONTRACT)
    with pytest.raises(vx.InputDomainError):
        N.check(N.VX_E_RANGE)


def test_host_validation_matches_reference():
    with pytest.raises(vx.InputDomainError):
        vx.PointCloud(np.array([[np.nan, 0, 0]]), np.zeros((1, 3)), np.zeros(1))
    with pytest.raises(vx.InputDomainError):
        vx.PointCloud(np.zeros((1, 3)), np.full((1, 3), 2.0), np.zeros(1))
    with pytest.raises(vx.InputDomainError):
        vx.VoxelMap(0.0, 1e-4, 10, 0.3)
    with pytest.raises(vx.InputDomainError):
        vx.GprProblem(x=np.zeros((0, 2)), f=[], noise_diag=[], x_star=[[0, 0]])
    with pytest.raises(ValueError):
        vx.PipelineConfig(voxel_size=-1)
    with pytest.raises(ValueError):
        vx.PipelineConfig(kernel="cubic")


def test_lifecycle_rules_on_host_cells():
    cloud = vx.PointCloud(np.zeros((12, 3)), np.full((12, 3), 0.5), np.full(12, 0.01))
    cell = vx.VoxelCell(key=vx.VoxelKey(1, 2, 3), raw=cloud)
    assert vx.classify_voxel(cell, tau=10, eta=0.3) is vx.VoxelState.READY
    cell.state = vx.VoxelState.READY
    pred = vx.VoxelPrediction(vx.VoxelKey(1, 2, 3), np.zeros((9, 3)), np.full((9, 3), 0.5),
                              np.full(9, 0.05))
    vx.update_voxel_variances(cell, pred, tau=10, eta=0.3)
    assert cell.state is vx.VoxelState.CONVERGED
    bad = vx.VoxelPrediction(vx.VoxelKey(9, 9, 9), np.zeros((4, 3)), np.zeros((4, 3)),
                             np.zeros(4))
    with pytest.raises(vx.ContractViolationError):
        vx.update_voxel_variances(cell, bad, tau=10, eta=0.3)


def test_frame_update_set_semantics():
    u = vx.FrameUpdateSet([(0, 0, 0), (2, 2, 2)])
    assert len(u) == 2 and u.keys[1] == vx.VoxelKey(2, 2, 2)
    assert list(u) == [vx.VoxelKey(0, 0, 0), vx.VoxelKey(2, 2, 2)]
    v = vx.FrameUpdateSet(array=np.array([[0, 0, 0], [2, 2, 2]]))
    assert u == v


def test_gaussian_map_amortised_extend():
    g = vx.GaussianMap()
    prims = [vx.GaussianPrimitive(np.full(3, i), np.ones(3), [1, 0, 0, 0], 0.5, np.zeros(3),
                                  vx.VoxelKey(i, 0, 0)) for i in range(300)]
    for p in prims:
        g.extend([p])
    assert len(g) == 300
    back = g.primitive(123)
    np.testing.assert_array_equal(back.position, np.full(3, 123.0))
    assert back.source_key == vx.VoxelKey(123, 0, 0)
    h = g.copy()
    assert len(h) == 300 and np.array_equal(h.positions, g.positions)


def test_config_roundtrip():
    c = vx.PipelineConfig.from_mapping({"voxel_size": "0.5", "tau": "12", "kernel": "matern52"})
    assert c.voxel_size == 0.5 and c.tau == 12 and c.kernel == "matern52"
    assert any(line.startswith("voxel_size=") for line in c.to_lines())


def test_renderer_host_helpers_match_reference_semantics():
    """renderer.py host helpers (the reference exposes them, renderer.py:150-179):
    depth_order is stable with index ties; alpha_patch applies ceiling and skip;
    render() itself has no CPU path."""
    from paper_2410_17084_b200 import renderer as R
    depth = np.array([2.0, 1.0, 1.0, 3.0, 0.5])
    valid = np.array([True, True, True, False, True])
    np.testing.assert_array_equal(R.depth_order(depth, valid), [4, 1, 2, 0])
    a = R.alpha_patch(np.array([1.0, 1.0]), np.array([[0.5, 0.0], [0.0, 0.5]]), 1.0, 0, 3, 0, 3)
    assert a.max() == R.ALPHA_CEILING                       # centre clamped to 0.99
    faint = R.alpha_patch(np.array([1.0, 1.0]), np.eye(2), 0.5 / 255.0, 0, 3, 0, 3)
    assert np.all(faint == 0.0)                             # below 1/255: skipped
    g = R.gaussian_patch(np.array([0.0, 0.0]), np.eye(2), 0, 2, 0, 1)
    np.testing.assert_allclose(g, [[1.0, np.exp(-0.5)]])
    import torch
    if not torch.cuda.is_available():
        from paper_2410_17084_b200 import _native as N
        with pytest.raises(N.NativeUnavailable):
            R.render([], vx.Camera(fx=1, fy=1, cx=0, cy=0, width=4, height=4))


def test_image_for_camera_crops_and_rejects():
    """The device samples a (height, width, 3) float64 block: larger images are
    cropped to the pixels the reference indexes, smaller ones raise IndexError
    before any device read (no CPU fallback is involved: host validation only)."""
    import numpy as np
    from paper_2410_17084_b200.camera import Camera
    from paper_2410_17084_b200.splat_init import image_for_camera
    cam = Camera(fx=10.0, fy=10.0, cx=3.5, cy=2.5, width=8, height=6)
    img = np.arange(7 * 9 * 4, dtype=float).reshape(7, 9, 4)
    out = image_for_camera(cam, img)
    assert out.shape == (6, 8, 3) and out.flags.c_contiguous
    np.testing.assert_array_equal(out, img[:6, :8, :3])
    exact = np.zeros((6, 8, 3))
    assert image_for_camera(cam, exact) is exact
    for bad in (np.zeros((5, 8, 3)), np.zeros((6, 7, 3)), np.zeros((6, 8)), np.zeros((6, 8, 2))):
        try:
            image_for_camera(cam, bad)
        except IndexError:
            continue
        raise AssertionError(f"shape {bad.shape} accepted")


def test_event_log_materialises_transitions_on_read():
    """transitions / solve_log are numpy-backed read-only lists: same rows,
    order and types as the per-event objects they replace (a first solve that
    converges passes through ACTIVE, voxel_map.py:250-261)."""
    import numpy as np
    from paper_2410_17084_b200.voxel_map import StateTransition, VoxelKey, VoxelMap, VoxelState
    vm = VoxelMap(0.5, 1e-4, 10, 0.3)
    k = np.array([[1, 2, 3], [4, 5, 6], [7, 8, 9]], dtype=np.int64)
    vm._events.append(("t", 0, k, np.array([0, 0, 0]), np.array([1, 1, 1])))
    # solves: READY->ACTIVE, READY->CONVERGED (two steps), ACTIVE->ACTIVE (re-fit, none)
    vm._events.append(("s", 1, k, np.array([1, 1, 2]), np.array([2, 3, 2])))
    tr = vm.transitions
    want = [StateTransition(0, VoxelKey(1, 2, 3), VoxelState.UNREADY, VoxelState.READY),
            StateTransition(0, VoxelKey(4, 5, 6), VoxelState.UNREADY, VoxelState.READY),
            StateTransition(0, VoxelKey(7, 8, 9), VoxelState.UNREADY, VoxelState.READY),
            StateTransition(1, VoxelKey(1, 2, 3), VoxelState.READY, VoxelState.ACTIVE),
            StateTransition(1, VoxelKey(4, 5, 6), VoxelState.READY, VoxelState.ACTIVE),
            StateTransition(1, VoxelKey(4, 5, 6), VoxelState.ACTIVE, VoxelState.CONVERGED)]
    assert len(tr) == 6 and list(tr) == want and tr == want
    assert tr[-1] == want[-1] and tr[3:5] == want[3:5]
    assert type(tr[0].key) is VoxelKey and tr[0].new is VoxelState.READY
    assert list(vm.solve_log) == [(1, VoxelKey(*r)) for r in k.tolist()]
    assert vm.audit_transitions() == []
