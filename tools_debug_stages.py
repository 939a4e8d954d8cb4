import sys, time, faulthandler
faulthandler.dump_traceback_later(100, exit=True)
import numpy as np, torch, ctypes as C
sys.path.insert(0, '.')
import paper_2410_17084_b200 as vx
from paper_2410_17084_b200 import _native as N
from oracle import voxsplat_oracle as O
from workloads import scenes
def p(*a): print(*a, flush=True)
# generic problem mode
rng = np.random.default_rng(5)
n = 100
x = rng.uniform(0, 0.5, (n, 2)); f = rng.normal(0, 0.05, n); nz = np.full(n, 1e-4); xs = rng.uniform(0, 0.5, (81, 2))
try:
    r = vx.gpr_solve(vx.GprProblem(x, f, nz, xs, 1.0))
    mu, var, _ = O.posterior(x, f, nz, xs, 1.0)
    p("generic problem: max|dmu|", np.abs(r.mu_star - mu).max(), "max|dvar|", np.abs(r.sigma_star_diag - var).max())
except Exception as e:
    p("generic problem error", repr(e))
config = vx.PipelineConfig(voxel_size=0.5)
for lo, hi in ((12, 30), (40, 60), (70, 120)):
    pos, col, counts, keys, owner = scenes.planar_map(50, bins=((lo, hi),), probs=(1.0,), seed=1)
    vmap = vx.VoxelMap.from_config(config); vmap._h()
    d1, d2 = N.to_device(pos), N.to_device(col)
    info = N.VxFrameInfo()
    rc = vmap._lib.vx_map_store_frame(vmap._h(), N.ptr(d1), N.ptr(d2), len(pos), C.byref(info), N.stream_ptr())
    torch.cuda.synchronize(); p(lo, hi, "store rc", rc, info.touched)
    vmap._configure_solver(config)
    di = N.VxDensifyInfo()
    t0 = time.time()
    rc = vmap._lib.vx_map_densify(vmap._h(), C.byref(di), N.stream_ptr())
    torch.cuda.synchronize(); p(lo, hi, "densify rc", rc, N.last_error(), di.candidates, di.solved, di.degenerate, di.chol_failed, di.max_train, time.time()-t0)
