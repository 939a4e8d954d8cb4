#!/usr/bin/env python
"""Benchmark: per-voxel GPR + Gaussian-init throughput (voxels/s, ms/scan).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--voxels V]

Default workload (BASELINE.json config 4): ONE ~1M-voxel synthetic planar map
(points-per-voxel histogram of the 32-beam scan, ~25.5M points, 0.5 m voxels)
ingested as ONE scan into an empty map: hash -> per-voxel FP64 GPR (81-point
grid) -> Gaussian init for every first solve.  A step is one such ingest into
a freshly cleared map.  Inputs (1.2 GB) exceed L2, so no explicit flush is
needed.  Under torchrun the same map is hash-sharded over the ranks
(`ShardedEngine`: every rank holds the whole scan, keeps the voxels it owns;
strong scaling, no data-path collective), and the frame's predictions and
Gaussian records are gathered to rank 0 over NCCL (`gather`, and inside `e2e`).

`value` is timed with CUDA events on the launching stream with inputs already
in HBM, max over ranks; `e2e` runs the same step through the public API
(`MappingEngine.ingest_stream(fetch_records=True)`) from pinned host tensors:
H2D of points, colours and image, and D2H of the frame's Gaussian records into
pinned host memory, both inside the timed region (`e2e_map_resident`: the
round-1 variant without the record D2H).  `--impl reference` times the CPU
oracle (NumPy/SciPy restatement of the reference, oracle/voxsplat_oracle.py)
on a bounded sample with all host cores; `cpu_baseline` is the same
measurement in a fresh subprocess.

Extra keys on the JSON line: `roofline` (dominant kernel vs the in-run FP64
peak, DRAM traffic from the committed ncu capture), `stage_roofline` (every
stage vs its roof), `stage_ms`, `tail` (config 4 with the Livox n-histogram),
`trajectory` (config 2, ms/scan with re-fits), `scans` (configs 1 and 3, ms
per single scan through the host API, plus a 640x480 render of the scan's
Gaussians), `render` (the config-4 map's Gaussians rendered at 640x480),
`gather` (N > 1), `cpu_baseline`, `clocks`, `gpu_launches`.
"""

from __future__ import annotations

import os

# The CPU legs (cpu_baseline, --impl reference) run P single-threaded oracle
# processes; a multi-threaded BLAS per process is ~8x slower on these small
# solves.  Must be set before NumPy/SciPy load OpenBLAS.
for _v in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ.setdefault(_v, "1")

import argparse
import json
import math
import multiprocessing as mp
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from workloads import scenes  # noqa: E402

METRIC = "per-voxel GPR+Gaussian-init voxels/sec; ms/scan"
UNIT = "voxels/s"
TAU = 10
NSTAR = 81


def gpr_flops(n):
    """Algorithmic FP64 flops of one solve (n* = 81)."""
    n = np.asarray(n, dtype=np.float64)
    m = NSTAR
    return n ** 3 / 3 + n * n * m + n * n + 4 * n * m + 6 * (n * (n + 1) / 2 + n * m)


# ---------------------------------------------------------------------------
# workload
# ---------------------------------------------------------------------------

def make_workload(n_voxels, rank=0, seed=0):
    side = int(math.ceil(math.sqrt(n_voxels)))
    pos, col, counts, keys, owner = scenes.planar_map(n_voxels, voxel_size=0.5, seed=seed + rank,
                                                      key_offset=(0, rank * (side + 8), 0))
    # a downward camera over the map for colour sampling
    cx = 0.25 * side
    cy = 0.5 * (rank * (side + 8) + side / 2)
    R, t = scenes.look_at((cx, cy, 150.0), (cx, cy + 1e-3, 0.0), up=(0.0, 1.0, 0.0))
    cam = dict(fx=500.0, fy=500.0, cx=319.5, cy=239.5, width=640, height=480, R=R, t=t)
    img = np.random.default_rng(seed + 99).uniform(0.0, 1.0, (480, 640, 3))
    return pos, col, counts, keys, owner, cam, img


# ---------------------------------------------------------------------------
# clocks sampler (B200_PROFILING.md clocks line)
# ---------------------------------------------------------------------------

class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.path = f"/tmp/vx_clocks_{os.getpid()}.csv"

    def start(self):
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.f.close()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            p = [x.strip() for x in line.split(",")]
            if len(p) < 9:
                continue
            try:
                sm.append(float(p[1]))
                mx = float(p[2])
            except ValueError:
                continue
            for nm, v in zip(names, p[5:9]):
                if v.lower() in ("active", "1"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU oracle leg (cpu_baseline and --impl reference)
# ---------------------------------------------------------------------------

_JOBS = []   # set before the worker pool forks: workers inherit, nothing is pickled


def _oracle_job(i):
    return _oracle_worker(_JOBS[i])


def _oracle_worker(args):
    pos, col, cam, img, cfg = args
    from oracle import voxsplat_oracle as O
    omap = O.OracleMap(0.5, 1e-4, TAU, 0.3)
    ocam = O.OracleCamera(cam["fx"], cam["fy"], cam["cx"], cam["cy"], cam["width"],
                          cam["height"], cam["R"], cam["t"])
    t0 = time.perf_counter()
    res = O.ingest(omap, pos, col, O.DensifyConfig(), camera=ocam, image=img)
    return len(res["predictions"]), time.perf_counter() - t0


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def reference_line(args, world):
    """The CPU oracle on a bounded sample of the config-4 map, all host cores.

    A step = the oracle's store_frame -> densify -> Gaussian init of every
    `ref_sample`-th voxel of the map, split over P single-BLAS-thread worker
    processes (pool started before the timed steps); `ms_per_step` is that
    measured sample step, the full-map time is extrapolated in its own field.
    """
    procs = len(os.sched_getaffinity(0))
    pos, col, counts, keys, owner, cam, img = make_workload(args.voxels, 0)
    mask = owner % args.ref_sample == 0
    spos, scol, sown = pos[mask], col[mask], owner[mask]
    shard = (sown // args.ref_sample) % procs
    _JOBS[:] = [(spos[shard == r], scol[shard == r], cam, img, None) for r in range(procs)]
    walls, rates, busy = [], [], []
    with mp.get_context("fork").Pool(procs) as pool:
        pool.map(_noop, range(procs))                 # workers up before timing
        # (no warm-up steps: the oracle keeps no state between steps)
        for _ in range(args.steps):
            t0 = time.perf_counter()
            out = pool.map(_oracle_job, range(procs), chunksize=1)
            wall = time.perf_counter() - t0
            solved = sum(o[0] for o in out)
            walls.append(wall)
            rates.append(solved / wall)
            busy.append(max(o[1] for o in out))
    v = float(np.median(rates))
    ms = float(np.median(walls)) * 1e3
    full = args.voxels * (counts >= TAU).mean()
    sample = (f"every {args.ref_sample}th voxel of the {args.voxels}-voxel map ({solved} solved "
              f"voxels, {int(mask.sum())} points) per step, {procs} worker processes "
              f"(1 BLAS thread each), {cpu_model()}")
    return {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "ms_per_step_what": "measured wall time of one sample step (the bounded sample below)",
            "ms_full_map_extrapolated": full / v * 1e3,
            "slowest_worker_ms": float(np.median(busy)) * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": f"config4: ONE {args.voxels}-voxel planar map, one scan, "
                                   "0.5 m voxels (bounded sample)", "voxels": args.voxels},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": procs, "kind": "port",
                             "sample": sample, "cpu_model": cpu_model()},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def _noop(_):
    return 0


def run_reference(args, rank, world):
    if rank != 0:
        return
    print(json.dumps(reference_line(args, world)), flush=True)


def cpu_baseline_subprocess(args):
    """cpu_baseline of the GPU line: the SAME measurement as `--impl reference`,
    run in a fresh process (no CUDA context, nothing forked from this one)."""
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
           "--warmup", "0", "--voxels", str(args.voxels), "--ref-sample", str(args.ref_sample)]
    env = {k: v for k, v in os.environ.items()
           if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    try:
        out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env)
        line = json.loads(out.stdout.strip().splitlines()[-1])
        cb = dict(line["cpu_baseline"])
        cb["sample_ms"] = line["ms_per_step"]
        return cb
    except Exception as e:   # reported, never fatal for the GPU line
        return {"value": None, "unit": UNIT, "error": f"{type(e).__name__}: {e}"}


# ---------------------------------------------------------------------------
# GPU leg
# ---------------------------------------------------------------------------

def buckets_of(sol):
    """Training-set sizes of the solved voxels per size bucket (csrc launch_voxel_solve)."""
    return {"gpr_n16": sol[sol <= 16], "gpr_n24": sol[(sol > 16) & (sol <= 24)],
            "gpr_n32": sol[(sol > 24) & (sol <= 32)],
            "gpr_n64": sol[(sol > 32) & (sol <= 64)],
            "gpr_n96": sol[(sol > 64) & (sol <= 96)],
            "gpr_n128": sol[(sol > 96) & (sol <= 128)],
            "gpr_n160": sol[(sol > 128) & (sol <= 160)], "gpr_n_large": sol[sol > 160]}


def stage_report(prof, counts, npts, steps, peak64, hbm):
    """(stage_ms, stage_roofline): every stage against its own roof (north star:
    HBM GB/s for hashing and Gaussian init, FP64 for the solves); algorithmic
    work per SURVEY 8(d)."""
    sol = counts[counts >= TAU]
    bucket = buckets_of(sol)
    stage_ms = {k: round(v[0] / steps, 4) for k, v in prof.items()}
    stage_roofline = {}
    for k, (tms, _) in prof.items():
        if tms <= 0 or k in ("densify",):
            continue
        if k in bucket and len(bucket[k]):
            tf = float(gpr_flops(bucket[k]).sum()) * steps / (tms / 1e3) / 1e12
            stage_roofline[k] = {"bound": "fp64", "achieved": round(tf, 3), "unit": "TFLOP/s",
                                 "frac": round(tf / peak64, 4), "voxels": int(len(bucket[k]))}
        elif k in ("hash", "splat", "pca"):
            per = {"hash": 104.0 * npts,                    # read xyz+rgb, write xyz, rgb, noise
                   "splat": (81 * 56 + 9 * 136) * float(len(sol)),
                   "pca": 24.0 * float(sol.sum())}[k]
            gbs = per * steps / (tms / 1e3) / 1e9
            stage_roofline[k] = {"bound": "hbm", "achieved": round(gbs, 1), "unit": "GB/s",
                                 "frac": round(gbs / hbm, 4)}
    return stage_ms, stage_roofline


def run_tail(args, peak64, hbm):
    """Config 4, tail variant: the same 1M-voxel planar map with
    the points-per-voxel histogram of the Livox-style rosette scan (config 3,
    n up to ~750), ingested as one scan; device-timed with inputs in HBM."""
    import torch
    import paper_2410_17084_b200 as vx
    from paper_2410_17084_b200 import _native as N
    pos, col, counts, keys, owner = scenes.planar_map(args.tail_voxels, voxel_size=0.5, seed=5,
                                                      bins=scenes.TAIL_BINS, probs=scenes.TAIL_PROBS)
    side = int(math.ceil(math.sqrt(args.tail_voxels)))
    R, t = scenes.look_at((0.25 * side, 0.25 * side, 150.0), (0.25 * side, 0.25 * side + 1e-3, 0.0),
                          up=(0.0, 1.0, 0.0))
    cam = vx.Camera(500.0, 500.0, 319.5, 239.5, 640, 480, R, t)
    img = torch.from_numpy(np.random.default_rng(98).uniform(0.0, 1.0, (480, 640, 3))).cuda()
    npts = len(pos)
    d_xyz, d_rgb = torch.from_numpy(pos).cuda(), torch.from_numpy(col).cuda()
    solved = int((counts >= TAU).sum())
    eng = vx.MappingEngine(vx.PipelineConfig(voxel_size=0.5, tau=TAU),
                           voxel_capacity=int(args.tail_voxels * 1.05), point_capacity=int(npts * 1.6),
                           gaussian_capacity=9 * solved + 1024)
    steps = max(1, min(args.steps, args.tail_steps))
    for _ in range(2):
        eng.reset()
        rep = eng.ingest_device(d_xyz, d_rgb, npts, cam, img)
    torch.cuda.synchronize()
    N.profile(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        eng.reset()
        rep = eng.ingest_device(d_xyz, d_rgb, npts, cam, img)
    e1.record()
    torch.cuda.synchronize()
    prof = N.profile_read()
    N.profile(False)
    ms = e0.elapsed_time(e1) / steps
    stage_ms, stage_roof = stage_report(prof, counts, npts, steps, peak64, hbm)
    sol = counts[counts >= TAU]
    flops = float(gpr_flops(sol).sum())
    gpr_ms = sum(v for k, v in stage_ms.items() if k.startswith("gpr_"))
    out = {"workload": f"config4 tail variant: {args.tail_voxels}-voxel planar map, config-3 "
                       f"(Livox rosette) points-per-voxel histogram, n {int(sol.min())}-{int(sol.max())}, "
                       f"{npts} points, one scan",
           "steps": steps, "ms_per_step": ms, "voxels_per_s": rep.voxels_solved / (ms / 1e3),
           "voxels_solved": int(rep.voxels_solved), "expected_solved": solved,
           "gpr_fp64_tflops": flops / (gpr_ms / 1e3) / 1e12 if gpr_ms else None,
           "gpr_frac_of_fp64_peak": flops / (gpr_ms / 1e3) / 1e12 / peak64 if gpr_ms else None,
           "stage_ms": stage_ms, "stage_roofline": stage_roof,
           "n_hist": {k: int(len(v)) for k, v in buckets_of(sol).items()}}
    del eng, d_xyz, d_rgb
    torch.cuda.empty_cache()
    return out


def run_trajectory(args, dev):
    """Config 2: a trajectory of 32-beam scans (pose +1 m/scan) with GPR re-fits.

    eta = 2e-5 keeps solved voxels ACTIVE so later scans re-fit them from
    raw ∪ pseudo points.  Timed through the streaming
    public API (pinned host frames, H2D overlapped), ms per scan.
    """
    import torch
    import paper_2410_17084_b200 as vx
    sc = scenes.OutdoorScene.make(0)
    frames = []
    for f in range(args.traj_scans):
        pos, col = scenes.config1_scan(seed=0, frame=f)
        pin = scenes.camera_for(f, 160, 120, 100.0)
        img = scenes.render_image(sc, pin)
        cam = vx.Camera(pin.fx, pin.fy, pin.cx, pin.cy, pin.width, pin.height, pin.R, pin.t)
        frames.append((torch.from_numpy(pos).pin_memory(), torch.from_numpy(col).pin_memory(),
                       cam, torch.from_numpy(img).pin_memory()))
    config = vx.PipelineConfig(voxel_size=0.5, eta=2e-5)
    eng = vx.MappingEngine(config)
    eng.ingest_stream(frames)                     # warm-up pass over the trajectory
    eng.reset()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    reps = eng.ingest_stream(frames)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    solved = sum(r.voxels_solved for r in reps)
    return {"workload": f"config2: {args.traj_scans} scans of the 32-beam outdoor scene, "
                        "pose +1 m/scan, eta=2e-5 (re-fits)",
            "ms_per_scan": ms / len(frames), "voxels_per_s": solved / (ms / 1e3),
            "solved_per_scan": solved / len(frames),
            "refits_per_scan": (solved - sum(r.newly_active for r in reps)) / len(frames),
            "points_per_scan": float(np.mean([len(f[0]) for f in frames]))}


def run_dropin(args):
    """The reference's own MappingPipeline.ingest_frame (pipeline.py:139-187,
    unmodified, from the pip-installed reference in baseline/_ref) driving this
    package through the INTEGRATION.md §1 module substitution, on the config-2
    trajectory; ms per scan next to MappingEngine.ingest on the same frames.
    The per-voxel Python loops of ingest_frame (state checks, expansion,
    GaussianMap.extend) are the caller's and are inside the number."""
    if not os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "voxsplat")):
        return {"unavailable": "baseline/_ref (pip-installed reference) is absent"}
    sys.path.insert(0, ROOT)
    from tests.test_integration_recipe import run_recipe
    try:
        r = run_recipe(nframes=args.traj_scans, rays=60000)
    except Exception as e:
        return {"error": f"{type(e).__name__}: {str(e)[-300:]}"}
    ms, ems = r["ms_per_frame"][2:], r["engine_ms_per_frame"][2:]
    return {"workload": f"config2: {args.traj_scans} scans of the 32-beam outdoor scene, eta=2e-5, "
                        "160x120 images",
            "api": "reference MappingPipeline.ingest_frame (baseline/_ref, unmodified) on "
                   "voxsplat.{errors,config,camera,voxel_map,gpr,splat_init,renderer} := this "
                   "package (INTEGRATION.md 1)",
            "ms_per_scan": float(np.median(ms)), "engine_ms_per_scan": float(np.median(ems)),
            "outputs_equal_engine": bool(all(r["same"].values()) and r["reps"] == r["ereps"]),
            "gaussians": r["n"]}


def render_ms(gaussians, cam, reps=10):
    """Median device time of one 640x480 render of device-resident records
    (renderer.render_device: projection, depth-ordered tile binning, blend)."""
    import torch
    from paper_2410_17084_b200 import renderer as R
    for _ in range(2):
        R.render_device(gaussians, cam)
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        R.render_device(gaussians, cam)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


def run_scans(args):
    """Configs 1 and 3: ms per single scan into an empty map, end to end.

    Each repetition resets the map and ingests one scan through the public
    host API (`MappingEngine.ingest`: copy into pinned staging, H2D of the
    points, colours and a 640x480 image, hash -> densify -> Gaussian init,
    ingest report read back), timed on the host (the call synchronises on the
    report); median of `reps` after warm-up.  These scans (50k / 34k points)
    are launch-latency bound, the reason the roofline is quoted on config 4.
    """
    import torch
    import paper_2410_17084_b200 as vx
    sc = scenes.OutdoorScene.make(0)
    pin = scenes.camera_for(0, 640, 480, 400.0)
    img = scenes.render_image(sc, pin)
    cam = vx.Camera(pin.fx, pin.fy, pin.cx, pin.cy, pin.width, pin.height, pin.R, pin.t)
    out = {}
    for name, fn, label in (("config1", scenes.config1_scan, "32-beam line-scan"),
                            ("config3", scenes.config3_scan, "Livox-style rosette")):
        pos, col = fn(seed=0, frame=0)
        eng = vx.MappingEngine(vx.PipelineConfig(voxel_size=0.5))
        times, rep = [], None
        for i in range(5 + args.scan_reps):
            eng.reset()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            rep = eng.ingest(pos, col, cam, img)
            dt = time.perf_counter() - t0
            if i >= 5:
                times.append(dt * 1e3)
        out[name] = {"workload": f"{name}: one {label} scan ({len(pos)} points, 0.5 m voxels) "
                                 f"into an empty map, H2D + ingest + report D2H",
                     "ms_per_scan": float(np.median(times)), "ms_p90": float(np.percentile(times, 90)),
                     "points": len(pos), "voxels_solved": int(rep.voxels_solved),
                     "gaussians": int(rep.primitives_added),
                     "render_640x480_device_ms": render_ms(eng.gaussians_device(), cam)}
    return out


def run_gpu(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import paper_2410_17084_b200 as vx
    from paper_2410_17084_b200 import _native as N

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    N.lib()

    pos, col, counts, keys, owner, cam_d, img = make_workload(args.voxels, 0)      # ONE map, sharded over the ranks
    npts = len(pos)
    cam = vx.Camera(cam_d["fx"], cam_d["fy"], cam_d["cx"], cam_d["cy"], cam_d["width"],
                    cam_d["height"], cam_d["R"], cam_d["t"])
    config = vx.PipelineConfig(voxel_size=0.5, tau=TAU)
    solved_expected = int((counts >= TAU).sum())

    # host pinned inputs (e2e) and device-resident inputs (value)
    h_xyz = torch.from_numpy(pos).pin_memory()
    h_rgb = torch.from_numpy(col).pin_memory()
    h_img = torch.from_numpy(img).pin_memory()
    sharded = None
    lo, hi = rank * npts // world, (rank + 1) * npts // world
    if world > 1:
        # ONE config-4 map hash-sharded over the ranks: every rank
        # holds (and H2Ds) rows [lo, hi) of the scan; ShardedEngine.ingest_sliced
        # sends each point to the rank owning its voxel (one all-to-all) and
        # the ranks store / densify / initialise the voxels they own
        h_xyz, h_rgb = h_xyz[lo:hi], h_rgb[lo:hi]
    d_xyz, d_rgb, d_img = (t.to(dev) for t in (h_xyz, h_rgb, h_img))
    if world > 1:
        from paper_2410_17084_b200 import sharding
        sharded = sharding.ShardedEngine(config, rank, world,
                                         voxel_capacity=int(args.voxels * 1.05 / world) + 4096,
                                         point_capacity=int(npts * 1.6 / world) + 65536,
                                         gaussian_capacity=9 * solved_expected // world + 65536)
        eng = sharded.engine
    else:
        eng = vx.MappingEngine(config, voxel_capacity=int(args.voxels * 1.05),
                               point_capacity=int(npts * 1.6),
                               gaussian_capacity=9 * solved_expected + 1024)

    def step_device():
        eng.reset()
        if sharded is not None:
            return sharded.ingest_sliced(d_xyz, d_rgb, hi - lo, lo, cam, d_img)
        return eng.ingest_device(d_xyz, d_rgb, npts, cam, d_img)

    sliced = (lambda dx, dc, n, c, di: sharded.ingest_sliced(dx, dc, n, lo, c, di)) \
        if sharded is not None else None

    fetched = {"records": 0, "bytes": 0}

    def got_records(rep, host):
        # the frame's Gaussian records have landed in pinned host memory
        fetched["records"] = int(host["position"].shape[0]) if host else 0
        fetched["bytes"] = sum(int(t.numel()) * t.element_size() for t in host.values())

    def run_e2e(k):
        # public streaming API: pinned host frames, H2D of frame i+1 overlapped
        # with the device work of frame i; each frame's Gaussian records D2H into
        # pinned host memory overlapped with frame i+1 (the host GaussianMap of
        # pipeline.py:161-171); N > 1: the frame's predictions + records are also
        # gathered to rank 0 over NCCL (sharding.gather_frame)
        frames = [(h_xyz, h_rgb, cam, h_img)] * k
        on_frame = (lambda rep: sharded.gather_frame(dst=0)) if sharded is not None else None
        return eng.ingest_stream(frames, reset_each=True, on_frame=on_frame,
                                 fetch_records=True, on_records=got_records, ingest_fn=sliced)

    def run_e2e_resident(k):
        # variant kept for comparison with round 1: outputs stay in HBM
        frames = [(h_xyz, h_rgb, cam, h_img)] * k
        return eng.ingest_stream(frames, reset_each=True, ingest_fn=sliced)

    for _ in range(args.warmup):
        rep = step_device()
    run_e2e(3)            # warm the streaming path (side streams + double buffers)
    run_e2e_resident(2)
    torch.cuda.synchronize()
    chk = torch.tensor([float(rep.voxels_solved)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(chk)
    if chk.item() < 0.99 * solved_expected:
        raise RuntimeError(f"solved {chk.item()} of {solved_expected} expected voxels")
    peak64 = N.fp64_peak_tflops()
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass

    def timed(fn, k, profile=False):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        if profile:
            N.profile(True)
        l0 = N.launch_count()
        s = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        reps = [fn() for _ in range(k)]
        e1.record(s)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        launches = N.launch_count() - l0
        prof = N.profile_read() if profile else None
        if profile:
            N.profile(False)
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            if profile:   # share of the dominant stage from rank 0's timers
                pass
        return float(t.item()), reps, launches, prof

    # clocks sampled over both timed regions (device steps and the e2e stream)
    clocks = Clocks(local_rank)
    clocks.start()
    time.sleep(0.3)                 # nvidia-smi up before the timed region
    ms, reps, launches, prof = timed(step_device, args.steps, profile=True)
    solved = sum(r.voxels_solved for r in reps) / args.steps
    tot_solved = torch.tensor([solved], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tot_solved)
    ms_step = ms / args.steps
    value = float(tot_solved.item()) / (ms_step / 1e3)

    t_wall = time.perf_counter()
    e2e_ms, e2e_reps, _, _ = timed(lambda: run_e2e(args.steps), 1)
    e2e_wall_ms = (time.perf_counter() - t_wall) * 1e3
    e2e_value = float(tot_solved.item()) / (e2e_ms / args.steps / 1e3)
    clk = clocks.stop()
    res_ms, _, _, _ = timed(lambda: run_e2e_resident(args.steps), 1)
    h2d = h_xyz.numel() * 8 + h_rgb.numel() * 8 + h_img.numel() * 8
    # Gaussian records of the frame (136 B each) + frame/densify info structs
    d2h = fetched["bytes"] + 7 * 8 * 2 + 21 * 8

    # roofline of the dominant kernel (FP64 pipe for the GPR solves)
    stages = {k: v for k, v in prof.items() if k != "densify" and v[1] > 0}
    top = max(stages, key=lambda k: stages[k][0])
    top_ms, top_n = stages[top]
    # this rank's share of the work (a hash-sharded map: the voxels it owns)
    counts_r, npts_r = counts, npts
    if world > 1:
        from paper_2410_17084_b200 import sharding as _sh
        counts_r = counts[_sh.owner_of(keys, world) == rank]
        npts_r = int(counts_r.sum())
    sol = counts_r[counts_r >= TAU]
    bucket = buckets_of(sol)
    if top in bucket:
        flops = float(gpr_flops(bucket[top]).sum()) * args.steps
        achieved = flops / (top_ms / 1e3) / 1e12
        # DRAM traffic per launch: bytes/voxel of this kernel from the committed
        # ncu --set full capture (tools/ncu_traffic.py) x voxels in this launch
        traffic, tnote = None, "no committed ncu capture for this kernel"
        tfile = sorted(f for f in os.listdir(os.path.join(ROOT, "profiles"))
                       if f.endswith("_traffic.json")) if os.path.isdir(
                           os.path.join(ROOT, "profiles")) else []
        if tfile:
            tj = json.load(open(os.path.join(ROOT, "profiles", tfile[-1])))
            if top in tj:
                traffic = tj[top]["bytes_per_voxel"] * len(bucket[top])
                tnote = (f"profiles/{tfile[-1]}: {tj[top]['bytes_per_voxel']:.0f} B/voxel measured "
                         f"(dram read+write) x {len(bucket[top])} voxels; algorithmic "
                         f"{56 * (float(bucket[top].mean()) + NSTAR):.0f} B/voxel")
        roof = {"kernel": top, "bound": "fp64", "achieved": achieved, "peak": peak64,
                "unit": "TFLOP/s", "frac": achieved / peak64,
                "peak_source": "measured in-run FP64 peak, max of DFMA and DMMA microbenchmarks (vx_fp64_peak)",
                "traffic": traffic, "traffic_note": tnote, "launch_ms": top_ms / top_n,
                "share_of_step": top_ms / ms}
    else:
        # hashing / splat are HBM-bound: algorithmic bytes per point = 104
        bts = (104.0 * npts_r if top == "hash" else 1224.0 * len(sol)) * args.steps
        achieved = bts / (top_ms / 1e3) / 1e9
        pk = float(peaks.get("hbm_gbs", 6548.8))
        roof = {"kernel": top, "bound": "hbm", "achieved": achieved, "peak": pk, "unit": "GB/s",
                "frac": achieved / pk, "peak_source": "MEASURED_PEAKS.json hbm_gbs",
                "traffic": None, "launch_ms": top_ms / top_n, "share_of_step": top_ms / ms}
    hbm = float(peaks.get("hbm_gbs", 6548.8))
    stage_ms, stage_roofline = stage_report(prof, counts_r, npts_r, args.steps, peak64, hbm)

    # N > 1: the one collective of the path, the hand-off of the
    # frame's predictions and Gaussian records from every shard to rank 0
    # (sharding.gather_frame: all-gather of counts, grouped NCCL send/recv
    # gather-v, stable sort by the first-touch order key); timed after a step
    gather = None
    if sharded is not None:
        step_device()
        for _ in range(2):
            sharded.gather_frame(dst=0)
        dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g = sharded.gather_frame(dst=0)
        e1.record()
        torch.cuda.synchronize()
        gms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
        dist.all_reduce(gms, op=dist.ReduceOp.MAX)
        if rank == 0:
            nb = sum(int(v.numel()) * v.element_size() for part in g.values() for v in part.values())
            gather = {"what": "frame predictions (81 x xyz, rgb, var) + Gaussian records of every "
                              "shard -> rank 0 in global first-touch order (sharding.gather_frame: "
                              "grouped NCCL send/recv gather-v + order-key sort), CUDA events, "
                              "max over ranks",
                      "voxels": int(g["predictions"]["keys"].shape[0]),
                      "records": int(g["gaussians"]["position"].shape[0]),
                      "ms": float(gms.item()), "bytes_at_rank0": nb,
                      "GB_per_s_into_rank0": nb * (world - 1) / world / (float(gms.item()) / 1e3) / 1e9}
        del g
    # the map's Gaussians (9 per solved voxel) rendered from the bench camera
    render = {"workload": f"{eng.num_gaussians} Gaussians of the config-4 map, 640x480, "
                          "renderer.render_device (SURVEY 8(f) row 4)",
              "device_ms": render_ms(eng.gaussians_device(), cam)}
    tail = run_tail(args, peak64, hbm) if (args.tail_voxels > 0 and world == 1) else None
    traj = None
    if args.traj_scans > 0:
        traj = run_trajectory(args, dev)
    scans = run_scans(args) if args.scan_reps > 0 else None
    dropin = run_dropin(args) if (args.traj_scans > 0 and rank == 0) else None

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline_subprocess(args)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": f"config4: ONE {args.voxels}-voxel planar map ingested as "
                                   f"one scan ({npts} points, 0.5 m voxels, n*=81, "
                                   f"Gaussian init for all first solves)",
                       "voxels": args.voxels, "points": npts,
                       "solved_per_step": float(tot_solved.item()),
                       "l2": (f"inputs {48 * npts / 1e9:.2f} GB > 126 MB L2, no flush"
                              if 48 * npts > 126e6 else "inputs fit in L2"),
                       "parallelism": (f"hash-shard x{world}: one map, voxels owned by "
                                       f"mix64(key) % {world}; each rank holds 1/{world} of the "
                                       f"scan and one all-to-all moves the points to their "
                                       f"owners (ShardedEngine.ingest_sliced)"
                                       if world > 1 else "single GPU")},
            "roofline": roof,
            "stage_ms": stage_ms,
            "stage_roofline": stage_roofline,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms / args.steps,
                    "wall_ms_per_step": e2e_wall_ms / args.steps,
                    "records_fetched_per_step": fetched["records"],
                    "api": "MappingEngine.ingest_stream(fetch_records=True): pinned host frames "
                           "H2D (frame i+1 overlapped with frame i), the frame's Gaussian records "
                           "D2H into pinned host memory on a third stream (overlapped with frame "
                           "i+1), ingest report read back" +
                           ("; N>1: + sharded.gather_frame to rank 0 every frame" if world > 1 else "")},
            "e2e_map_resident": {"value": float(tot_solved.item()) / (res_ms / args.steps / 1e3),
                                 "unit": UNIT, "ms_per_step": res_ms / args.steps,
                                 "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": 7 * 8 * 2 + 21 * 8,
                                 "api": "MappingEngine.ingest_stream: the round-1 e2e, outputs stay "
                                        "in HBM (only the ingest report comes back)"},
            "gpu_launches": launches,
            "tail": tail,
            "trajectory": traj,
            "dropin": dropin,
            "scans": scans,
            "render": render,
            "gather": gather,
            "clocks": clk,
            "peaks": {"fp64_tflops_measured": peak64, "hbm_gbs": peaks.get("hbm_gbs")},
        }
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--voxels", type=int, default=1_000_000)
    ap.add_argument("--ref-sample", type=int, default=16)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--traj-scans", type=int, default=20)
    ap.add_argument("--scan-reps", type=int, default=20)
    ap.add_argument("--tail-voxels", type=int, default=1_000_000)
    ap.add_argument("--tail-steps", type=int, default=3)
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        import torch
        if args.impl == "reference":
            if rank != 0:
                return
        else:
            # VX_BENCH_BACKEND=gloo: exercise the N>1 code path with several ranks
            # on one device (a functional check only; numbers need NCCL + N GPUs)
            backend = os.environ.get("VX_BENCH_BACKEND", "nccl")
            local_rank %= max(torch.cuda.device_count(), 1)
            torch.cuda.set_device(local_rank)
            if backend == "nccl":
                dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
            else:
                dist.init_process_group(backend)
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_gpu(args, rank, world, local_rank)
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
