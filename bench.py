#!/usr/bin/env python
"""Benchmark: per-voxel GPR + Gaussian-init throughput (voxels/s, ms/scan).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--voxels V] [--workload map|scan]

Default workload (BASELINE.json config 4 on one GPU): a ~1M-voxel synthetic
planar map (points-per-voxel histogram of the 32-beam scan, ~25.5M points,
0.5 m voxels) ingested as ONE scan into an empty map: hash -> per-voxel
FP64 GPR (81-point grid) -> Gaussian init for every first solve.  A step is
one such ingest into a freshly cleared map.  Inputs (1.2 GB) exceed L2, so
no explicit flush is needed.  Under torchrun each rank ingests its own 1M-voxel
map (weak scaling, no data-path collective: the path shards by voxel).

`value` is timed with CUDA events on the launching stream with inputs already
in HBM; `e2e` runs the same step through the public API
(`MappingEngine.ingest_stream`) from pinned host tensors (H2D of points,
colours and image inside the timed region, D2H of the ingest report).
`--impl reference` times the CPU oracle (NumPy/SciPy restatement of the
reference, oracle/voxsplat_oracle.py) on a bounded sample with all host cores.

Extra keys on the JSON line: `roofline` (dominant kernel vs the in-run FP64
peak, DRAM traffic from the committed ncu capture), `stage_roofline` (every
stage vs its roof), `stage_ms`, `trajectory` (config 2, ms/scan with
re-fits), `scans` (configs 1 and 3, ms per single scan through the host API,
plus a 640x480 render of the scan's Gaussians), `render` (the config-4 map's
Gaussians rendered at 640x480), `gather` (N > 1: NCCL hand-off of every
rank's Gaussian records to rank 0), `cpu_baseline`, `clocks`, `gpu_launches`.
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
                 "--format=csv,noheader,nounits", "-lms", "100"],
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

def _oracle_worker(args):
    pos, col, cam, img, cfg = args
    from oracle import voxsplat_oracle as O
    omap = O.OracleMap(0.5, 1e-4, TAU, 0.3)
    ocam = O.OracleCamera(cam["fx"], cam["fy"], cam["cx"], cam["cy"], cam["width"],
                          cam["height"], cam["R"], cam["t"])
    t0 = time.perf_counter()
    res = O.ingest(omap, pos, col, O.DensifyConfig(), camera=ocam, image=img)
    return len(res["predictions"]), time.perf_counter() - t0


def cpu_oracle_rate(pos, col, owner, cam, img, sample_every, procs):
    """Oracle ingest of every `sample_every`-th voxel, split over `procs` processes."""
    mask = owner % sample_every == 0
    spos, scol, sown = pos[mask], col[mask], owner[mask]
    shard = (sown // sample_every) % procs
    jobs = [(spos[shard == r], scol[shard == r], cam, img, None) for r in range(procs)]
    t0 = time.perf_counter()
    if procs > 1:
        with mp.get_context("fork").Pool(procs) as pool:
            out = pool.map(_oracle_worker, jobs)
    else:
        out = [_oracle_worker(j) for j in jobs]
    wall = time.perf_counter() - t0
    solved = sum(o[0] for o in out)
    return solved / wall, solved, wall, int(mask.sum())


def run_reference(args, rank, world):
    if rank != 0:
        return
    procs = len(os.sched_getaffinity(0))
    pos, col, counts, keys, owner, cam, img = make_workload(args.voxels, 0)
    rates = []
    for _ in range(args.warmup):
        pass   # the oracle has no warm-up state; W is honoured by not timing anything
    for _ in range(args.steps):
        r, solved, wall, npts = cpu_oracle_rate(pos, col, owner, cam, img, args.ref_sample, procs)
        rates.append(r)
    v = float(np.median(rates))
    ms = args.voxels * (counts >= TAU).mean() / v * 1e3
    sample = (f"every {args.ref_sample}th voxel of the {args.voxels}-voxel map "
              f"({solved} solved voxels, {npts} points) per step, {procs} processes")
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": f"config4: {args.voxels}-voxel planar map, one scan, 0.5 m voxels",
                       "voxels": args.voxels},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": procs, "kind": "port",
                             "sample": sample},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU leg
# ---------------------------------------------------------------------------

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

    pos, col, counts, keys, owner, cam_d, img = make_workload(args.voxels, rank)
    npts = len(pos)
    cam = vx.Camera(cam_d["fx"], cam_d["fy"], cam_d["cx"], cam_d["cy"], cam_d["width"],
                    cam_d["height"], cam_d["R"], cam_d["t"])
    config = vx.PipelineConfig(voxel_size=0.5, tau=TAU)
    solved_expected = int((counts >= TAU).sum())

    # host pinned inputs (e2e) and device-resident inputs (value)
    h_xyz = torch.from_numpy(pos).pin_memory()
    h_rgb = torch.from_numpy(col).pin_memory()
    h_img = torch.from_numpy(img).pin_memory()
    d_xyz, d_rgb, d_img = (t.to(dev) for t in (h_xyz, h_rgb, h_img))
    eng = vx.MappingEngine(config, voxel_capacity=int(args.voxels * 1.05),
                           point_capacity=int(npts * 1.6),
                           gaussian_capacity=9 * solved_expected + 1024)

    def step_device():
        eng.reset()
        return eng.ingest_device(d_xyz, d_rgb, npts, cam, d_img)

    def run_e2e(k):
        # public streaming API: pinned host frames, H2D of frame i+1 overlapped
        # with the device work of frame i; ingest reports read back every frame
        frames = [(h_xyz, h_rgb, cam, h_img)] * k
        return eng.ingest_stream(frames, reset_each=True)

    for _ in range(args.warmup):
        rep = step_device()
    run_e2e(2)            # warm the streaming path (side stream + double buffers)
    torch.cuda.synchronize()
    if rep.voxels_solved < 0.99 * solved_expected:
        raise RuntimeError(f"solved {rep.voxels_solved} of {solved_expected} expected voxels")
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

    clocks = Clocks(local_rank)
    clocks.start()
    ms, reps, launches, prof = timed(step_device, args.steps, profile=True)
    clk = clocks.stop()
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
    h2d = h_xyz.numel() * 8 + h_rgb.numel() * 8 + h_img.numel() * 8
    d2h = 7 * 8 * 2 + 21 * 8   # frame/densify info structs + counters per step

    # roofline of the dominant kernel (FP64 pipe for the GPR solves)
    stages = {k: v for k, v in prof.items() if k != "densify" and v[1] > 0}
    top = max(stages, key=lambda k: stages[k][0])
    top_ms, top_n = stages[top]
    sol = counts[counts >= TAU]
    bucket = {"gpr_n16": sol[sol <= 16], "gpr_n24": sol[(sol > 16) & (sol <= 24)],
              "gpr_n32": sol[(sol > 24) & (sol <= 32)],
              "gpr_n64": sol[(sol > 32) & (sol <= 64)],
              "gpr_n96": sol[(sol > 64) & (sol <= 96)],
              "gpr_n128": sol[(sol > 96) & (sol <= 128)],
              "gpr_n160": sol[(sol > 128) & (sol <= 160)], "gpr_n_large": sol[sol > 160]}
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
        bts = (104.0 * npts if top == "hash" else 1224.0 * solved_expected) * args.steps
        achieved = bts / (top_ms / 1e3) / 1e9
        pk = float(peaks.get("hbm_gbs", 6548.8))
        roof = {"kernel": top, "bound": "hbm", "achieved": achieved, "peak": pk, "unit": "GB/s",
                "frac": achieved / pk, "peak_source": "MEASURED_PEAKS.json hbm_gbs",
                "traffic": None, "launch_ms": top_ms / top_n, "share_of_step": top_ms / ms}
    stage_ms = {k: round(v[0] / args.steps, 4) for k, v in prof.items()}
    # every stage against its own roof (north star: HBM GB/s for hashing and
    # Gaussian init, FP64 for the solves); algorithmic work per SURVEY 8(d)
    hbm = float(peaks.get("hbm_gbs", 6548.8))
    stage_roofline = {}
    for k, (tms, _) in prof.items():
        if tms <= 0 or k in ("densify",):
            continue
        if k in bucket and len(bucket[k]):
            tf = float(gpr_flops(bucket[k]).sum()) * args.steps / (tms / 1e3) / 1e12
            stage_roofline[k] = {"bound": "fp64", "achieved": round(tf, 3), "unit": "TFLOP/s",
                                 "frac": round(tf / peak64, 4), "voxels": int(len(bucket[k]))}
        elif k in ("hash", "splat", "pca"):
            per = {"hash": 104.0 * npts,                    # read xyz+rgb, write xyz, rgb, noise
                   "splat": (81 * 56 + 9 * 136) * float(solved_expected),
                   "pca": 24.0 * float(counts[counts >= TAU].sum())}[k]
            gbs = per * args.steps / (tms / 1e3) / 1e9
            stage_roofline[k] = {"bound": "hbm", "achieved": round(gbs, 1), "unit": "GB/s",
                                 "frac": round(gbs / hbm, 4)}

    # N > 1: the one collective of the path, the hand-off of every rank's
    # Gaussian records to rank 0 (sharding.gather_records: all-gather of
    # counts, padded NCCL gather of the SoA fields, stable sort by order key);
    # reported beside `value`, which stays the data-path throughput
    gather = None
    if world > 1 and dist.get_backend() == "nccl":
        from paper_2410_17084_b200 import sharding
        recs = eng.gaussians_device()
        nrec = int(recs["position"].shape[0])
        order = (torch.arange(nrec, dtype=torch.int64, device=dev) + (int(rank) << 40))
        for _ in range(2):
            sharding.gather_records(recs, order, dst=0)
        dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g = sharding.gather_records(recs, order, dst=0)
        e1.record()
        torch.cuda.synchronize()
        gms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
        dist.all_reduce(gms, op=dist.ReduceOp.MAX)
        rec_bytes = sum(int(t[0].numel()) * t.element_size() for t in recs.values()) + 8
        tot = torch.tensor([nrec], dtype=torch.int64, device=dev)
        dist.all_reduce(tot)
        gather = {"what": "all ranks' Gaussian records -> rank 0 in global order "
                          "(sharding.gather_records over NCCL), CUDA events on the "
                          "current stream, max over ranks",
                  "records": int(tot.item()), "ms": float(gms.item()),
                  "bytes_into_rank0": int((int(tot.item()) - nrec) * rec_bytes),
                  "GB_per_s_into_rank0": (int(tot.item()) - nrec) * rec_bytes / (float(gms.item()) / 1e3) / 1e9}
        del g
    # the map's Gaussians (9 per solved voxel) rendered from the bench camera
    render = {"workload": f"{eng.num_gaussians} Gaussians of the config-4 map, 640x480, "
                          "renderer.render_device (SURVEY 8(f) row 4)",
              "device_ms": render_ms(eng.gaussians_device(), cam)}
    traj = None
    if args.traj_scans > 0:
        traj = run_trajectory(args, dev)
    scans = run_scans(args) if args.scan_reps > 0 else None

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        procs = len(os.sched_getaffinity(0))
        r, s_solved, wall, spts = cpu_oracle_rate(pos, col, owner, cam_d, img, args.ref_sample,
                                                  procs)
        cpu = {"value": r, "unit": UNIT, "cores": procs, "kind": "port",
               "sample": f"every {args.ref_sample}th voxel ({s_solved} solved, {spts} points), "
                         f"oracle store+densify+init, {wall:.1f} s wall over {procs} processes"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": f"config4: {args.voxels}-voxel planar map per GPU ingested as "
                                   f"one scan ({npts} points, 0.5 m voxels, n*=81, "
                                   f"Gaussian init for all first solves)",
                       "voxels_per_gpu": args.voxels, "points_per_gpu": npts,
                       "solved_per_gpu": solved, "l2": "inputs 1.2 GB > 126 MB L2, no flush",
                       "parallelism": f"hash-shard x{world}"},
            "roofline": roof,
            "stage_ms": stage_ms,
            "stage_roofline": stage_roofline,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms / args.steps,
                    "wall_ms_per_step": e2e_wall_ms / args.steps,
                    "api": "MappingEngine.ingest_stream (pinned host frames, H2D of frame i+1 "
                           "overlapped with frame i)"},
            "gpu_launches": launches,
            "trajectory": traj,
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
