#!/usr/bin/env python
"""Benchmark of the kriging interpolation path (interpolated voxels/s).

Workload (BASELINE.json configs[3], the configuration the metric is quoted on
"at 1/2/4/8 B200"): the C4 high-dynamic-range spine phantom, 512x512 12-bit
slices, K = 256 known slices per GPU, upsampling factor 8 (7 missing planes
per gap), 32 Z sub-parts per GPU, reference defaults (exponential variogram,
linear drift, fp64, no variance).  A step is one pass of the whole kriging
path over the resident stack: plane stats -> pair draw -> binned
semivariogram -> TRF fit -> 112 stencil solves per part -> streaming
prediction of 467,927,040 voxels (per GPU), run as the library's default
schedule: 32 per-part fit -> solve -> predict chains on side streams, so parts
whose fit converges early stream their planes while other fits still iterate
(``--serial``: one launch per stage; per-stage times always come from a
serial-schedule pass).  Scaling is weak: under torchrun
every rank owns its own 256-slice stack and receives a one-slice halo from
the next rank over NCCL inside the timed step.

``--impl reference`` times the reference on the host cores instead: the
unmodified volkrig ``fit_variogram`` + ``fill_missing`` per Z sub-part from
the git-ignored ``baseline/_ref`` install (``tools/vendor_ref.py``), a process
pool over sub-parts, a bounded sample of the same workload per step; without
that install it falls back to the oracle port and labels the line "port".
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

# one hardware work queue per part chain (the default schedule runs S = 32
# fit -> solve -> predict chains on side streams); must precede CUDA init
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "interpolated voxels/sec (kriging path)"
UNIT = "voxel/s"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), float(d.get("sm_max_mhz", 1965.0)), "measured"
    except Exception:
        return 6650.0, 1965.0, "fallback"


# arithmetic the prediction stencil runs in (solves and fits are fp64 always)
DTYPES = {"fp64": "f64", "fp32": "f32",
          "fixed": "u8xs8->s32 (24-bit fixed-point values x 32-bit fixed-point weights, exact)"}


def _profile_traffic(name: str):
    """dram bytes per launch of the prediction kernel from the committed ncu
    summary (profiles/*.json), or None."""
    path = os.path.join(ROOT, "profiles", "predict_traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d.get(name)
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi sampling during the timed region (clocks + throttle)."""

    Q = ("timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        self.t0 = self.t1 = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
                out = ""
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def mark(self, start: bool):
        """Wall-clock bounds of the timed region (samples are filtered to it)."""
        if start:
            self.t0 = time.time()
        else:
            self.t1 = time.time()

    def summary(self):
        import datetime
        rows = []
        for ln in getattr(self, "lines", []):
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                ts = datetime.datetime.strptime(parts[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                rows.append((ts, float(parts[1]), float(parts[2]), float(parts[3]), parts[4:8]))
            except ValueError:
                continue
        if self.t0 is not None and self.t1 is not None and rows:
            inside = [r for r in rows if self.t0 - 0.03 <= r[0] <= self.t1 + 0.03]
            if not inside:                    # region shorter than the sampling period
                inside = sorted(rows, key=lambda r: abs(r[0] - 0.5 * (self.t0 + self.t1)))[:2]
            rows = inside
        rows = [r[1:] for r in rows]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i, v in enumerate(r[3]) if v.lower() == "active"})
        return {"sm_mhz": float(np.median([r[0] for r in rows])), "sm_max_mhz": rows[0][1],
                "power_w_max": max(r[2] for r in rows), "reasons": reasons, "samples": len(rows)}


# --------------------------------------------------------------------------
# CPU reference arm: the unmodified reference (volkrig, installed into the
# git-ignored baseline/_ref by tools/vendor_ref.py) when it is there, else the
# oracle port of its algorithm (labelled "port")
# --------------------------------------------------------------------------

REF_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "baseline", "_ref")


def cpu_kind() -> str:
    """"reference" when the vendored volkrig is present, else "port"."""
    return "reference" if os.path.isfile(os.path.join(REF_DIR, "volkrig", "kriging.py")) else "port"


def _cpu_worker(args):
    os.environ["OMP_NUM_THREADS"] = "1"
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    slices, b, e, factor, drift = args
    if cpu_kind() == "reference":
        # what the reference's reconstruct_block does per Z sub-part
        # (SPEC.md:401-404): fit_variogram on the known voxels, fill_missing
        if REF_DIR not in sys.path:
            sys.path.insert(0, REF_DIR)
        from volkrig.kriging import fill_missing, fit_variogram
        from volkrig.model import VolumeGrid
        nk = e - b + 1
        data = np.full(((nk - 1) * factor + 1,) + slices.shape[1:], np.nan, dtype=np.float32)
        data[::factor] = slices[b:e + 1]
        grid = VolumeGrid(data)
        kz, ky, kx = np.nonzero(~grid.missing_mask)
        coords = np.column_stack([kx, ky, kz]).astype(np.float64)
        model = fit_variogram((coords, data[kz, ky, kx].astype(np.float64)))
        out = fill_missing(grid, model, drift=drift)
        return out.data.shape[0]
    from oracle import kriging_oracle as O
    out, _, _ = O.reconstruct_zpart(slices, b, e, factor, drift=drift)
    return out.shape[0]


def _subpart_ranges(k, n_parts):
    """Equal Z sub-parts of k known slices, each with its trailing halo slice
    (the reference's split; same as zshard / the oracle)."""
    from paper_2303_09523_b200.block_pipeline import subpart_ranges
    return subpart_ranges(k, n_parts)


def cpu_reference_sample(ks, factor, n_parts, cores, pool=None, n_sample=None, drift="linear"):
    """Run the reference (or its port) on a bounded sample of sub-parts with a
    process pool; returns (voxels, seconds, sample description)."""
    ranges = _subpart_ranges(ks.shape[0], n_parts)
    n_sample = n_sample or min(len(ranges), cores)
    sel = ranges[:n_sample]
    H, W = ks.shape[1:]
    vox = sum((e - b) * (factor - 1) * H * W for b, e in sel)
    jobs = [(ks[b:e + 1].copy(), 0, e - b, factor, drift) for b, e in sel]
    t0 = time.perf_counter()
    if pool is None:
        for j in jobs:
            _cpu_worker(j)
    else:
        pool.map(_cpu_worker, jobs)
    dt = time.perf_counter() - t0
    who = "volkrig fit_variogram + fill_missing" if cpu_kind() == "reference" else "oracle port"
    return vox, dt, f"{who}: {n_sample} of {n_parts} sub-parts ({vox} voxels), pool of {cores}"


def _host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def run_reference(args, cfg, ks):
    import multiprocessing as mp
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return 0
    cores = _host_cores()
    ctx = mp.get_context("fork")
    with ctx.Pool(cores) as pool:
        pool.map(_cpu_worker, [(ks[:2].copy(), 0, 1, cfg.factor, args.drift)] * cores)   # warm
        for _ in range(args.warmup):
            cpu_reference_sample(ks, cfg.factor, cfg.n_subparts, cores, pool, n_sample=min(cores, 4),
                                 drift=args.drift)
        times, vox = [], 0
        for _ in range(args.steps):
            v, dt, sample = cpu_reference_sample(ks, cfg.factor, cfg.n_subparts, cores, pool,
                                                 drift=args.drift)
            times.append(dt)
            vox = v
    ms = 1e3 * float(np.median(times))
    value = vox / (ms / 1e3)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": _data_desc(cfg),
        "config": _config(cfg, args, world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": cpu_kind(),
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def _data_desc(cfg):
    return f"synthetic (seeded {cfg.name} phantom, {cfg.quantise} values; no clinical MRI available)"


def _l2_desc(cfg):
    T = cfg.n_known + (cfg.n_known - 1) * (cfg.factor - 1)
    vin = cfg.n_known * cfg.height * cfg.width * 4 / 1e6
    vout = T * cfg.height * cfg.width * 4 / 1e6
    if vin + vout > 126:
        return (f"no flush: per-GPU inputs {vin:.0f} MB and outputs {vout:.0f} MB exceed the 126 MB L2")
    return f"inputs {vin:.0f} MB + outputs {vout:.0f} MB fit the 126 MB L2 (small config, no flush)"


def _config(cfg, args, world):
    values = ("normalised to [0, 1] (non-integer floats: the 16-tap fp64 stencil path)"
              if args.values == "normalized" else
              f"{cfg.quantise} grey levels as float32 (integer-valued: the exact-split / x<->y symmetric rows)"
              if cfg.quantise in ("u8", "u12") else "float32 in [0, 1]")
    return {"workload": f"{cfg.name} {cfg.height}x{cfg.width}, K={cfg.n_known} known slices/GPU, "
                        f"factor {cfg.factor}, {cfg.n_subparts} Z sub-parts/GPU",
            "kind": "exponential", "drift": args.drift, "accum": args.accum,
            "return_variance": bool(args.variance), "max_pairs": 100000, "seed": 0,
            "input_values": values,
            "parallelism": f"zparts x {world} GPU (weak, 1-slice NCCL halo)",
            "l2": _l2_desc(cfg),
            "pair_draws": "redrawn every step",
            "fit": "device TRF reproducing scipy's fit bit for bit (tests/test_gpu_fit_parity.py)"}


# --------------------------------------------------------------------------
# GPU arm
# --------------------------------------------------------------------------

def run_gpu(args, cfg, ks):
    import torch
    import torch.distributed as dist

    from paper_2303_09523_b200 import ZPartKriging
    from paper_2303_09523_b200.zshard import core_planes, exchange_halo

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        # communicator set-up lines on stderr (nranks / transport per rank)
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream()
    owned = torch.from_numpy(ks).to(dev)
    has_halo = rank < world - 1
    K_loc = cfg.n_known + int(has_halo)
    H, W, f = cfg.height, cfg.width, cfg.factor
    zk = ZPartKriging(K_loc, H, W, f, cfg.n_subparts, accum=args.accum, drift=args.drift,
                      redraw_pairs=not os.environ.get("VK_DIAG_NO_REDRAW"),
                      part_len=cfg.n_known // cfg.n_subparts, overlap=not args.serial)
    # per-stage / per-kernel times come from the serial schedule (one launch
    # per stage on one stream); the default chained schedule interleaves them
    zs = zk if args.serial else ZPartKriging(K_loc, H, W, f, cfg.n_subparts, accum=args.accum,
                                             drift=args.drift, redraw_pairs=True,
                                             part_len=cfg.n_known // cfg.n_subparts, overlap=False)
    zs.plan.set_timing(max(1, args.steps))
    stack = torch.empty((K_loc, H, W), dtype=torch.float32, device=dev)
    stack[:cfg.n_known].copy_(owned)
    out, var = zk.allocate(bool(args.variance))
    vox_local = zk.interpolated_voxels
    kernels = zk.plan.info

    def step():
        if world > 1:
            # the next rank's first plane lands in the halo slot directly
            exchange_halo(stack[0], rank, world, out=stack[cfg.n_known] if has_halo else None)
        zk.run(stack, out, var)

    for _ in range(max(3, args.warmup)):
        step()
    zk.finish()
    kpe = zk.plan.info["kernels_per_execute"] + (1 if world > 1 else 0) * 0
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    pred_ms, stage_acc = [], {}
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        time.sleep(0.6)                      # nvidia-smi start-up, outside the region
        clk.mark(True)
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize()
        clk.mark(False)
    zk.finish()
    if zs is not zk:                         # serial-schedule pass for the stage times
        for _ in range(2):
            zs.run(stack, out, var)
        zs.finish()
        zs.plan.set_timing(max(1, args.steps))
        for _ in range(args.steps):
            zs.run(stack, out, var)
        zs.finish()
    for back in range(args.steps):          # per-launch stage events, read after
        st = zs.plan.stage_ms(back)
        pred_ms.append(st["predict"])
        for k2, v in st.items():
            stage_acc[k2] = stage_acc.get(k2, 0.0) + v
    serial_ms = sum(stage_acc.values()) / args.steps
    t_ms = ev0.elapsed_time(ev1)
    if world > 1:
        t = torch.tensor([t_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_ms = float(t.item())
        v = torch.tensor([float(vox_local)], device=dev, dtype=torch.float64)
        dist.all_reduce(v)
        vox_total = float(v.item())
    else:
        vox_total = float(vox_local)
    ms_step = t_ms / args.steps
    value = vox_total / (ms_step / 1e3)

    # roofline of the prediction kernel (algorithmic bytes per launch)
    hbm_peak, sm_max, peak_kind = _peaks()
    T = zk.depth
    alg_bytes = 4 * (K_loc + T) * H * W + (8 * T * H * W if args.variance else 0)
    pred_avg = float(np.mean(pred_ms))
    achieved = alg_bytes / (pred_avg / 1e3) / 1e9
    # fp64 pipe cap of the streaming kernel at the measured 58 DFMA/clk/SM
    # (tools/fp64_microbench.cu, profiles/fp64_microbench_r01.json).  FP64
    # pipe operations per voxel: integer planes below 2^22 take the x<->y
    # symmetric interior rows -- 10 DFMA + 20/G pair-sum conversions + 1
    # output conversion + 2*floor(G/2)/G mirror-pair DADDs; other data the
    # 16-tap form -- 16 DFMA + 2 DADD (S, D) + 1 + 2*floor(G/2)/G
    G = f - 1
    vmax = float(np.abs(ks).max())
    sym = bool(np.all(ks == np.rint(ks)) and vmax < 2.0 ** 22)
    # exact-split FFMA2 rows: integer planes below 2^17 whose
    # magnitude is within 4x the range -- no FP64-pipe work in interior rows;
    # per warp row step (128 G voxels) 40 G FFMA2 at two FMA-pipe cycles and
    # 104 + 4 (6 floor(G/2) + G mod 2) FADD
    split = bool(sym and args.accum == "fp64" and vmax < 2.0 ** 17
                 and vmax <= 4.0 * float(ks.max() - ks.min()))
    fp64_ops = (10 + 20 / G if sym else 18) + 1 + 2 * (G // 2) / G
    fp64_cap = 148 * 58 * sm_max * 1e6 / fp64_ops
    fma_cycles = 2 * 40 * G + 104 + 4 * (6 * (G // 2) + G % 2)
    fma_cap = 148 * 4 * sm_max * 1e6 * (128 * G) / fma_cycles
    vps = vox_local / (pred_avg / 1e3)
    roof = {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
            "frac": achieved / hbm_peak, "traffic": _profile_traffic(args.accum),
            "kernel": "predict_fast_kernel", "bytes_per_launch": alg_bytes,
            "launch_ms": pred_avg, "peak_kind": peak_kind,
            "launch_ms_from": "serial schedule, CUDA events around the streaming kernel's launch "
                              "(the stencil-table kernels close the solve stage)",
            "rows": ("exact-split FFMA2 symmetric rows" if split else
                     "x<->y symmetric DFMA rows" if sym and args.accum == "fp64" else
                     "16-tap DFMA rows" if args.accum == "fp64" else "fp32 FFMA2 rows"),
            "fma_pipe_frac": vps / fma_cap if split else None,
            "fp64_pipe_frac": vps / fp64_cap if args.accum == "fp64" and not split else None,
            "fp64_ops_per_voxel": round(fp64_ops, 3) if args.accum == "fp64" and not split else None}
    stages = {k2: v / args.steps for k2, v in stage_acc.items()}
    stages["sum_serial"] = serial_ms

    # pipelined throughput (reported beside `value`, not instead of it): two
    # independent plans alternate on two streams, so step i+1's statistics,
    # pair draw, fits and solves overlap step i's prediction -- a stream of
    # volumes as a serving pipeline runs it; every step does all of its work
    pipelined = None
    if not args.no_pipelined:
        pipelined = run_pipelined(args, cfg, stack, K_loc, rank, world, dev, stream)

    # end to end through the public API with host buffers (every rank: its
    # own slab H2D, halo exchange, kriging path, its output D2H)
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, cfg, ks, stream, rank, world, dev)

    # the reference-shaped calls a drop-in user makes (kriging.py:264, :458):
    # per sub-part, fit_variogram on the part's (coords, values) samples and
    # fill_missing on its host NaN grid -- numpy in, numpy out, every upload,
    # plan lookup and download inside the timed region; a bounded sample of
    # the step's sub-parts (the samples and grids are the caller's own data,
    # built outside the timed region)
    dropin = None
    if rank == 0 and not args.no_e2e:
        dropin = run_dropin(args, cfg, ks)

    # strong scaling: ONE volume (the base config's K slices) split over the
    # ranks by Z sub-parts, halo over the C-ABI NCCL communicator inside the
    # step; the gather of the core planes to rank 0 timed separately
    strong = None
    if world > 1 or args.scaling == "strong":
        strong = run_strong(args, rank, world, dev, stream)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import multiprocessing as mp
        cores = _host_cores()
        with mp.get_context("fork").Pool(cores) as pool:
            pool.map(_cpu_worker, [(ks[:2].copy(), 0, 1, cfg.factor, args.drift)] * cores)
            v, dt, sample = cpu_reference_sample(ks, cfg.factor, cfg.n_subparts, cores, pool,
                                                 drift=args.drift)
        cpu = {"value": v / dt, "unit": UNIT, "cores": cores, "kind": cpu_kind(), "sample": sample}

    scaling = "weak"
    if args.scaling == "strong":
        scaling, value, ms_step = "strong", strong["value"], strong["ms_per_step"]
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None,
            "dtype": DTYPES[args.accum],
            "data": _data_desc(cfg),
            "config": _config(cfg, args, world),
            "schedule": "serial" if args.serial else "per-part fit->solve->predict chains",
            "roofline": roof, "stage_ms_serial": stages, "cpu_baseline": cpu, "e2e": e2e,
            "pipelined": pipelined, "dropin_e2e": dropin, "strong": strong,
            "gpu_launches": kpe * args.steps, "clocks": clk.summary(),
        }
        if scaling == "strong":
            line["config"]["parallelism"] = (f"one {cfg.n_known}-slice volume split over {world} GPU by Z "
                                             f"sub-parts (strong, 1-slice NCCL halo)")
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def run_strong(args, rank, world, dev, stream):
    """Strong scaling of the same metric: the base config's stack split by Z
    sub-parts (zshard.strong_shard: rank r owns parts [r S/N, (r+1) S/N) and
    receives the next rank's first slice), the halo exchanged on the plan's
    stream through the C ABI's NCCL communicator (vk_halo_exchange) inside
    every timed step.  Device time per step, max over ranks; the gather of
    every rank's core planes to rank 0 (vk_gather_core) is timed on its own."""
    import torch
    import torch.distributed as dist
    from paper_2303_09523_b200 import ZPartKriging
    from paper_2303_09523_b200.phantoms import CONFIGS, phantom_planes
    from paper_2303_09523_b200.zshard import NativeComm, core_planes, strong_shard
    base = CONFIGS[args.config]
    K, H, W, f, S = base.n_known, base.height, base.width, base.factor, base.n_subparts
    sh = strong_shard(K, S, rank, world)
    own = sh.k1 - sh.k0 + 1
    stack = torch.empty((sh.n_local, H, W), dtype=torch.float32, device=dev)
    stack[:own].copy_(torch.from_numpy(_values(args, base, phantom_planes(base, base.known_z[sh.k0:sh.k1 + 1]))))
    comm = NativeComm(rank, world) if world > 1 else None
    zk = ZPartKriging(sh.n_local, H, W, f, sh.n_parts, accum=args.accum, drift=args.drift,
                      redraw_pairs=True, part_len=sh.part_len)
    out, var = zk.allocate(bool(args.variance))

    def step():
        if comm is not None:
            comm.halo(stack[0], out=stack[own] if sh.has_halo else None, stream=stream)
        zk.run(stack, out, var)

    for _ in range(max(3, args.warmup)):
        step()
    zk.finish()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    zk.finish()
    ms = e0.elapsed_time(e1) / args.steps
    core = core_planes(out, f, sh.has_halo).reshape(-1)
    gather_ms = None
    if comm is not None:
        counts = [None] * world
        dist.all_gather_object(counts, int(core.numel()))
        comm.gather(core, counts, stream=stream)               # warm
        torch.cuda.synchronize()
        dist.barrier()
        e0.record(stream)
        comm.gather(core, counts, stream=stream)
        e1.record(stream)
        torch.cuda.synchronize()
        gather_ms = e0.elapsed_time(e1)
        t = torch.tensor([ms, gather_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, gather_ms = float(t[0].item()), float(t[1].item())
        comm.close()
    vox = (K - 1) * (f - 1) * H * W
    res = {"value": vox / (ms / 1e3), "unit": UNIT, "ms_per_step": ms, "steps": args.steps,
           "volume": f"{base.name}: K={K}, {S} sub-parts in total, {sh.n_parts} per GPU",
           "halo": "vk_halo_exchange (C-ABI NCCL send/recv) inside the step"}
    if gather_ms is not None:
        res.update({"gather_ms": gather_ms, "gather_to_rank0_gbs": (((K - 1) * f + 1) * H * W * 4
                                                                    - int(core.numel()) * 4) / (gather_ms / 1e3) / 1e9,
                    "gather": "vk_gather_core: every rank's core planes into rank 0's volume (timed alone)"})
    return res


def _values(args, cfg, planes):
    """--values normalized: the stack rescaled to [0, 1] floats (as the
    reference pipeline's normalize_stack would feed it), which takes the
    16-tap fp64 stencil rows instead of the integer-only symmetric rows."""
    if args.values != "normalized":
        return planes
    hi = {"u8": 255.0, "u12": 4095.0}.get(cfg.quantise, 1.0)
    return (planes / np.float32(hi)).astype(np.float32)


def run_pipelined(args, cfg, stack, K_loc, rank, world, dev, stream):
    """Device throughput with consecutive steps overlapped: ``--depth`` plans
    (each with its own workspace, output volume and input copy) take steps in
    turn on their own streams, so a step's statistics, fits and solves run
    while earlier steps stream their predictions.  Device time over K steps,
    max over ranks."""
    import torch
    import torch.distributed as dist
    from paper_2303_09523_b200 import ZPartKriging
    H, W, f = cfg.height, cfg.width, cfg.factor
    depth = max(1, args.depth)
    streams = [torch.cuda.Stream(device=dev) for _ in range(depth)]
    plans = [ZPartKriging(K_loc, H, W, f, cfg.n_subparts, accum=args.accum, drift=args.drift,
                          redraw_pairs=True, part_len=cfg.n_known // cfg.n_subparts,
                          overlap=args.pipe_chains) for _ in range(depth)]
    stacks = [stack.clone() for _ in range(depth)]
    outs = [p.allocate(bool(args.variance)) for p in plans]
    ev_start = torch.cuda.Event()

    def step(i):
        b = i % depth
        with torch.cuda.stream(streams[b]):
            plans[b].run(stacks[b], *outs[b])

    for i in range(2 * depth):
        step(i)
    torch.cuda.synchronize()
    for p in plans:
        p.finish()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0.record(stream)
    ev_start.record(stream)
    for st in streams:
        st.wait_event(ev_start)
    for i in range(args.steps):
        step(i)
    for st in streams:
        ev = torch.cuda.Event()
        ev.record(st)
        stream.wait_event(ev)
    e1.record(stream)
    torch.cuda.synchronize()
    for p in plans:
        p.finish()
    ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    vox = float(plans[0].interpolated_voxels) * world
    return {"value": vox / (ms / 1e3), "unit": UNIT, "ms_per_step": ms, "steps": args.steps,
            "depth": depth, "plan_schedule": "per-part chains" if args.pipe_chains else "stage order",
            "scheme": f"{depth} plans x {depth} streams in turn: a step's stats/pairs/bins/fits/solves "
                      "overlap earlier steps' predictions; every step runs the whole path "
                      "(no halo exchange in this loop)"}


def run_dropin(args, cfg, ks, n_sample=4, reps=2):
    """Reference-shaped drop-in calls on host numpy grids (see run_gpu)."""
    import torch
    from paper_2303_09523_b200 import VolumeGrid, fill_missing, fit_variogram
    from paper_2303_09523_b200.block_pipeline import subpart_ranges
    planes = _values(args, cfg, ks)
    ranges = subpart_ranges(cfg.n_known, cfg.n_subparts, cfg.n_known // cfg.n_subparts)
    pick = ranges[:: max(1, len(ranges) // n_sample)][:n_sample]
    inputs = []
    for (b, e) in pick:
        # the caller's data: the part's NaN grid (known slice i at z = (i - b) f)
        # and its known voxels in np.nonzero order as (x, y, z) samples
        data = np.full(((e - b) * cfg.factor + 1, cfg.height, cfg.width), np.nan, dtype=np.float32)
        data[::cfg.factor] = planes[b:e + 1]
        mask = np.isnan(data)
        kz, ky, kx = np.nonzero(~mask)
        samples = (np.column_stack([kx, ky, kz]).astype(np.float64), data[kz, ky, kx].astype(np.float64))
        inputs.append((VolumeGrid(data, mask), samples))
    vox = sum(int(g.missing_mask.sum()) for g, _ in inputs)
    g0, smp0 = inputs[0]
    out = None
    for _ in range(2):                         # plan cache, scratch, and the pinned host blocks
        for g, smp in inputs:                  # of the steady state (the previous result is still
            out = fill_missing(g, fit_variogram(smp, "exponential"), args.drift)   # held): warm
    torch.cuda.synchronize()
    t_fit = t_fill = 0.0
    t0 = time.perf_counter()
    for _ in range(reps):
        for g, smp in inputs:
            ta = time.perf_counter()
            mdl = fit_variogram(smp, "exponential")              # returns after its device sync
            tb = time.perf_counter()
            out = fill_missing(g, mdl, args.drift)
            t_fit += tb - ta
            t_fill += time.perf_counter() - tb
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / reps
    assert out.data.dtype == np.float32
    n_calls = reps * len(inputs)
    return {"value": vox / dt, "unit": UNIT, "ms_per_part": 1e3 * dt / len(inputs),
            "fit_ms_per_part": 1e3 * t_fit / n_calls, "fill_ms_per_part": 1e3 * t_fill / n_calls,
            "parts_timed": len(inputs), "reps": reps,
            "calls": "fit_variogram((coords, values)) + fill_missing(VolumeGrid(host NaN grid), model) "
                     "per sub-part, numpy in / numpy out (host wall clock, synchronized)",
            "h2d_bytes_per_part": int(smp0[0].nbytes + smp0[1].nbytes + g0.data.nbytes + g0.missing_mask.nbytes),
            "d2h_bytes_per_part": int(g0.data.nbytes + g0.missing_mask.nbytes)}


def run_e2e(args, cfg, ks, stream, rank=0, world=1, dev=None):
    """Same metric through the public API from pinned host buffers: every
    step uploads its known slices, (exchanges the halo,) runs the kriging
    path and downloads the whole reconstructed volume.  Steps are
    double-buffered across three streams -- upload of step i+1 and download
    of step i-1 overlap step i's compute (PCIe is full duplex) -- and every
    step still moves all of its bytes.  Device time, max over ranks."""
    import torch
    import torch.distributed as dist
    from paper_2303_09523_b200 import ZPartKriging
    from paper_2303_09523_b200.zshard import exchange_halo
    H, W = cfg.height, cfg.width
    K = cfg.n_known
    has_halo = rank < world - 1
    K_loc = K + int(has_halo)
    # host input per buffer: the K known slices plus, on a rank with a halo,
    # the next rank's first slice (downloaded each step, 1 plane), so the
    # download can take every known plane of the output from host memory
    host_in = [torch.empty((K_loc, H, W), dtype=torch.float32).pin_memory() for _ in range(2)]
    for h in host_in:
        h[:K].copy_(torch.from_numpy(ks))
    zk1 = ZPartKriging(K_loc, H, W, cfg.factor, cfg.n_subparts, accum=args.accum, drift=args.drift,
                       redraw_pairs=True, part_len=K // cfg.n_subparts)
    dev_in = [torch.empty((K_loc, H, W), dtype=torch.float32, device=dev or "cuda") for _ in range(2)]
    bufs = [zk1.allocate(bool(args.variance)) for _ in range(2)]
    host_out = [torch.empty(bufs[0][0].shape, dtype=torch.float32).pin_memory() for _ in range(2)]
    host_var = ([torch.empty(bufs[0][1].shape, dtype=torch.float64).pin_memory() for _ in range(2)]
                if args.variance else [None, None])
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
    ev_in = [torch.cuda.Event() for _ in range(2)]
    ev_done = [torch.cuda.Event() for _ in range(2)]
    ev_out = [torch.cuda.Event() for _ in range(2)]
    for e in ev_done + ev_out:
        e.record(stream)

    def step(i):
        b = i % 2
        with torch.cuda.stream(s_in):                  # upload (input buffer free after step i-2)
            s_in.wait_event(ev_done[b])
            dev_in[b][:K].copy_(host_in[b][:K], non_blocking=True)
            ev_in[b].record(s_in)
        stream.wait_event(ev_in[b])
        stream.wait_event(ev_out[b])                   # output buffer downloaded (step i-2)
        if world > 1:
            exchange_halo(dev_in[b][0], rank, world, out=dev_in[b][K] if has_halo else None)
        out, var = bufs[b]
        zk1.run(dev_in[b], out, var)
        ev_done[b].record(stream)
        with torch.cuda.stream(s_out):                 # download
            s_out.wait_event(ev_done[b])
            if has_halo:
                host_in[b][K].copy_(dev_in[b][K], non_blocking=True)
            # interpolated planes from the device, known planes from host_in
            zk1.download(out, host_in[b], host_out[b], stream=s_out)
            if var is not None:
                host_var[b].copy_(var, non_blocking=True)
            ev_out[b].record(s_out)

    for i in range(2):
        step(i)
    torch.cuda.synchronize()
    zk1.finish()
    steps = max(2, min(args.steps, 12))        # pipeline fill: ~6 ms once, ~35 ms per step
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0.record(stream)
    for i in range(steps):
        step(i)
    for e in ev_out:                                   # region ends when the last download lands
        stream.wait_event(e)
    e1.record(stream)
    torch.cuda.synchronize()
    zk1.finish()
    ms = e0.elapsed_time(e1) / steps
    vox = float(zk1.interpolated_voxels)
    if world > 1:
        t = torch.tensor([ms, vox], device=dev, dtype=torch.float64)
        tm = t[:1].clone()
        dist.all_reduce(tm, op=dist.ReduceOp.MAX)
        tv = t[1:].clone()
        dist.all_reduce(tv)
        ms, vox = float(tm.item()), float(tv.item())
    out, var = bufs[0]
    d2h = (out.numel() - K_loc * H * W) * 4 + int(has_halo) * H * W * 4
    d2h += var.numel() * 8 if var is not None else 0
    # the leg's bound: device-to-host PCIe, measured here with one pinned
    # 512 MiB copy (best of 3, CUDA events)
    probe_d = out.view(-1)[:128 << 20]
    probe_h = host_out[0].view(-1)[:128 << 20]
    best = float("inf")
    for _ in range(3):
        e0.record(s_out)
        with torch.cuda.stream(s_out):
            probe_h.copy_(probe_d, non_blocking=True)
        e1.record(s_out)
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    link = probe_d.numel() * 4 / (best / 1e3) / 1e9
    return {"value": vox / (ms / 1e3), "unit": UNIT,
            "h2d_bytes_per_step": K * H * W * 4, "d2h_bytes_per_step": d2h,
            "host_copy_bytes_per_step": K_loc * H * W * 4,
            "ms_per_step": ms, "steps": steps, "per_rank_bytes": True,
            "pipelining": "double-buffered: upload i+1 / compute i / download i-1 on 3 streams",
            "download": "vk_plan_download: interpolated planes device-to-host (one strided copy), "
                        "known planes host-to-host from the step's input (bit-identical to the device copies)",
            "roofline": {"bound": "pcie_d2h", "achieved": d2h / (ms / 1e3) / 1e9, "peak": link, "unit": "GB/s",
                         "frac": d2h / (ms / 1e3) / 1e9 / link,
                         "peak_kind": "measured in this run: pinned 512 MiB device-to-host copy"}}


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="C4")
    ap.add_argument("--accum", default="fp64", choices=["fp64", "fp32", "fixed"])
    ap.add_argument("--variance", action="store_true")
    ap.add_argument("--drift", default="linear", choices=["linear", "constant"])
    ap.add_argument("--values", default="native", choices=["native", "normalized"],
                    help="normalized: the stack rescaled to [0, 1] (non-integer input)")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak (default): every GPU owns a C4-sized stack; strong: one stack split "
                         "over the GPUs (also reported beside the weak value when N > 1)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-pipelined", action="store_true")
    ap.add_argument("--depth", type=int, default=4, help="plans in flight for the pipelined figure")
    ap.add_argument("--pipe-chains", action="store_true",
                    help="pipelined figure with the per-part chain schedule inside each plan "
                         "(default: each plan's stages in launch order on its own stream)")
    ap.add_argument("--serial", action="store_true",
                    help="time the serial schedule (one launch per stage) instead of the "
                         "default per-part chains")
    args = ap.parse_args(argv)
    args.warmup = max(3, args.warmup)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "b200":
        return _launch_ranks(args, sys.argv[1:] if argv is None else list(argv))

    from paper_2303_09523_b200.phantoms import CONFIGS, known_slices
    import dataclasses
    base = CONFIGS[args.config]
    rank = int(os.environ.get("RANK", "0"))
    cfg = dataclasses.replace(base, seed=base.seed + 1000 * rank) if rank else base
    if args.impl == "reference":
        if rank != 0:
            return 0
        return run_reference(args, base, _values(args, base, known_slices(base)))
    return run_gpu(args, cfg, _values(args, cfg, known_slices(cfg)))


def _launch_ranks(args, argv):
    """``--gpus N`` outside torchrun: launch the N ranks here (one process per
    GPU, torch.distributed.run on 127.0.0.1), failing loudly when fewer GPUs
    are visible."""
    import socket
    import torch
    n = torch.cuda.device_count()
    if n < args.gpus:
        print(json.dumps({"error": f"--gpus {args.gpus} requested but only {n} GPU(s) visible"}), flush=True)
        return 2
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + argv
    return subprocess.call(cmd)


if __name__ == "__main__":
    sys.exit(main())
