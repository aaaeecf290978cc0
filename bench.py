#!/usr/bin/env python3
"""Benchmark: cone-beam forward + FDK back-projection GUPS at 512^3 x 720 views.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (one rank per GPU)

One step = forward projection A x of a 512^3 Shepp-Logan volume (0.5 mm) to a
720-view 1024^2 (0.6 mm) circular cone-beam sinogram, then FDK
(cosine pre-weight + shepp_logan row filter + (sid/w)^2-weighted voxel-driven
back projection + pi/V) of that sinogram.  Both operators count N_vox * V
voxel-view updates, so value = 2 * 512^3 * 720 / step time (whole job).
N > 1: views sharded for A + one NCCL all-gather of the sinogram, z-slabs
(with cropped detector row bands) for FDK -- fixed total work (strong scaling).

Prints ONE JSON line on rank 0.  Timing: CUDA events on the launching
stream, barrier + synchronize around the K timed steps, max over ranks.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

VOL = (512, 512, 512)
SPACING = (0.5, 0.5, 0.5)
DET = (1024, 1024)
DET_SP = (0.6, 0.6)
VIEWS = 720
SDD, SID = 1200.0, 750.0
STEP_SCALE = 0.5
FILTER = "shepp_logan"
WORKLOAD = ("cfg4: cone-beam circular 512^3 @0.5 mm, 720 views over 2pi, 1024^2 detector @0.6 mm, "
            "sdd 1200 / sid 750: forward projection + FDK (shepp_logan) back-projection")
METRIC = "cone-beam back/forward-projection GUPS at 512³×720 views, 1/2/4/8 B200 vs CPU"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-views", type=int, default=0, help="views in the CPU sample (0 = auto)")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# helpers
# ---------------------------------------------------------------------------


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.proc = None
        self.gpu = gpu_index
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200", "-i", str(gpu_index)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except (FileNotFoundError, OSError):
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
            out, _ = self.proc.communicate()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
            except ValueError:
                continue
            for name, flag in zip(names, parts[5:9]):
                if flag.lower() in ("active", "1"):
                    reasons.add(name)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


FP_KERNEL = "cone_fp4z_kernel"  # the default forward projector (TK_FP_ALGO=ldg4z)
BP_KERNEL = "cone_bp_tma_kernel"  # the default back projector (TK_BP_ALGO=tma)


def ncu_traffic():
    """DRAM bytes per launch of the dominant kernel from the newest committed
    ncu capture of the same configuration (profiles/ncu_*.json)."""
    for p in sorted((ROOT / "profiles").glob("ncu_*.json"), reverse=True):  # newest round/letter first
        try:
            d = json.loads(p.read_text())
        except (ValueError, OSError):
            continue
        k = d.get(FP_KERNEL) or {}
        if "dram_bytes_per_launch" in k and k.get("config") == "cfg4-full":
            return float(k["dram_bytes_per_launch"]), f"profiles/{p.name}"
    return None, None


def gather_roofline(fp_bytes, fp_ms, bp_bytes, bp_ms, clocks):
    """Both projectors are gather-bound: their ceiling is the L1 load data path
    (LSU writeback, 128 B/clk/SM; ncu derived__l1tex__lsu_writeback_bytes
    peak_sustained = 128 x 148 B/cycle), not HBM.  Algorithmic bytes: 32 B per
    trilinear sample (FP), 16 B per bilinear update (BP), SURVEY 8(d)."""
    p = ROOT / "MEASURED_PEAKS.json"
    sms = 148
    mhz = (clocks or {}).get("sm_mhz")
    if not mhz and p.exists():
        mhz = json.loads(p.read_text()).get("sm_max_mhz")
    mhz = float(mhz or 1965.0)
    per_clk, src = 128.0, "nominal 128 B/clk/SM"
    probes = sorted((ROOT / "profiles").glob("l1_peak_*.json"), reverse=True)  # scripts/l1_peak.cu
    if probes:
        try:
            per_clk = float(json.loads(probes[0].read_text())["ldg128_bytes_per_clk_sm"])
            src = f"measured LDG.128 {per_clk:.1f} B/clk/SM (profiles/{probes[0].name}, scripts/l1_peak.cu)"
        except (ValueError, KeyError, OSError):
            pass
    peak = per_clk * sms * mhz * 1e6 / 1e9  # GB/s
    fp = fp_bytes / (fp_ms * 1e-3) / 1e9
    bp = bp_bytes / (bp_ms * 1e-3) / 1e9
    return {"bound": "l1_load_path", "unit": "GB/s", "peak": round(peak, 1),
            "peak_source": f"{src} x {sms} SMs x {mhz:.0f} MHz (median SM clock in the timed region)",
            "forward": {"kernel": FP_KERNEL, "achieved": round(fp, 1), "frac": round(fp / peak, 4),
                        "bytes_per_unit": "32 B per trilinear sample"},
            "back": {"kernel": BP_KERNEL, "achieved": round(bp, 1), "frac": round(bp / peak, 4),
                     "bytes_per_unit": "16 B per voxel-view update"}}


def count_samples(geom, step, torch):
    """Exact number of trilinear samples of one forward projection: the same
    float64 clip / loop-count arithmetic as the kernel (reference
    _kernels.py:125-137), evaluated for every ray on the GPU."""
    src, minv = geom.ray_constants
    rows, cols = geom.detector_shape
    nz, ny, nx = geom.volume_shape
    sz, sy, sx = geom.volume_spacing
    h = torch.tensor([(nx + 1) * sx / 2, (ny + 1) * sy / 2, (nz + 1) * sz / 2], dtype=torch.float64,
                     device="cuda")
    r = torch.arange(rows, dtype=torch.float64, device="cuda")[:, None]
    c = torch.arange(cols, dtype=torch.float64, device="cuda")[None, :]
    total = 0
    for i in range(geom.n_projections):
        m = torch.tensor(minv[i], dtype=torch.float64, device="cuda")
        d = torch.stack([m[k, 0] * c + m[k, 1] * r + m[k, 2] for k in range(3)], dim=-1)
        d = d / torch.linalg.vector_norm(d, dim=-1, keepdim=True)
        p = torch.tensor(src[i], dtype=torch.float64, device="cuda")
        t0 = torch.full((rows, cols), -1e300, dtype=torch.float64, device="cuda")
        t1 = torch.full((rows, cols), 1e300, dtype=torch.float64, device="cuda")
        ok = torch.ones((rows, cols), dtype=torch.bool, device="cuda")
        for k in range(3):
            dk = d[..., k]
            par = dk.abs() <= 1e-12
            ok &= ~(par & ((p[k] < -h[k]) | (p[k] > h[k])))
            safe = torch.where(par, torch.ones_like(dk), dk)
            ta = (-h[k] - p[k]) / safe
            tb = (h[k] - p[k]) / safe
            t0 = torch.where(par, t0, torch.maximum(t0, torch.minimum(ta, tb)))
            t1 = torch.where(par, t1, torch.minimum(t1, torch.maximum(ta, tb)))
        span = (t1 - 1e-12 - t0) / step
        n = torch.where(ok & (t0 < t1) & (span > 0), torch.ceil(span), torch.zeros_like(span))
        total += int(n.sum().item())
    return total


# ---------------------------------------------------------------------------
# CPU baseline (oracle: float64 C restatement of the reference kernels)
# ---------------------------------------------------------------------------


def cpu_sample(n_views: int):
    """Time the oracle on `n_views` views spread over the 720-view orbit at full
    resolution; returns (gups_combined, fp_gups, fdk_gups, threads, seconds, desc)."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import numpy as np

    import oracle as ora

    threads = ora.num_threads()
    mats_all = ora.circular_matrices(VIEWS, 2 * math.pi, SDD, SID, DET, DET_SP)
    idx = np.linspace(0, VIEWS, n_views, endpoint=False).astype(int)
    mats = mats_all[idx]
    vol = ora.shepp_logan_3d(VOL)
    step = ora.step_of(SPACING, STEP_SCALE)
    t0 = time.perf_counter()
    sino = ora.forward_cone_3d(vol, SPACING, mats, DET, step)
    t1 = time.perf_counter()
    filt = ora.filter_stage_cone(sino, SDD, SID, DET_SP, FILTER)
    rec = ora.back_cone_3d(filt, mats, SID, VOL, SPACING, weighted=True)
    rec *= math.pi / VIEWS
    t2 = time.perf_counter()
    nvox = VOL[0] * VOL[1] * VOL[2]
    fp_gups = nvox * n_views / (t1 - t0) / 1e9
    fdk_gups = nvox * n_views / (t2 - t1) / 1e9
    comb = 2 * nvox * n_views / (t2 - t0) / 1e9
    desc = (f"oracle (float64 C + OpenMP, bit-exact to the reference kernels) on {n_views} of 720 "
            f"views spread over the orbit, full 512^3 / 1024^2 resolution; FP {t1 - t0:.2f} s, "
            f"filter+BP {t2 - t1:.2f} s; GUPS extrapolate linearly in views")
    return comb, fp_gups, fdk_gups, threads, t2 - t0, desc


def auto_cpu_views(threads: int) -> int:
    # ~0.8 s per view of FP + ~0.2 s of FDK on 8 cores: aim for ~10-30 s of CPU work
    return int(min(48, max(4, threads // 2)))


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    sys.path.insert(0, str(ROOT / "oracle"))
    import oracle as ora

    threads = ora.num_threads()
    nv = args.cpu_views or auto_cpu_views(threads)
    for _ in range(max(0, min(args.warmup, 1))):
        cpu_sample(max(1, nv // 4))
    vals, secs = [], 0.0
    desc = ""
    for _ in range(args.steps):
        comb, fpg, fdkg, threads, sec, desc = cpu_sample(nv)
        vals.append(comb)
        secs += sec
    value = statistics.median(vals)
    ms_step = 2 * VOL[0] * VOL[1] * VOL[2] * VIEWS / (value * 1e9) * 1e3
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "GUPS",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms_step, 1), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic Shepp-Logan 512^3 phantom",
        "config": {"workload": WORKLOAD, "sample_views": nv},
        "cpu_baseline": {"value": round(value, 4), "unit": "GUPS", "cores": threads, "kind": "port",
                         "sample": desc},
        "e2e": {"value": round(value, 4), "unit": "GUPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2511_08427_b200 as tk
    from paper_2511_08427_b200 import _lib, distributed as D
    from paper_2511_08427_b200.filters import filter_stage_tensor
    from paper_2511_08427_b200.projectors import bp_cone_tensor_ex, fp_tensor

    world, rank, local = dist_env()
    # TK_BENCH_BACKEND=gloo runs the multi-rank code path with several ranks
    # sharing the visible GPU(s) -- a functional check of the sharding, row bands
    # and collectives on a 1-GPU box, not a measurement (the driver uses NCCL)
    backend = os.environ.get("TK_BENCH_BACKEND", "nccl")
    if backend != "nccl":
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    _lib.load()

    geom = tk.circular_cone_geometry(VOL, SPACING, DET, DET_SP, VIEWS, 2 * math.pi, SDD, SID)
    step = STEP_SCALE * min(SPACING)
    vb, ve = D.shard_bounds(VIEWS, world, rank)
    sub = D.subset_geometry(geom, slice(vb, ve))
    z0, z1 = D.shard_bounds(VOL[0], world, rank)
    r0, r1 = D.row_band(geom, z0, z1) if world > 1 else (0, DET[0])
    counts = [D.shard_bounds(VIEWS, world, r)[1] - D.shard_bounds(VIEWS, world, r)[0] for r in range(world)]

    vol = tk.phantoms.shepp_logan_3d(VOL, device=dev)
    local_sino = torch.empty((ve - vb, *DET), dtype=torch.float32, device=dev)
    band = torch.empty((VIEWS, r1 - r0, DET[1]), dtype=torch.float32, device=dev)
    slab = torch.empty((z1 - z0, VOL[1], VOL[2]), dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step_fn(ev=None):
        if ev:
            ev[0].record(stream)
        fp_tensor(vol, sub, step, out=local_sino)
        if ev:
            ev[1].record(stream)
        full = D.gather_views(local_sino, counts) if world > 1 else local_sino
        if ev:
            ev[2].record(stream)
        src = full[:, r0:r1, :].contiguous() if world > 1 else full
        filter_stage_tensor(src, geom, FILTER, out=band, row_offset=r0)
        if ev:
            ev[3].record(stream)
        bp_cone_tensor_ex(band, geom, True, r0, z0, z1 - z0, out=slab)
        slab.mul_(math.pi / VIEWS)
        if ev:
            ev[4].record(stream)

    for _ in range(args.warmup):
        step_fn()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()

    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(args.steps)]
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sampler = ClockSampler(local) if rank == 0 else None
    launches0 = _lib.launch_count()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    start.record(stream)
    for k in range(args.steps):
        step_fn(evs[k])
    end.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = sampler.stop() if sampler else None
    launches = _lib.launch_count() - launches0
    elapsed = start.elapsed_time(end)
    phases = np.array([[e[i].elapsed_time(e[i + 1]) for i in range(4)] for e in evs])  # ms
    ph = phases.mean(axis=0)
    t = torch.tensor([elapsed, *ph], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    elapsed, fp_ms, gather_ms, filt_ms, bp_ms = (float(v) for v in t.cpu())
    ms_step = elapsed / args.steps
    nvox = VOL[0] * VOL[1] * VOL[2]
    value = 2 * nvox * VIEWS / (ms_step * 1e-3) / 1e9

    # -- end to end through the public boundary with pinned host buffers --------------
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, tk, torch, dist, D, geom, world, rank, dev, vol, step, counts, sub,
                      z0, z1, r0, r1)

    # -- roofline of the dominant kernel (forward projection) --------------------------
    samples = count_samples(sub, step, torch)
    fp_bytes = 32.0 * samples  # 8 fp32 taps per trilinear sample
    hbm_peak, peak_kind = measured_peaks()
    achieved = fp_bytes / (fp_ms * 1e-3) / 1e9
    traffic, traffic_src = ncu_traffic()
    bp_updates = (z1 - z0) * VOL[1] * VOL[2] * VIEWS
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "GUPS", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 3),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic: Shepp-Logan 512^3 phantom generated on device; 720-view circular orbit",
        "config": {"workload": WORKLOAD, "volume": list(VOL), "views": VIEWS, "detector": list(DET),
                   "step_mm": step, "filter": FILTER,
                   "parallelism": f"FP views/{world} + NCCL all-gather, FDK z-slab/{world} with row bands"
                   if world > 1 else "single GPU",
                   "l2": "no flush: inputs larger than L2 (sinogram 3.0 GB, volume 0.54 GB vs 126 MB L2)"},
        "kernels": {
            "forward_projection": {"ms": round(fp_ms, 3), "gups": round(nvox * (ve - vb) / (fp_ms * 1e-3) / 1e9, 2),
                                   "samples": samples, "gsamples_per_s": round(samples / (fp_ms * 1e-3) / 1e9, 2)},
            "all_gather": {"ms": round(gather_ms, 3)},
            "filter": {"ms": round(filt_ms, 3)},
            "back_projection": {"ms": round(bp_ms, 3), "gups": round(bp_updates / (bp_ms * 1e-3) / 1e9, 2),
                                "gather_gbs": round(16.0 * bp_updates / (bp_ms * 1e-3) / 1e9, 1)},
        },
        "roofline": {"bound": "hbm", "kernel": FP_KERNEL, "achieved": round(achieved, 1),
                     "peak": hbm_peak, "unit": "GB/s", "frac": round(achieved / hbm_peak, 4),
                     "traffic": traffic, "traffic_source": traffic_src,
                     "peak_source": f"{peak_kind} MEASURED_PEAKS.json hbm_gbs",
                     "note": "achieved = algorithmic gather bytes (32 B per trilinear sample x exact sample "
                             "count) / CUDA-event kernel time; gathers are served mostly by L1/L2, so "
                             "frac > 1 is possible -- traffic is the DRAM bytes ncu measured"},
        "gather_roofline": gather_roofline(fp_bytes, fp_ms, 16.0 * bp_updates, bp_ms, clocks),
        "gpu_launches": int(launches),
        "clocks": clocks,
        "e2e": e2e,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            sys.path.insert(0, str(ROOT / "oracle"))
            import oracle as ora

            nv = args.cpu_views or auto_cpu_views(ora.num_threads())
            comb, fpg, fdkg, threads, sec, desc = cpu_sample(nv)
            line["cpu_baseline"] = {"value": round(comb, 4), "unit": "GUPS", "cores": threads,
                                    "kind": "port", "sample": desc,
                                    "fp_gups": round(fpg, 4), "fdk_gups": round(fdkg, 4)}
        except Exception as exc:  # noqa: BLE001
            line["cpu_baseline"] = {"value": None, "error": repr(exc)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def run_e2e(args, tk, torch, dist, D, geom, world, rank, dev, vol, step, counts, sub, z0, z1, r0, r1):
    """Same step through the public API with host buffers: pinned volume in,
    H2D, forward projection, (N>1: NCCL all-gather), FDK, D2H of the
    sinogram and of the reconstruction, every step."""
    from paper_2511_08427_b200 import ops
    from paper_2511_08427_b200.filters import filter_stage_tensor
    from paper_2511_08427_b200.projectors import bp_cone_tensor_ex, fp_tensor

    host_vol = torch.empty(VOL, dtype=torch.float32, pin_memory=True)
    host_vol.copy_(vol)
    cfg = {"geometry_kind": "cone3d", "volume_shape": list(VOL), "volume_spacing": list(SPACING),
           "detector_shape": list(DET), "detector_spacing": list(DET_SP), "number_of_projections": VIEWS,
           "angular_range": 2 * math.pi, "sdd": SDD, "sid": SID, "filter_kind": FILTER,
           "step_scale": STEP_SCALE}
    nbytes = lambda t: t.numel() * t.element_size()  # noqa: E731
    if world == 1:
        def one():
            sino_h = ops.py_forward_project(host_vol, cfg)        # H2D vol, D2H sinogram
            rec_h = ops.py_fbp(sino_h, cfg)                       # H2D sinogram, D2H volume
            return nbytes(host_vol) + nbytes(sino_h), nbytes(sino_h) + nbytes(rec_h)
    else:
        host_sino = torch.empty((counts[rank], *DET), dtype=torch.float32, pin_memory=True)
        host_slab = torch.empty((z1 - z0, VOL[1], VOL[2]), dtype=torch.float32, pin_memory=True)

        def one():
            v = host_vol.to(dev, non_blocking=True)
            loc = fp_tensor(v, sub, step)
            host_sino.copy_(loc, non_blocking=True)
            full = D.gather_views(loc, counts)
            band = filter_stage_tensor(full[:, r0:r1, :].contiguous(), geom, FILTER, row_offset=r0)
            sl = bp_cone_tensor_ex(band, geom, True, r0, z0, z1 - z0)
            sl.mul_(math.pi / VIEWS)
            host_slab.copy_(sl, non_blocking=True)
            torch.cuda.current_stream(dev).synchronize()
            return nbytes(host_vol), nbytes(host_sino) + nbytes(host_slab)

    one()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    steps = max(1, args.steps)
    t0 = time.perf_counter()
    h2d = d2h = 0
    for _ in range(steps):
        h2d, d2h = one()
    torch.cuda.synchronize()
    dt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
    if world > 1:
        dist.barrier()
        dist.all_reduce(dt, op=dist.ReduceOp.MAX)
    sec = float(dt.item()) / steps
    nvox = VOL[0] * VOL[1] * VOL[2]
    return {"value": round(2 * nvox * VIEWS / sec / 1e9, 3), "unit": "GUPS", "ms_per_step": round(sec * 1e3, 1),
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "path": "ops.py_forward_project + ops.py_fbp on pinned host tensors" if world == 1
            else "pinned H2D + view-sharded FP + NCCL all-gather + z-slab FDK + pinned D2H"}


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
