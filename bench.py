#!/usr/bin/env python3
"""Benchmark: cone-beam forward + FDK back-projection GUPS at 512^3 x 720 views.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--fdk zslab|angle] [--chunks C] [--dry-run]

One step = forward projection A x of a 512^3 Shepp-Logan volume (0.5 mm) to a
720-view 1024^2 (0.6 mm) circular cone-beam sinogram, then FDK (cosine
pre-weight + shepp_logan row filter + (sid/w)^2-weighted voxel-driven back
projection + pi/V) of that sinogram.  Both operators count N_vox * V voxel-view
updates, so value = 2 * 512^3 * 720 / step time (whole job, strong scaling).

N > 1 (one process per GPU; `--gpus N` without torchrun re-launches itself
under torch.distributed.run with N ranks): views sharded for A; the FDK is
z-slab sharded, each rank receiving only its detector row band of every view
through an uneven NCCL all-to-all issued per view chunk under the next chunk's
projection (`--fdk zslab`, default), or angle-sharded with a reduce-scatter of
partial volumes (`--fdk angle`, the comparison path).

Prints ONE JSON line on rank 0.  Timing: CUDA events on the launching stream,
barrier + synchronize around the K timed steps, max over ranks.
`--impl reference` times the reference's own CPU implementation (tomokit's
numba kernels from baseline/_ref; the float64 C port in oracle/ when that
install is absent) on the host cores, rank 0 only.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import re
import math
import os
import socket
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
NVOX = VOL[0] * VOL[1] * VOL[2]
WORKLOAD = ("cfg4: cone-beam circular 512^3 @0.5 mm, 720 views over 2pi, 1024^2 detector @0.6 mm, "
            "sdd 1200 / sid 750: forward projection + FDK (shepp_logan) back-projection")
METRIC = "cone-beam back/forward-projection GUPS at 512³×720 views, 1/2/4/8 B200 vs CPU"
FP_KERNEL = "cone_fp_kernel"  # the default forward projector
BP_KERNEL = "cone_bp_tma_kernel"  # the default back projector


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--fdk", choices=["zslab", "p2p", "angle"], default="zslab",
                    help="N>1 FDK decomposition: z-slabs fed by a row-band all-to-all (zslab) or by the "
                         "forward-projection kernel storing rays into peers' band buffers (p2p, NVLink "
                         "symmetric memory), or angle shards + reduce-scatter")
    ap.add_argument("--chunks", type=int, default=4, help="N>1: view chunks of the FP/all-to-all pipeline")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-views", type=int, default=0, help="views in the CPU sample (0 = auto)")
    ap.add_argument("--dry-run", action="store_true",
                    help="launch the N ranks (gloo, no GPU work) and report what world they formed")
    return ap.parse_args()


def config(world: int, fdk: str, chunks: int) -> dict:
    """The workload description -- identical in both arms."""
    if world == 1:
        par = "single GPU"
    elif fdk == "zslab":
        par = (f"dp{world}: FP views/{world}; FDK z-slabs/{world} fed by an uneven NCCL all-to-all of "
               f"detector row bands in {chunks} view chunks")
    elif fdk == "p2p":
        par = (f"dp{world}: FP views/{world} storing each ray into the owning ranks' row-band buffers over "
               f"NVLink peer memory (symmetric memory, no collective); FDK z-slabs/{world}")
    else:
        par = f"dp{world}: FP views/{world}; FDK angle shards/{world} + NCCL reduce-scatter of the volume"
    return {"workload": WORKLOAD, "volume": list(VOL), "views": VIEWS, "detector": list(DET),
            "step_mm": STEP_SCALE * min(SPACING), "filter": FILTER, "parallelism": par,
            "l2": "no flush: inputs larger than L2 (sinogram 3.0 GB, volume 0.54 GB vs 126 MB L2)"}


# ---------------------------------------------------------------------------
# launch helpers
# ---------------------------------------------------------------------------


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def relaunch_under_torchrun(n: int) -> None:
    """`python bench.py --gpus N` without a launcher: exec torch.distributed.run
    with N local ranks (127.0.0.1 rendezvous) on the same arguments."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve()),
           *sys.argv[1:]]
    sys.stdout.flush()
    os.execv(sys.executable, cmd)


def check_world(args, world: int) -> None:
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but the launcher started {world} rank(s)")


def run_dry(args) -> int:
    """Form the N-rank group exactly as the real run does (gloo instead of NCCL,
    no device work) and report it: the CPU test of the launch path."""
    import torch
    import torch.distributed as dist

    world, rank, _ = dist_env()
    check_world(args, world)
    if world > 1:
        dist.init_process_group("gloo")
        t = torch.tensor([rank], dtype=torch.int64)
        got = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(got, t)
        ranks = [int(x) for x in got]
        dist.destroy_process_group()
    else:
        ranks = [0]
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "ranks": ranks,
                          "config": config(world, args.fdk, args.chunks)}), flush=True)
    return 0


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.proc = None
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


# ---------------------------------------------------------------------------
# roofline inputs
# ---------------------------------------------------------------------------


def hbm_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        if d.get("hbm_gbs"):
            return float(d["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (driver-measured copy bandwidth)"
    return 6650.0, "fallback B200_PROFILING.md HBM copy figure"


def l1_peak():
    """The L1 load-path ceiling measured NOW, on this lease (libtkprobe.so:
    LDG.128 with every quarter-warp on one L1-resident line, and conflict-free
    LDS.32).  Falls back to the newest committed probe JSON."""
    try:
        lib = ctypes.CDLL(str(ROOT / "paper_2511_08427_b200" / "libtkprobe.so"))
        out = (ctypes.c_double * 4)()
        if lib.tkp_l1_peak(out) == 0 and out[0] > 0:
            return {"ldg128_gbs": round(out[0], 1), "lds32_gbs": round(out[1], 1), "sms": int(out[2]),
                    "max_clock_mhz": out[3], "source": "measured on this lease (libtkprobe.so tkp_l1_peak)"}
    except OSError:
        pass
    probes = sorted((ROOT / "profiles").glob("l1_peak_*.json"), reverse=True)
    if probes:
        d = json.loads(probes[0].read_text())
        d["source"] = f"profiles/{probes[0].name} (committed probe, earlier lease)"
        return d
    return {"ldg128_gbs": 36380.0, "lds32_gbs": 30900.0, "source": "round-1 probe values"}


def ncu_traffic(kernel: str):
    """DRAM bytes per launch of `kernel` from the newest committed full ncu
    capture of the cfg4 configuration (profiles/ncu_*.json)."""
    caps = list((ROOT / "profiles").glob("ncu_*.json")) + list((ROOT / "profiles").glob("r*/ncu_*.json"))
    def tag(q):  # ncu_r02aq_... sorts after ncu_r02k_...: (round, letter count, letters)
        m = re.match(r"ncu_r(\d+)([a-z]*)_", q.name)
        return (int(m.group(1)), len(m.group(2)), m.group(2)) if m else (-1, 0, q.name)

    for p in sorted(caps, key=tag, reverse=True):
        try:
            d = json.loads(p.read_text())
        except (ValueError, OSError):
            continue
        k = d.get(kernel) or {}
        if "dram_bytes_per_launch" in k and k.get("config") == "cfg4-full":
            # a capture of a launch over a view subset (the back projector runs 720 views as
            # two launches) is scaled to the whole call the bench times
            scale = VIEWS / float(k.get("views", VIEWS))
            return float(k["dram_bytes_per_launch"]) * scale, str(p.relative_to(ROOT))
    return None, None


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


def roofline(samples, fp_ms, fp_views, bp_updates, bp_ms, l1):
    """Roofline of the dominant kernel (the forward projector) against the bound
    that binds it -- the L1 load path -- plus its HBM position.

    * achieved = ALGORITHMIC gather bytes (32 B per trilinear sample x the exact
      sample count) / CUDA-event kernel time; peak = the LDG.128
      ceiling measured on this lease;
    * hbm: algorithmic HBM bytes of one launch (volume read + sinogram write,
      4 (N_vox + V R C)) against the driver-measured copy bandwidth, and the
      ncu DRAM bytes of the same kernel over those algorithmic bytes (re-reads).
    """
    peak = float(l1["ldg128_gbs"])
    fp_bytes = 32.0 * samples
    achieved = fp_bytes / (fp_ms * 1e-3) / 1e9
    hbm, hbm_src = hbm_peak()
    alg_hbm = 4.0 * (NVOX + fp_views * DET[0] * DET[1])
    traffic, traffic_src = ncu_traffic(FP_KERNEL)
    bp_ach = 16.0 * bp_updates / (bp_ms * 1e-3) / 1e9
    bp_traffic, bp_src = ncu_traffic(BP_KERNEL)
    return {
        "bound": "l1_load_path", "kernel": FP_KERNEL, "achieved": round(achieved, 1), "peak": round(peak, 1),
        "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": traffic,
        "algorithmic_bytes_per_launch": fp_bytes,
        "peak_source": f"LDG.128 L1 ceiling, {l1.get('source')}",
        "traffic_source": traffic_src,
        "hbm": {"algorithmic_bytes_per_launch": alg_hbm, "achieved": round(alg_hbm / (fp_ms * 1e-3) / 1e9, 1),
                "peak": hbm, "frac": round(alg_hbm / (fp_ms * 1e-3) / 1e9 / hbm, 5), "peak_source": hbm_src,
                "traffic_over_algorithmic": round(traffic / alg_hbm, 2) if traffic else None},
        "back": {"kernel": BP_KERNEL, "bound": "l1_load_path", "achieved": round(bp_ach, 1),
                 "peak": round(peak, 1), "frac": round(bp_ach / peak, 4),
                 "lds32_peak": l1.get("lds32_gbs"),
                 "frac_of_lds32": round(bp_ach / float(l1["lds32_gbs"]), 4) if l1.get("lds32_gbs") else None,
                 "bytes_per_unit": "16 B per voxel-view update", "traffic": bp_traffic,
                 "traffic_source": bp_src},
    }


# ---------------------------------------------------------------------------
# CPU arms: the reference's own numba kernels (baseline/_ref) or the C port
# ---------------------------------------------------------------------------


def cpu_model() -> str:
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except (OSError, subprocess.SubprocessError):
        pass
    return "unknown"


def _tomokit():
    """Import the unmodified reference (tomokit) from baseline/_ref, numba on every host thread."""
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "tomokit").is_dir():
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/tk_numba_cache")
    if str(ref) not in sys.path:
        sys.path.insert(0, str(ref))
    try:
        import numba

        import tomokit  # noqa: F401
        from tomokit import _kernels
    except ImportError:
        return None
    numba.set_num_threads(os.cpu_count() or 1)
    _kernels.warmup()  # compile once (pkg/tests/conftest.py:11-15)
    return numba.get_num_threads()


def sample_views(n_views: int):
    import numpy as np

    return np.linspace(0, VIEWS, n_views, endpoint=False).astype(int)


class CpuArm:
    """One bounded sample of the workload on the host: the full 512^3 volume and
    1024^2 detector on `n_views` views spread over the 720-view orbit, forward
    projection + FDK.  GUPS is a rate, so the sample's rate is the value."""

    def __init__(self, n_views: int):
        self.n_views = n_views
        self.threads = _tomokit()
        self.kind = "reference" if self.threads else "port"
        if self.kind == "reference":
            from tomokit import filters, geometry, phantoms, projectors

            mats = geometry.circular_trajectory_3d(VIEWS, 2 * math.pi, SDD, SID, DET, DET_SP)
            self.geom = geometry.GeometryCone3D(VOL, SPACING, DET, DET_SP,
                                                [mats[i] for i in sample_views(n_views)], SDD, SID)
            self.vol = phantoms.shepp_logan_3d(VOL, SPACING)
            self._fp = lambda: projectors.forward_project_cone_3d(self.vol, self.geom)
            self._fdk = lambda s: filters.fdk_cone_3d(s, self.geom, FILTER)
        else:
            sys.path.insert(0, str(ROOT / "oracle"))
            import oracle as ora

            self.threads = ora.num_threads()
            mats = ora.circular_matrices(VIEWS, 2 * math.pi, SDD, SID, DET, DET_SP)[sample_views(n_views)]
            vol = ora.shepp_logan_3d(VOL)
            step = ora.step_of(SPACING, STEP_SCALE)
            self._fp = lambda: ora.forward_cone_3d(vol, SPACING, mats, DET, step)
            self._fdk = lambda s: ora.fdk_cone_3d(s, mats, SDD, SID, DET_SP, VOL, SPACING, FILTER)

    def describe(self) -> str:
        what = ("tomokit (the unmodified reference, baseline/_ref) numba kernels, "
                "forward_project_cone_3d + fdk_cone_3d" if self.kind == "reference"
                else "oracle/ float64 C + OpenMP port of the reference kernels (tomokit not importable)")
        return (f"{what} on {self.threads} threads ({cpu_model()}); sample = {self.n_views} of 720 views "
                f"spread over the orbit at the full 512^3 volume / 1024^2 detector")

    def run(self):
        t0 = time.perf_counter()
        sino = self._fp()
        t1 = time.perf_counter()
        self._fdk(sino)
        t2 = time.perf_counter()
        upd = NVOX * self.n_views
        return {"gups": 2 * upd / (t2 - t0) / 1e9, "fp_gups": upd / (t1 - t0) / 1e9,
                "fdk_gups": upd / (t2 - t1) / 1e9, "seconds": t2 - t0, "fp_s": t1 - t0, "fdk_s": t2 - t1}


def default_cpu_views() -> int:
    return 8  # ~4-8 s per FP+FDK sample on 16 host cores


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    arm = CpuArm(args.cpu_views or default_cpu_views())  # compiles the numba kernels (warmup())
    for _ in range(args.warmup):
        arm.run()  # untimed
    runs = [arm.run() for _ in range(args.steps)]
    secs = sum(r["seconds"] for r in runs)
    value = 2 * NVOX * arm.n_views * len(runs) / secs / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "GUPS",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(secs / len(runs) * 1e3, 1), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic Shepp-Logan 512^3 phantom",
        "config": config(args.gpus, args.fdk, args.chunks),
        "cpu_baseline": {"value": round(value, 4), "unit": "GUPS", "cores": arm.threads, "kind": arm.kind,
                         "cpu_model": cpu_model(), "sample": arm.describe(),
                         "fp_gups": round(statistics.median(r["fp_gups"] for r in runs), 4),
                         "fdk_gups": round(statistics.median(r["fdk_gups"] for r in runs), 4)},
        "e2e": {"value": round(value, 4), "unit": "GUPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": "each step is one bounded sample (the sample's views at full resolution); ms_per_step is "
                "that sample's time, value its GUPS rate",
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
    check_world(args, world)
    # TK_BENCH_BACKEND=gloo runs the multi-rank code path with several ranks
    # sharing the visible GPU(s) -- a functional check of the sharding, row bands
    # and collectives on a 1-GPU box, not a measurement (the driver uses NCCL)
    backend = os.environ.get("TK_BENCH_BACKEND", "nccl") if world > 1 else "none"
    if backend == "gloo":
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    _lib.load()
    l1 = l1_peak() if rank == 0 else None

    geom = tk.circular_cone_geometry(VOL, SPACING, DET, DET_SP, VIEWS, 2 * math.pi, SDD, SID)
    step = STEP_SCALE * min(SPACING)
    vb, ve = D.shard_bounds(VIEWS, world, rank)
    sub = D.subset_geometry(geom, slice(vb, ve))
    bands = D.slab_bands(geom, world)
    z0, z1, r0, r1 = bands[rank]
    angle = world > 1 and args.fdk == "angle"
    p2p = world > 1 and args.fdk == "p2p"
    if angle:
        z0, z1 = rank * VOL[0] // world, (rank + 1) * VOL[0] // world
    n_chunks = max(1, args.chunks) if world > 1 else 1

    vol = tk.phantoms.shepp_logan_3d(VOL, device=dev)
    stream = torch.cuda.current_stream(dev)
    if world == 1:
        sino = torch.empty((VIEWS, *DET), dtype=torch.float32, device=dev)
        filt = torch.empty_like(sino)
        slab = torch.empty(VOL, dtype=torch.float32, device=dev)
    elif angle:
        sino = torch.empty((ve - vb, *DET), dtype=torch.float32, device=dev)
        filt = torch.empty_like(sino)
    else:
        band_raw = torch.empty((VIEWS, r1 - r0, DET[1]), dtype=torch.float32, device=dev)
        band = torch.empty_like(band_raw)
        slab = torch.empty((z1 - z0, VOL[1], VOL[2]), dtype=torch.float32, device=dev)
    order = None

    def step_fn(ev=None):
        nonlocal order, slab
        rec = (lambda i: ev[i].record(stream)) if ev else (lambda i: None)
        rec(0)
        if world == 1:
            fp_tensor(vol, geom, step, out=sino)
            rec(1)
            rec(2)
            filter_stage_tensor(sino, geom, FILTER, out=filt)
            rec(3)
            bp_cone_tensor_ex(filt, geom, True, 0, 0, VOL[0], out=slab)
            slab.mul_(math.pi / VIEWS)
        elif angle:
            fp_tensor(vol, sub, step, out=sino)
            rec(1)
            rec(2)
            filter_stage_tensor(sino, geom, FILTER, out=filt)
            rec(3)
            _, slab = D.fdk_angle_sharded(filt, geom, FILTER, rank, world, filter_fn=lambda s: s)
        elif p2p:
            got = D.forward_project_p2p(vol, geom, step, rank, world, bands=bands)
            rec(1)
            rec(2)
            filter_stage_tensor(got, geom, FILTER, out=band, row_offset=r0)
            rec(3)
            bp_cone_tensor_ex(band, geom, True, r0, z0, z1 - z0, out=slab)
            slab.mul_(math.pi / VIEWS)
        else:
            _, order = D.forward_project_and_exchange(
                vol, geom, step, rank, world, n_chunks=n_chunks, bands=bands, out=band_raw,
                on_chunk=lambda k: rec(1) if k == n_chunks - 1 else None)
            rec(2)  # the stream has waited for every chunk's all-to-all
            filter_stage_tensor(band_raw, geom, FILTER, out=band, row_offset=r0)
            rec(3)
            bp_cone_tensor_ex(band, geom, True, r0, z0, z1 - z0, out=slab, views=order)
            slab.mul_(math.pi / VIEWS)
        rec(4)

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
    elapsed, fp_ms, xchg_ms, filt_ms, bp_ms = (float(v) for v in t.cpu())
    ms_step = elapsed / args.steps
    value = 2 * NVOX * VIEWS / (ms_step * 1e-3) / 1e9

    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, tk, torch, dist, D, geom, world, rank, dev, vol, step, sub, bands, n_chunks)

    samples = count_samples(sub, step, torch)
    bp_views = VIEWS if not angle else ve - vb
    bp_updates = (z1 - z0 if not angle else VOL[0]) * VOL[1] * VOL[2] * bp_views
    cfg = config(world, args.fdk, n_chunks)
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "GUPS", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 3),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic: Shepp-Logan 512^3 phantom generated on device; 720-view circular orbit",
        "config": cfg,
        "kernels": {
            "forward_projection": {"ms": round(fp_ms, 3), "views": ve - vb,
                                   "gups": round(NVOX * (ve - vb) / (fp_ms * 1e-3) / 1e9, 2),
                                   "samples": samples, "gsamples_per_s": round(samples / (fp_ms * 1e-3) / 1e9, 2)},
            "exchange": {"ms": round(xchg_ms, 3),
                         "what": "none" if world == 1 else ("none (angle shards)" if angle else
                                                            "peer stores inside the FP kernel + barrier" if p2p
                                                            else "row-band all-to-all tail after the last FP chunk"),
                         "recv_bytes_per_rank": 0 if world == 1 or angle else
                         4 * DET[1] * VIEWS * (r1 - r0) * (world - 1) // world},
            "filter": {"ms": round(filt_ms, 3)},
            "back_projection": {"ms": round(bp_ms, 3), "gups": round(bp_updates / (bp_ms * 1e-3) / 1e9, 2),
                                "includes": "reduce-scatter of the partial volume" if angle else "pi/V scale"},
        },
        "gpu_launches": int(launches),
        "clocks": clocks,
        "e2e": e2e,
    }
    if rank == 0:
        line["roofline"] = roofline(samples, fp_ms, ve - vb, bp_updates, bp_ms, l1)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            arm = CpuArm(args.cpu_views or default_cpu_views())
            r = arm.run()
            line["cpu_baseline"] = {"value": round(r["gups"], 4), "unit": "GUPS", "cores": arm.threads,
                                    "kind": arm.kind, "cpu_model": cpu_model(), "sample": arm.describe(),
                                    "seconds": round(r["seconds"], 2), "fp_gups": round(r["fp_gups"], 4),
                                    "fdk_gups": round(r["fdk_gups"], 4)}
        except Exception as exc:  # noqa: BLE001
            line["cpu_baseline"] = {"value": None, "error": repr(exc)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def run_e2e(args, tk, torch, dist, D, geom, world, rank, dev, vol, step, sub, bands, n_chunks):
    """Same step through the public API with host buffers: pinned volume in,
    H2D, forward projection, (N>1: row-band exchange), FDK, D2H of the
    sinogram and of the reconstruction, every step."""
    from paper_2511_08427_b200 import ops
    from paper_2511_08427_b200.filters import filter_stage_tensor
    from paper_2511_08427_b200.projectors import bp_cone_tensor_ex

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
        z0, z1, r0, r1 = bands[rank]
        host_band = torch.empty((VIEWS, r1 - r0, DET[1]), dtype=torch.float32, pin_memory=True)
        host_slab = torch.empty((z1 - z0, VOL[1], VOL[2]), dtype=torch.float32, pin_memory=True)

        def one():
            v = host_vol.to(dev, non_blocking=True)
            band, order = D.forward_project_and_exchange(v, geom, step, rank, world, n_chunks=n_chunks,
                                                         bands=bands)
            host_band.copy_(band, non_blocking=True)
            f = filter_stage_tensor(band, geom, FILTER, row_offset=r0)
            sl = bp_cone_tensor_ex(f, geom, True, r0, z0, z1 - z0, views=order)
            sl.mul_(math.pi / VIEWS)
            host_slab.copy_(sl, non_blocking=True)
            torch.cuda.current_stream(dev).synchronize()
            return nbytes(host_vol), nbytes(host_band) + nbytes(host_slab)

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
    return {"value": round(2 * NVOX * VIEWS / sec / 1e9, 3), "unit": "GUPS", "ms_per_step": round(sec * 1e3, 1),
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "path": "ops.py_forward_project + ops.py_fbp on pinned host tensors" if world == 1
            else "pinned H2D + view-sharded FP + row-band all-to-all + z-slab FDK + pinned D2H of the "
                 "rank's band and slab"}


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch_under_torchrun(args.gpus)  # does not return
    # NCCL's communicator-init lines (ranks, NVLink/NVLS transport) go to stderr,
    # keeping stdout for the one JSON line
    os.environ.setdefault("NCCL_DEBUG", "INFO")
    os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    if args.dry_run:
        return run_dry(args)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
