#!/usr/bin/env python
"""HyRes throughput benchmark (BASELINE.json metric: voxels/s and ms per cube).

python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config large]

A step is one full HyRes pass (north_star stages (1)-(6)) over one synthetic
cube resident in HBM.  Default workload: `large` (1024 x 1024 x 224 fp32, the
north_star target; the cube is 940 MB, larger than the 126 MB L2, so no L2
flush is needed between steps).  For N > 1 (torchrun, one rank per GPU) the
default is the pixel-sharded single cube (hyde_hyres_sharded: rank g holds pixel
rows [gR/N, (g+1)R/N), NCCL inside libhyde: Gram all-reduce, slab <-> component
all-to-all for the wavelet stage; strong scaling); independent
replica cubes (seed = rank, weak scaling) are reported beside it under
"replicas" (--replicas makes them the headline).  --config batched shards the
64 independent cubes round-robin (no data-path collective).

Reports one JSON line (rank 0): value = whole-job voxels/s; e2e = the same
metric through the C-ABI with HOST buffers (H2D + D2H inside the timed
region); roofline = the dominant stage's algorithmic bytes / its CUDA-event
duration vs MEASURED_PEAKS.json; cpu_baseline = the fp64 oracle on the host.
`--impl reference` times the oracle itself (the reference arm of this tier).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from harness import dist as hd  # noqa: E402
from harness import synth  # noqa: E402

METRIC = "HyRes voxels/sec and ms/cube"
UNIT = "voxels/s"


NOMINAL_HBM_GBS = 8000.0   # BASELINE.json north_star "~8 TB/s" (B200_PROFILING.md: 7.7 HGX / 8 DGX)
PEAKS_FILE = os.path.join(ROOT, "profiles", "r02_peaks.json")      # tools/probe_peaks.cu on a B200 of this pool
TRAFFIC_FILE = os.path.join(ROOT, "profiles", "r02_traffic.json")  # ncu --set full dram bytes per launch


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d.get("hbm_gbs", 6650.0)), float(d.get("bf16_tflops", 1590.0)), "measured"
    return 6650.0, 1590.0, "fallback (B200_PROFILING.md)"


def probe_peaks():
    """fp64 / int8-tensor peaks measured by tools/probe_peaks.cu (committed JSON), or {}."""
    try:
        return json.load(open(PEAKS_FILE))
    except Exception:  # noqa: BLE001
        return {}


def ncu_traffic(kernel):
    """DRAM bytes (read + write) per launch of `kernel` from the committed ncu capture, or None."""
    try:
        d = json.load(open(TRAFFIC_FILE))
        v = d["kernels"].get(kernel)
        return None if v is None else {"bytes": v, "source": d.get("source")}
    except Exception:  # noqa: BLE001
        return None


# ------------------------------------------------------------------ clocks (NVML)
class ClockSampler:
    """Polls SM clock and clock-event reasons every ~5 ms in a thread."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, pci_bus_id: str | None):
        self.samples = []
        self.marks = []
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            if pci_bus_id:
                self.h = pynvml.nvmlDeviceGetHandleByPciBusId(pci_bus_id.encode())
            else:
                self.h = pynvml.nvmlDeviceGetHandleByIndex(0)
            self.nv = pynvml
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # noqa: BLE001
            self.err = str(e)

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                mhz = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                try:
                    rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                except Exception:  # noqa: BLE001
                    rs = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                self.samples.append((time.perf_counter(), mhz, rs))
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.005)

    def start(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()

    def mark(self):
        self.marks.append(time.perf_counter())

    def stop(self):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0,
                    "note": getattr(self, "err", "no samples")}
        t0, t1 = (self.marks[0], self.marks[-1]) if len(self.marks) >= 2 else (0, float("inf"))
        inside = [s for s in self.samples if t0 <= s[0] <= t1]
        src = "timed region"
        if len(inside) < 3:   # very short timed region: use warm-up + timed samples
            inside = self.samples[-max(3, len(inside)):]
            src = "warm-up + timed region (timed region shorter than 3 samples)"
        mhz = [s[1] for s in inside]
        reasons = set()
        for s in inside:
            for bit, name in self.REASONS.items():
                if s[2] & bit:
                    reasons.add(name)
        return {"sm_mhz": float(statistics.median(mhz)), "sm_max_mhz": float(self.max_mhz),
                "reasons": sorted(reasons), "samples": len(inside), "window": src}


# ------------------------------------------------------------------ algorithmic bytes
def level_shapes(rows, cols, levels):
    """Subband shape per level: (ceil(h/2), ceil(w/2)) of the previous LL (R5)."""
    out, h, w = [], rows, cols
    for _ in range(levels):
        h, w = (h + 1) // 2, (w + 1) // 2
        out.append((h, w))
    return out


def dwt_image_bytes(rows, cols, levels):
    """Per image and level: read the level input, write LL + 3 detail subbands."""
    h, w, b = rows, cols, 0
    for (hs, ws) in level_shapes(rows, cols, levels):
        b += 4 * h * w + 4 * 4 * hs * ws
        h, w = hs, ws
    return b


def coeff_count(rows, cols, levels):
    sh = level_shapes(rows, cols, levels)
    return 3 * sum(h * w for h, w in sh) + sh[-1][0] * sh[-1][1]


def stage_bytes(cfg, levels, rank, comps, chunks):
    """Algorithmic HBM bytes per step for each stage: the minimum
    each stage must move.  comps = candidate components projected/transformed."""
    n, b = cfg.rows * cfg.cols, cfg.bands
    nc = coeff_count(cfg.rows, cfg.cols, levels)
    dwt_img = dwt_image_bytes(cfg.rows, cfg.cols, levels)
    return {
        "gram": 4 * n * b,
        "project": chunks * 4 * n * b + 4 * n * comps,
        "dwt": comps * dwt_img,
        "sure": comps * 4 * nc,                     # one read of N_c coefficients (soft threshold is applied by the IDWT)
        "idwt": rank * dwt_img,
        "recon": 4 * n * rank + 4 * n * b,
    }


def wavelet_isolated(hy, torch, cube, cfg, levels, steps, hbm):
    """Stage-isolated A4 -> A5 -> A6a on ALL B eigen-images of the cube (SURVEY.md
    §8(d): the end-to-end path transforms only a few components, too short for a
    stable HBM fraction).  Setup (not timed): G by the library's Gram, sigma by
    K2, the whitened eigenvectors by torch.linalg.eigh and E = W^T Y by a torch
    matmul.  Timed: hyde_wavelet_shrink (DWT levels + one SURE launch + IDWT
    levels with the fused soft threshold), `steps` calls, CUDA events per stage."""
    b, n = cfg.bands, cfg.rows * cfg.cols
    y = cube.view(b, n)
    G = hy.stages.gram(cube)
    sigma, _, _ = hy.stages.eig(G, n, 1, all_lam=False)
    gw = G / (sigma[:, None] * sigma[None, :]) / n
    _, V = torch.linalg.eigh(gw)
    W = (V.flip(1) / sigma[:, None]).to(torch.float32)
    E = (W.t() @ y).view(b, cfg.rows, cfg.cols).contiguous()
    del G, gw, V, W
    out = torch.empty_like(E)
    hy.stages.wavelet_shrink(E, levels, out=out, stats=False)
    hy.stages.wavelet_shrink(E, levels, out=out, stats=False)
    torch.cuda.synchronize()
    dev = cube.device.index
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # DWT + SURE alone (the analysis-only call): its own wall time
    hy.stages.wavelet_shrink(E, levels, stats=False, analyze_only=True)
    torch.cuda.synchronize()
    e0.record(st)
    for _ in range(steps):
        hy.stages.wavelet_shrink(E, levels, stats=False, analyze_only=True)
    e1.record(st)
    torch.cuda.synchronize()
    ds_wall = e0.elapsed_time(e1) / steps
    hy.profile_enable(dev, True)
    e0.record(st)
    for _ in range(steps):
        hy.stages.wavelet_shrink(E, levels, out=out, stats=False)
    e1.record(st)
    torch.cuda.synchronize()
    stg = hy.profile_read(dev)
    hy.profile_enable(dev, False)
    ms = e0.elapsed_time(e1) / steps
    nc = coeff_count(cfg.rows, cfg.cols, levels)
    lvl = b * dwt_image_bytes(cfg.rows, cfg.cols, levels)
    byt = {"dwt": lvl, "sure": b * 4 * nc, "idwt": lvl}
    res = {"images": b, "rows": cfg.rows, "cols": cfg.cols, "levels": levels, "ms": round(ms, 4),
           "timing": "CUDA events around the calls (wall); per-stage ms from the library's stage events; "
                     "dwt+sure = wall time of the analysis-only call (out = NULL)"}
    tot_b, tot_t = 0, 0.0
    for k in ("dwt", "sure", "idwt"):
        t = stg[k][0] / steps
        gbs = byt[k] / (t * 1e-3) / 1e9
        res[k] = {"ms": round(t, 4), "bytes": byt[k], "GBps": round(gbs, 1), "frac_hbm": round(gbs / hbm, 4)}
        tot_b += byt[k]
        tot_t += t
    ds_b = byt["dwt"] + byt["sure"]
    ds_t = ds_wall
    res["dwt+sure"] = {"ms": round(ds_t, 4), "bytes": ds_b, "GBps": round(ds_b / (ds_t * 1e-3) / 1e9, 1),
                       "frac_hbm": round(ds_b / (ds_t * 1e-3) / 1e9 / hbm, 4)}
    res["dwt+sure+idwt"] = {"ms": round(ms, 4), "bytes": tot_b,
                            "GBps": round(tot_b / (ms * 1e-3) / 1e9, 1),
                            "frac_hbm": round(tot_b / (ms * 1e-3) / 1e9 / hbm, 4),
                            "busy_ms_sum": round(tot_t, 4)}
    # the method's minimum: DWT one read of N + one write of N_c
    # per image (a fused multi-level transform), SURE one read of N_c
    mb = b * (4 * n + 4 * nc + 4 * nc)
    res["dwt+sure_min_bytes"] = {"bytes": mb, "frac_hbm": round(mb / (ds_t * 1e-3) / 1e9 / hbm, 4),
                                 "frac_nominal_8tbs": round(mb / (ds_t * 1e-3) / 1e9 / NOMINAL_HBM_GBS, 4)}
    res["dwt+sure"]["frac_nominal_8tbs"] = round(ds_b / (ds_t * 1e-3) / 1e9 / NOMINAL_HBM_GBS, 4)
    del E, out
    torch.cuda.empty_cache()
    return res


def cpu_baseline(cube, reps=2):
    from oracle import hyres_ref as O
    cores = len(os.sched_getaffinity(0))
    try:
        from threadpoolctl import threadpool_info
        thr = max([d.get("num_threads", 1) for d in threadpool_info()] or [1])
    except Exception:  # noqa: BLE001
        thr = cores
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        O.hyres(cube)
        ts.append(time.perf_counter() - t0)
    t = float(np.mean(ts))
    return t, cores, thr


# ------------------------------------------------------------------ reference arm
def config_dict(cfg, world, batched, sharded, ncube, nbytes):
    """The workload keys of a bench line -- identical for both arms at N = 1
    (the reference arm's sample is the same seed-0 cube); run results go under
    "result"."""
    return {"workload": cfg.name, "rows": cfg.rows, "cols": cfg.cols, "bands": cfg.bands,
            "cubes_per_rank": ncube,
            "seeds": (f"batch of {cfg.batch} (seeds 0..{cfg.batch - 1}) round-robin over ranks"
                      if batched else ("one cube (seed 0), pixel-row slabs per rank (hyde_hyres_sharded)"
                                       if sharded else f"rank r uses seed r (0..{world - 1})")),
            "l2": (f"inputs larger than L2 ({nbytes / 1e6:.0f} MB per rank > 126 MB L2); no flush"
                   if nbytes > 126e6 else "cube fits in L2: steps run back to back (L2-warm)")}


def run_reference(args, cfg, rank, world):
    if rank != 0:
        return 0
    s = synth.make_cube(cfg, 0)
    cube = s.noisy
    from oracle import hyres_ref as O
    for _ in range(args.warmup):
        O.hyres(cube)
    ts = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        O.hyres(cube)
        ts.append(time.perf_counter() - t0)
    t = float(np.mean(ts))
    v = cfg.voxels / t
    cores = len(os.sched_getaffinity(0))
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(cfg, 1, cfg.batch > 1, False, 1, cube.nbytes),
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
                         "sample": f"full {cfg.name} cube per step (oracle.hyres, numpy fp64, as it stands)"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ our arm
def k2_flops(B):
    """Algorithmic fp64 flops of K2: Gauss-Jordan inverse of
    G + dI (2 B^3), Householder tridiagonalisation (4/3 B^3) and the
    accumulation of Q (4/3 B^3); the tridiagonal eigenpairs are O(B^2)."""
    return (2.0 + 4.0 / 3.0 + 4.0 / 3.0) * B ** 3


def cube_stream(hy, torch, cube, cfg, k, steps):
    """Throughput of a stream of k cubes (copies of the bench cube, each fully
    processed) through hyde_hyres_batched: its lanes overlap one cube's
    latency-bound eigensolver (one 16-SM cluster) with the other cubes'
    HBM-bound stages.  Reported beside the single-cube number, not instead of it."""
    cubes = cube.unsqueeze(0).expand(k, *cube.shape).contiguous()
    outs = torch.empty_like(cubes)
    for _ in range(2):
        hy.hyres_batched(cubes, outs)
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(steps):
        hy.hyres_batched(cubes, outs)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    del cubes, outs
    torch.cuda.empty_cache()
    return {"cubes_per_call": k, "calls": steps, "ms_per_call": round(ms, 4),
            "ms_per_cube": round(ms / k, 4), "value": k * cfg.voxels / (ms * 1e-3), "unit": "voxels/s",
            "path": "hyde_hyres_batched on k copies of the seed-0 cube (device-resident), CUDA events"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="large", choices=["tiny", "small", "medium", "wide", "large", "batched"])
    ap.add_argument("--e2e-steps", type=int, default=8)
    ap.add_argument("--stream-cubes", type=int, default=4,
                    help="extra measurement: throughput of a stream of this many copies of the cube "
                         "through hyde_hyres_batched (lanes overlap the cubes' stages); 0 = off")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--iso-steps", type=int, default=5,
                    help="steps of the stage-isolated DWT/SURE/IDWT leg on all B eigen-images (0: skip)")
    ap.add_argument("--shard", action="store_true",
                    help="one cube split into pixel-row slabs across the ranks (hyde_hyres_sharded; strong "
                         "scaling) -- the default for N > 1; at N = 1 it runs the path on a world-1 NCCL comm")
    ap.add_argument("--replicas", action="store_true",
                    help="N > 1: independent cubes per rank (seed = rank, weak scaling) as the headline")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    cfg = synth.CONFIGS[args.config]
    rank, world, local = hd.env_rank()

    if args.impl == "reference":
        return run_reference(args, cfg, rank, world)

    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2204_06979_b200 as hy

    # Work of this rank: one cube (seed = rank; weak scaling) or, for the batched
    # workload, its round-robin shard of the fixed batch of independent cubes
    # (strong scaling).  No data-path collective either way.
    batched = cfg.batch > 1
    sharded = (args.shard or (world > 1 and not args.replicas)) and not batched
    seeds = hd.shard(cfg.batch, rank, world) if batched else ([0] if sharded else [rank])
    cubes_h = [np.ascontiguousarray(synth.make_cube(cfg, seed=sd).noisy) for sd in seeds]
    ncube = len(cubes_h)
    if sharded:
        # this rank's pixel-row slab of cube 0; the Gram all-reduce and the
        # slab <-> component all-to-all run through NCCL inside libhyde
        r0, r1 = hy.slab_rows(cfg.rows, rank, world)
        full_h = cubes_h[0]
        cubes_h = [np.ascontiguousarray(full_h[:, r0:r1, :])]
        comm = hy.NcclComm() if world > 1 else hy.nccl_comm_single()
        cube = torch.from_numpy(cubes_h[0]).cuda()
        out = torch.empty_like(cube)
        run = lambda: hy.hyres_sharded(cube, cfg.rows, comm, out, return_info=True)   # noqa: E731
    elif batched:
        cube = torch.from_numpy(np.stack(cubes_h)).cuda()
        out = torch.empty_like(cube)
        run = lambda: hy.hyres_batched(cube, out, return_info=True)   # noqa: E731
    else:
        cube = torch.from_numpy(cubes_h[0]).cuda()
        out = torch.empty_like(cube)
        run = lambda: hy.hyres(cube, out, return_info=True)   # noqa: E731
    props = torch.cuda.get_device_properties(local)
    bus = None
    try:
        bus = f"{props.pci_domain_id:08x}:{props.pci_bus_id:02x}:{props.pci_device_id:02x}.0"
    except Exception:  # noqa: BLE001
        pass
    clk = ClockSampler(bus)
    clk.start()

    _, info = run()
    if batched:
        info = info[0]
    for _ in range(args.warmup - 1):
        run()
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = hy.launch_count(local)
    clk.mark()
    e0.record(st)
    marks = [e0]
    for _ in range(args.steps):
        run()
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(st)
        marks.append(ev)
    e1.record(st)
    torch.cuda.synchronize()
    clk.mark()
    if world > 1:
        dist.barrier()
    per_step = [marks[i].elapsed_time(marks[i + 1]) for i in range(args.steps)]
    # the paper's protocol: drop the fastest and the
    # slowest step, average the rest -- reported beside the contract's mean
    olympic = (sum(sorted(per_step)[1:-1]) / (args.steps - 2)) if args.steps >= 3 else None
    launches = hy.launch_count(local) - launches0
    # stage table: the same number of steps again, with the library's per-stage
    # events on (outside the timed region: the events split the programmatic
    # dependent launches between stages)
    hy.profile_enable(local, True)
    for _ in range(args.steps):
        run()
    torch.cuda.synchronize()
    stages = hy.profile_read(local)
    hy.profile_enable(local, False)
    ms = e0.elapsed_time(e1) / args.steps
    ms_max = hd.max_over_ranks(ms, device="cuda")
    cubes_total = 1.0 if sharded else hd.sum_over_ranks(ncube, device="cuda")
    value = hd.whole_job_rate(cubes_total * cfg.voxels, ms_max * 1e-3)

    reps = None
    if sharded and world > 1:
        # independent replica cubes (seed = rank): weak scaling, no collective
        rcube = torch.from_numpy(np.ascontiguousarray(synth.make_cube(cfg, seed=rank).noisy)).cuda()
        rout = torch.empty_like(rcube)
        for _ in range(args.warmup):
            hy.hyres(rcube, rout)
        torch.cuda.synchronize()
        dist.barrier()
        r0e, r1e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        r0e.record(st)
        for _ in range(args.steps):
            hy.hyres(rcube, rout)
        r1e.record(st)
        torch.cuda.synchronize()
        rms = hd.max_over_ranks(r0e.elapsed_time(r1e) / args.steps, device="cuda")
        reps = {"value": hd.whole_job_rate(world * cfg.voxels, rms * 1e-3), "unit": UNIT, "ms_per_step": rms,
                "scaling": "weak", "path": "hyde_hyres_ex, one whole cube per rank (seed = rank), no collective"}
        del rcube, rout
        torch.cuda.empty_cache()

    hys = None
    if args.iso_steps > 0 and not batched and not sharded and rank == 0:
        # F1: HySime on the same cube -- Gram + sweep + raw
        # eigendecomposition of R_x (all B eigenpairs) + criterion
        hy.hysime(cube)
        torch.cuda.synchronize()
        ts = []
        for _ in range(3):
            t0 = time.perf_counter()
            hres = hy.hysime(cube)
            ts.append(time.perf_counter() - t0)
        hys = {"ms": round(1e3 * statistics.median(ts), 4), "k": hres["k"], "bands": cfg.bands,
               "timing": "host wall clock of the synchronous call (returns k), median of 3"}
    fpd = None
    if args.iso_steps > 0 and not batched and not sharded and rank == 0:
        # F2: FORPDN with the D16 default lambda -- Gram +
        # sweep (noise power), per-band DWT, lambda selection on B x B matrices,
        # Thomas solve along the bands, per-band IDWT
        fout = torch.empty_like(cube)
        _, flam = hy.forpdn(cube, fout, return_lambda=True)
        torch.cuda.synchronize()
        st_ = torch.cuda.current_stream()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(st_)
        for _ in range(3):
            hy.forpdn(cube, fout)
        f1.record(st_)
        torch.cuda.synchronize()
        fms = f0.elapsed_time(f1) / 3
        hbm_, _, _ = peaks()
        lvl = hy.stages.auto_levels(cfg.rows, cfg.cols)
        ncf = coeff_count(cfg.rows, cfg.cols, lvl)
        fb = (2 * cfg.bands * dwt_image_bytes(cfg.rows, cfg.cols, lvl)   # per-band DWT + IDWT levels
              + 4 * cfg.bands * cfg.rows * cfg.cols                       # Gram: one read (K1)
              + 8 * cfg.bands * ncf)                                       # solve: read W, write X
        fpd = {"ms": round(fms, 4), "lambda": flam, "bytes": fb, "GBps": round(fb / (fms * 1e-3) / 1e9, 1),
               "frac_hbm": round(fb / (fms * 1e-3) / 1e9 / hbm_, 4),
               "timing": "CUDA events over 3 calls (lambda by D16 each call)"}
        # F4: WSRRR with the D17 defaults (rank = HySime's k)
        wout = torch.empty_like(cube)
        hy.wsrrr(cube, wout)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        wres = hy.wsrrr(cube, wout)
        torch.cuda.synchronize()
        wms = (time.perf_counter() - t0) * 1e3
        nsw = len(wres["objective"])
        wb = (2 * cfg.bands * dwt_image_bytes(cfg.rows, cfg.cols, lvl)       # per-band DWT + IDWT levels
              + nsw * 2 * 4 * cfg.bands * ncf)                                 # each sweep reads W twice
        fpd_w = {"ms": round(wms, 3), "rank": wres["rank"], "lambda": wres["lam"], "sweeps": nsw,
                 "bytes": wb, "GBps": round(wb / (wms * 1e-3) / 1e9, 1),
                 "frac_hbm": round(wb / (wms * 1e-3) / 1e9 / hbm_, 4),
                 "timing": "host wall clock of the synchronous call (includes HySime for the rank)"}
        # F3: HyMiNoR's l1-l1 spectral stage on the HyRes output
        # (D19 defaults), one warp per pixel
        hout = torch.empty_like(cube)
        hy.hyres(cube, hout)
        lout = torch.empty_like(cube)
        hy.l1_spectral(hout, lout)
        torch.cuda.synchronize()
        h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        h0.record(st_)
        for _ in range(3):
            _, its = hy.l1_spectral(hout, lout, return_iters=True)
        h1.record(st_)
        torch.cuda.synchronize()
        lms = h0.elapsed_time(h1) / 3
        lb = 8 * cfg.bands * cfg.rows * cfg.cols                           # read M, write X
        fpd_h = {"l1_stage_ms": round(lms, 4), "hyres_plus_l1_ms": round(ms_max + lms, 4),
                 "mean_iters": round(float(its.float().mean()), 3), "bytes": lb,
                 "GBps": round(lb / (lms * 1e-3) / 1e9, 1), "frac_hbm": round(lb / (lms * 1e-3) / 1e9 / hbm_, 4),
                 "timing": "CUDA events over 3 calls of the l1 stage; + the bench's HyRes step time"}
        del fout, wout, hout, lout
    else:
        fpd_w = None
        fpd_h = None
    iso = None
    if args.iso_steps > 0 and not batched and not sharded and rank == 0:
        hbm_, _, _ = peaks()
        iso = wavelet_isolated(hy, torch, cube, cfg, info["levels"], args.iso_steps, hbm_)
    strm = None
    if args.stream_cubes > 1 and not batched and not sharded and rank == 0:
        strm = cube_stream(hy, torch, cube, cfg, args.stream_cubes, max(2, args.iso_steps // 2))

    # ---- end to end through the C-ABI with host buffers (pinned), H2D + D2H inside ----
    # hyde_hyres_host_stream: every step copies its cubes in and its results out;
    # the copies of neighbouring cubes overlap the current cube's compute
    pins = [torch.from_numpy(c).pin_memory() for c in cubes_h]
    pouts = [torch.empty_like(p).pin_memory() for p in pins]
    ne = max(args.e2e_steps, 1)
    if sharded:
        # each rank: its slab H2D, hyde_hyres_sharded, its slab D2H -- every step
        def e2e_step():
            x = pins[0].to("cuda", non_blocking=True)
            y = hy.hyres_sharded(x, cfg.rows, comm)
            pouts[0].copy_(y, non_blocking=True)
        e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(ne):
            e2e_step()
        torch.cuda.synchronize()
    else:
        hy.hyres_host_stream(pins[:1], pouts[:1], device=local)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        seq_in = [pins[i % ncube] for i in range(ne * ncube)]
        seq_out = [pouts[i % ncube] for i in range(ne * ncube)]
        t0 = time.perf_counter()
        hy.hyres_host_stream(seq_in, seq_out, device=local)
        torch.cuda.synchronize()
    e2e_s = hd.max_over_ranks((time.perf_counter() - t0) / ne, device="cuda")
    # the link's own floor for the same bytes: H2D of the inputs and D2H of the
    # outputs on two streams at once (full-duplex PCIe), device buffers only
    link_s = None
    if not sharded and args.e2e_steps > 0:
        din = torch.empty_like(pins[0], device="cuda")
        dout = torch.empty_like(pins[0], device="cuda")
        s_a, s_b = torch.cuda.Stream(), torch.cuda.Stream()
        reps = 3
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        for _ in range(reps):
            for i in range(ncube):
                with torch.cuda.stream(s_a):
                    din.copy_(pins[i], non_blocking=True)
                with torch.cuda.stream(s_b):
                    pouts[i].copy_(dout, non_blocking=True)
        torch.cuda.synchronize()
        link_s = (time.perf_counter() - t1) / reps
        del din, dout
    clk.stop()
    csum = clk.summary()

    # ---- roofline of the dominant stage ----
    hbm, _, src = peaks()
    rank_k = info["rank"]
    chunks = info["chunks_run"]
    comps = info["comps"]   # candidate components actually projected / transformed
    sb = {k: v * ncube for k, v in stage_bytes(cfg, info["levels"], rank_k, comps, chunks).items()}
    per = {}
    for name, (tms, nl) in stages.items():
        t = tms / args.steps
        d = {"ms": round(t, 5), "launches_per_step": nl / args.steps}
        if name in sb and t > 0:
            gbs = sb[name] / (t * 1e-3) / 1e9
            d.update({"bytes": sb[name], "GBps": round(gbs, 1), "frac_hbm": round(gbs / hbm, 4)})
        per[name] = d
    dws = sb["dwt"] + sb["sure"]
    tds = (stages["dwt"][0] + stages["sure"][0]) / args.steps
    per["dwt+sure"] = {"ms": round(tds, 5), "bytes": dws,
                       "GBps": round(dws / (tds * 1e-3) / 1e9, 1) if tds > 0 else None,
                       "frac_hbm": round(dws / (tds * 1e-3) / 1e9 / hbm, 4) if tds > 0 else None,
                       "frac_nominal_8tbs": round(dws / (tds * 1e-3) / 1e9 / NOMINAL_HBM_GBS, 4) if tds > 0 else None}
    # SURVEY §8(d) minimum for the in-step DWT+SURE: one read of N and one write of
    # N_c per transformed component (a fused multi-level DWT), one SURE read of N_c
    ncf = coeff_count(cfg.rows, cfg.cols, info["levels"])
    dmin = ncube * comps * 4 * (cfg.rows * cfg.cols + 2 * ncf)
    if tds > 0:
        per["dwt+sure"]["min_bytes"] = dmin
        per["dwt+sure"]["frac_hbm_min_bytes"] = round(dmin / (tds * 1e-3) / 1e9 / hbm, 4)
    dom = max((k for k in stages), key=lambda k: stages[k][0])
    t = stages[dom][0] / args.steps
    kern = {"eig": "k2_cluster_kernel", "gram": "gram_tc_kernel", "project": "project_kernel", "recon": "recon_kernel",
            "sure": "sure_kernel", "dwt": "dwt_fwd_kernel", "idwt": "dwt_inv_kernel"}.get(dom, dom)
    tr = ncu_traffic(kern)
    if dom in sb:
        ach = sb[dom] / (t * 1e-3) / 1e9
        roof = {"kernel": kern, "stage": dom, "bound": "hbm", "achieved": round(ach, 1), "peak": hbm,
                "unit": "GB/s", "frac": round(ach / hbm, 4), "traffic": tr["bytes"] if tr else None,
                "algorithmic_bytes": sb[dom], "peak_source": src, "share_of_step": round(t / ms_max, 4),
                "frac_nominal_8tbs": round(ach / NOMINAL_HBM_GBS, 4)}
    else:   # K2: one 16-CTA cluster, fp64, a B-step dependency chain
        ncta = hy.eig_cluster_size() or 16
        if batched:   # ONE launch of 8-CTA clusters for the whole batch: up to 18 clusters (144 SMs) at once
            ncta = 8 * min(ncube, 148 // 8)
        flops = ncube * k2_flops(cfg.bands)
        pk = probe_peaks()
        if pk.get("fp64_tflops_per_sm"):
            peak = ncta * float(pk["fp64_tflops_per_sm"])
            psrc = (f"measured: {ncta} SMs ({'the concurrent clusters' if batched else 'one cluster'}) x {pk['fp64_tflops_per_sm']} fp64 TFLOP/s per SM "
                    f"(tools/probe_peaks.cu, profiles/r02_peaks.json; whole GPU {pk.get('fp64_tflops')} TFLOP/s)")
        else:
            peak = ncta * 64 * 2 * 1.965e9 / 1e12      # DFMA/clk/SM x 2 flops x max SM clock
            psrc = f"derived: {ncta} SMs x 64 DFMA/clk x 2 x 1965 MHz"
        ach = flops / (t * 1e-3) / 1e12
        roof = {"kernel": kern, "stage": dom, "bound": "alu", "achieved": round(ach, 4), "peak": round(peak, 4),
                "unit": "TFLOP/s", "frac": round(ach / peak, 4), "traffic": tr["bytes"] if tr else None,
                "algorithmic_flops": flops,
                "peak_source": psrc + "; latency-bound (B sequential Householder steps)",
                "share_of_step": round(t / ms_max, 4)}
    if tr:
        roof["traffic_source"] = tr["source"]

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0
    nbytes = int(sum(c.nbytes for c in cubes_h))
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max, "ms_per_cube": ms_max / ncube,
        "ms_per_step_olympic": olympic, "ms_per_step_min": min(per_step), "ms_per_step_max": max(per_step),
        "higher_is_better": True, "scaling": "strong" if (batched or sharded) else "weak", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic",
        "config": config_dict(cfg, world, batched, sharded, ncube, nbytes),
        "result": {"rank": rank_k, "levels": info["levels"], "chunks": chunks, "components": comps},
        "roofline": roof,
        "stages": per,
        "e2e": {"value": (1 if sharded else world * ncube) * cfg.voxels / e2e_s, "unit": UNIT,
                "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes,
                "ms_per_step": e2e_s * 1e3, "steps": ne,
                "link_floor_ms": (link_s * 1e3) if link_s else None,
                "frac_of_link": (link_s / e2e_s) if link_s else None,
                "path": ("slab H2D + hyde_hyres_sharded + slab D2H per rank (pinned)" if sharded else
                         "hyde_hyres_host_stream (pinned host buffers; H2D of the next cube and D2H of "
                         "the previous one overlap the current cube)")},
        "gpu_launches": int(launches),
        "clocks": csum,
    }
    if iso is not None:
        line["wavelet_isolated"] = iso
    if reps is not None:
        line["replicas"] = reps
    if strm is not None:
        line["cube_stream"] = strm
    if hys is not None:
        line["hysime"] = hys
    if fpd is not None:
        line["forpdn"] = fpd
    if fpd_w is not None:
        line["wsrrr"] = fpd_w
    if fpd_h is not None:
        line["hyminor"] = fpd_h
    if world == 1 and not args.no_cpu_baseline:
        t, cores, thr = cpu_baseline(cubes_h[0], reps=2)
        line["cpu_baseline"] = {"value": cfg.voxels / t, "unit": UNIT, "cores": cores, "threads": thr,
                                "kind": "oracle",
                                "sample": f"2 full {cfg.name} cubes, oracle.hyres (numpy fp64), mean time"}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
