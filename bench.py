"""bench.py — throughput of the hot path of arXiv 1804.06304 on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl ours|reference]

One step = one pass of the whole hot path (resample
if anisotropic, Q14 blur + gradient magnitude, seeds, MC evolution of every
cell for T+1 iterations, E0 + overlap cull, label map) over one synthetic
volume resident in HBM.  Metric (BASELINE.json): contour ray-samples/s
(one ray-sample = one (cell, iteration, sample) triple, iteration T+1
included) and cells segmented/s.  N > 1: one process per GPU (torchrun),
z-slabs of the same volume (strong scaling), max over ranks.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402  (input generator: no method arithmetic)

METRIC = "contour ray-samples/sec and cells segmented/sec at 1/2/4/8 B200; HBM/L2 GB/s"
UNIT = "ray-samples/s"
# Algorithmic bytes per ray-sample: the d-linear gather reads
# 8 u16 taps in 3D (16 B) and 4 in 2D (8 B); the ray-march estimator (G27) also
# gathers one d-linear lookup per step.
GATHER_BYTES = {3: 16, 2: 8}
# Algorithmic issue slots per MC sample: Philox4x32-10 30 (3/4 block),
# uniforms 6, direction + radius 12 (5 SFU), position 3, d-linear gather 8 loads + 26 ALU,
# weights S, S_r, S_R 15, leaves 6, tree adds 5  ->  111 lane-ops per sample.
OPS_PER_SAMPLE = 111
# the estimator variants: control variate +1 (the subtraction);
# ray march (G27): Philox 3 blocks per 8-step ray 15, uniforms 2.5, direction per
# ray 1.25, step t 3, position 3, gather 34, t^2 weight 2, S 15, leaves 11 -> 87
OPS_BY_ESTIMATOR = {"mc": OPS_PER_SAMPLE, "cv": OPS_PER_SAMPLE + 1, "ray": 87}
# 2D (C2): Philox 1/2 block per sample 20, uniforms 4, direction + radius (sin, cos,
# sqrt) 8, position 2, bilinear gather 2 axes x 6 + 1 index + 4 conversions + 3 lerps x 2
# = 23 (+ 4 loads), S/S_r/S_R 15, leaves 4 + tree adds 4  ->  80
OPS_PER_SAMPLE_2D = 80
# L2 read bandwidth measured on this pool's B200 (scripts/micro/l2bw.cu,
# profiles/r2_l2bw.txt: best of the L2-resident working sets 16-96 MB)
L2_PEAK_GBPS = 19398.1
L2_PEAK_SOURCE = "measured, profiles/r2_l2bw.txt (scripts/micro/l2bw.cu)"
SMS = 148
LANES_PER_SM = 128


# ---------------------------------------------------------------- helpers
class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 4 + i and r[4 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    return int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0")), ws


def workload_name(cfg):
    iso = cfg.iso_n
    aniso = "" if tuple(iso) == tuple(cfg.n) else f" (raw {cfg.n[0]}x{cfg.n[1]}x{cfg.n[2]}, spacing {cfg.spacing})"
    dims = f"{iso[0]}x{iso[1]}" + (f"x{iso[2]}" if cfg.dim == 3 else "")
    nn = int(np.prod(cfg.count))
    return f"{cfg.name}: synthetic {dims}{aniso}, {nn} nuclei, N={cfg.n_samples}, T={cfg.max_iters}"


def hbm_peak():
    """The measured HBM copy bandwidth (MEASURED_PEAKS.json, driver-written), else
    B200_PROFILING.md's fallback."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured copy bandwidth)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "of fallback (B200_PROFILING.md: 6.65 TB/s)"


def spread(xs):
    """median and spread of per-step times (ms)."""
    return {"median": statistics.median(xs), "min": min(xs), "max": max(xs), "n": len(xs)}


def ncu_sol(config: str, kernel: str = "evolve_brick_kernel"):
    """the committed ncu --set full capture's speed-of-light
    percentages of the binding units (issue slots, shared-memory wavefronts)."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            e = json.load(f)[config][kernel]
        return {k: round(e[k] / 100.0, 4) for k in ("issue_pct", "shared_wavefront_pct") if k in e} | \
            {"source": e["source"]}
    except (OSError, KeyError, ValueError):
        return None


def workload_config(cfg, n_gpus=1, cull_every=0, estimator="mc", physical=False):
    """The `config` object of the JSON line: the workload definition only (both
    arms print the same one; measured counts such as cells and detections are
    top-level keys)."""
    iso = list(cfg.iso_n)
    vbytes = int(np.prod(iso)) * 2
    return {"workload": workload_name(cfg), "volume_iso": iso, "n_samples": cfg.n_samples,
            "iters": cfg.max_iters, "seed_mode": cfg.seed_mode,
            "parallelism": "1 GPU" if n_gpus <= 1 else f"z-slab x{n_gpus}", "cull_every": cull_every,
            "estimator": estimator, "physical": bool(physical),
            "l2": "inputs larger than L2 (u16 volume %.2f GiB > 126 MB)" % (vbytes / 2**30)
            if vbytes > 126 * 2**20 else "volume fits L2 (%.1f MiB); not flushed" % (vbytes / 2**20)}


def ncu_traffic(config: str, kernel: str = "evolve_brick_kernel"):
    """DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) per launch of the
    dominant kernel from the committed `ncu --set full` capture of this config
    (profiles/traffic.json, written from the .ncu-rep by scripts/ncu_traffic.py),
    or None when no capture of this config exists."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            t = json.load(f)
        e = t[config][kernel]
        return e["dram_bytes_per_launch"], e["source"]
    except (OSError, KeyError, ValueError):
        return None, None


# ---------------------------------------------------------------- CPU oracle sample
def crop_geometry(cfg, target_cells: int):
    """Crop box (lo, hi) and its seeded interior (ilo, ihi) for about target_cells cells."""
    n = cfg.iso_n
    vox_per_cell = float(np.prod(cfg.pitch[:cfg.dim])) / 1.5
    L = int(round((target_cells * vox_per_cell) ** (1.0 / cfg.dim)))
    L = max(32, min(L, min(n[:cfg.dim]) - 1))
    reach = int(math.ceil(4 * cfg.r0 + 1 + 2)) + 4
    c = [n[a] // 2 for a in range(3)]
    lo = [max(c[a] - L // 2 - reach, 0) if a < cfg.dim else 0 for a in range(3)]
    hi = [min(c[a] + L // 2 + reach, n[a] - 1) if a < cfg.dim else 0 for a in range(3)]
    ilo = [max(c[a] - L // 2, 0) if a < cfg.dim else 0 for a in range(3)]
    ihi = [min(c[a] + L // 2 - 1, n[a] - 1) if a < cfg.dim else 0 for a in range(3)]
    return lo, hi, ilo, ihi


def oracle_crop_run(cfg, raw_full, target_cells: int, threads: int):
    """The oracle as it stands on a bounded sample of the workload: a crop of the
    raw volume, a2 blur -> a4 maxima seeds (crop interior) -> a5/a6 evolution ->
    a7 cull.  raw_full: the (nz, ny, nx) volume, or a callable (lo, hi) -> crop.
    Returns (samples, seconds, description, cells)."""
    import oracle
    oracle.set_num_threads(threads)
    n = cfg.iso_n
    assert tuple(n) == tuple(cfg.n), "cpu sample needs an isotropic config"
    lo, hi, ilo, ihi = crop_geometry(cfg, target_cells)
    if callable(raw_full):
        crop = np.ascontiguousarray(raw_full(lo, hi))
    else:
        crop = np.ascontiguousarray(raw_full[lo[2]:hi[2] + 1, lo[1]:hi[1] + 1, lo[0]:hi[0] + 1])
    p = oracle.Params(r0=cfg.r0, n_samples=cfg.n_samples, max_iters=cfg.max_iters, dim=cfg.dim,
                      seed=cfg.philox_seed)
    t0 = time.perf_counter()
    B = oracle.blur(crop, cfg.dim, 1.0)
    seeds = oracle.seeds_maxima(B, cfg.dim, cfg.window, cfg.seed_threshold, org=lo, n_global=n,
                                lo=ilo, hi=ihi)
    cells = oracle.evolve(B, p, seeds, org=lo, n_global=n)
    oracle.cull(cells["c"].astype(np.float32), cells["R"].astype(np.float32),
                cells["E"].astype(np.float32), cells["flags"], cells["id"], cfg.dim, p.e0)
    dt = time.perf_counter() - t0
    samples = len(seeds) * (cfg.max_iters + 1) * cfg.n_samples
    desc = (f"{cfg.name} crop {hi[0]-lo[0]+1}x{hi[1]-lo[1]+1}x{hi[2]-lo[2]+1} at {lo}: a2 blur, a4 seeds, "
            f"a5/a6 evolution of {len(seeds)} cells, a7 cull (fp64 oracle, OpenMP)")
    return samples, dt, desc, len(seeds)


CPU_CELLS_PER_CORE = 100   # the crop sample (configs the plan below does not cover)
SUBSET = 100                # evolution of the cells with id = 0 mod 100
SLAB_PLANES = 16            # volume passes timed on a z-slab of this many owned planes


def cpu_sample(cfg, threads: int, part=None):
    """The crop sample (configs the SURVEY 8(d) plan does not cover: 2D and
    anisotropic raw grids): the centred crop of the workload holding
    ~CPU_CELLS_PER_CORE cells per core, a2 -> a4 -> a5/a6 -> a7 on it."""
    target = CPU_CELLS_PER_CORE * threads
    lo, hi, _, _ = crop_geometry(cfg, target)
    if part is None:
        part = synth.generate(cfg, lo[2], hi[2] + 1)

    def raw(lo_, hi_):
        return part[lo_[2] - lo[2]:hi_[2] - lo[2] + 1, lo_[1]:hi_[1] + 1, lo_[0]:hi_[0] + 1]
    return oracle_crop_run(cfg, raw, target_cells=target, threads=threads), part


class CpuPlan:
    """The oracle timed as SURVEY 8(d) plans it for the full-size 3D workloads:
    the volume passes (a2 blur, a4 MAXIMA) over a z-slab of SLAB_PLANES owned
    planes (+ their halo), extrapolated to the whole volume; the evolution
    (a5/a6) of the deterministic 1% subset (cells with id = 0 mod 100 of the
    full seed list), extrapolated to every cell; the a7 cull of the subset.
    Setup, untimed: the full volume's blur and seed list (the subset's inputs).
    Labels (a8) are not timed."""

    def __init__(self, cfg, threads: int, raw=None):
        import oracle
        self.cfg, self.threads = cfg, threads
        oracle.set_num_threads(threads)
        self.raw = synth.generate(cfg) if raw is None else raw
        self.B = oracle.blur(self.raw, 3, 1.0)
        if cfg.seed_mode == "lattice":
            self.seeds = oracle.seeds_lattice(cfg.n, 3, cfg.r0)[1]
        else:
            self.seeds = oracle.seeds_maxima(self.B, 3, cfg.window, cfg.seed_threshold)
        self.sub = np.arange(0, len(self.seeds), SUBSET, dtype=np.int64)
        self.p = oracle.Params(r0=cfg.r0, n_samples=cfg.n_samples, max_iters=cfg.max_iters, dim=3,
                               seed=cfg.philox_seed)
        nz = cfg.n[2]
        self.z0 = nz // 2 - SLAB_PLANES // 2
        self.z1 = self.z0 + SLAB_PLANES

    def step(self):
        import oracle
        cfg, nz = self.cfg, self.cfg.n[2]
        h = 4 + cfg.window   # blur radius ceil(4 sigma) + the MAXIMA window: the slab's halo
        lo, hi = max(self.z0 - h, 0), min(self.z1 + h, nz)
        t0 = time.perf_counter()
        Bs = oracle.blur(self.raw[lo:hi], 3, 1.0)   # the slab's planes blurred with its own halo
        if cfg.seed_mode != "lattice":
            oracle.seeds_maxima(Bs, 3, cfg.window, cfg.seed_threshold, org=(0, 0, lo), n_global=cfg.n,
                                lo=(0, 0, self.z0), hi=(cfg.n[0] - 1, cfg.n[1] - 1, self.z1 - 1))
        t_vol = time.perf_counter() - t0
        t0 = time.perf_counter()
        cells = oracle.evolve(self.B, self.p, self.seeds[self.sub], ids=self.sub)
        t_evo = time.perf_counter() - t0
        t0 = time.perf_counter()
        oracle.cull(cells["c"].astype(np.float32), cells["R"].astype(np.float32),
                    cells["E"].astype(np.float32), cells["flags"], cells["id"], 3, self.p.e0)
        t_cull = time.perf_counter() - t0
        n, k = len(self.seeds), len(self.sub)
        t_full = t_vol * nz / SLAB_PLANES + t_evo * n / k + t_cull
        return {"seconds_full_extrapolated": t_full, "seconds_measured": t_vol + t_evo + t_cull,
                "samples_full": n * (cfg.max_iters + 1) * cfg.n_samples,
                "t_volume_slab": t_vol, "t_evolve_subset": t_evo, "t_cull_subset": t_cull}

    def describe(self):
        return (f"{self.cfg.name}, SURVEY 8(d) plan, EXTRAPOLATED: a2 blur + a4 MAXIMA on planes "
                f"[{self.z0}, {self.z1}) + halo x {self.cfg.n[2] // SLAB_PLANES}; a5/a6 evolution of the "
                f"{len(self.sub)} cells with id = 0 mod {SUBSET} of {len(self.seeds)} x {SUBSET}; "
                f"a7 cull of the subset; a8 not timed (fp64 oracle, OpenMP, {self.threads} threads)")


def plan_applies(cfg) -> bool:
    return cfg.dim == 3 and tuple(cfg.iso_n) == tuple(cfg.n) and cfg.n[2] >= 4 * SLAB_PLANES


def cpu_baseline_entry(cfg, raw=None):
    threads = os.cpu_count() or 1
    if plan_applies(cfg):
        plan = CpuPlan(cfg, threads, raw)
        r = plan.step()
        v = r["samples_full"] / r["seconds_full_extrapolated"]
        return {"value": v, "unit": UNIT, "cores": threads, "kind": "oracle", "sample": plan.describe(),
                "extrapolated": True, "seconds_measured": round(r["seconds_measured"], 2),
                "seconds_full_extrapolated": round(r["seconds_full_extrapolated"], 1),
                "cells_per_s": len(plan.seeds) / r["seconds_full_extrapolated"]}
    (s, dt, desc, nc), _ = cpu_sample(cfg, threads)
    return {"value": s / dt, "unit": UNIT, "cores": threads, "kind": "oracle", "sample": desc,
            "seconds": round(dt, 2), "cells_per_s": nc / dt}


# ---------------------------------------------------------------- our arm
def run_ours(args):
    import torch
    rank, local_rank, world = dist_env()
    cfg = synth.CONFIGS[args.config]
    if args.n_samples:   # sweeps (e.g. the C5 N-sweep); the headline uses the config's N
        cfg = cfg.with_(n_samples=args.n_samples)
    if world > 1 or args.dist:
        if "WORLD_SIZE" not in os.environ:   # --dist at N = 1 without a launcher
            os.environ.update(RANK="0", LOCAL_RANK="0", WORLD_SIZE="1", MASTER_ADDR="127.0.0.1",
                              MASTER_PORT=str(_free_port()))
        from paper_1804_06304_b200 import dist as D
        return D.bench_rank(args, cfg)
    torch.cuda.set_device(local_rank)
    from paper_1804_06304_b200 import pipeline, snk
    p = pipeline.params_for(cfg, image_term=snk.IMAGE_INTENSITY, cta_warps=args.cta_warps,
                            kernel_variant=args.kernel_variant, cull_every=args.cull_every,
                            estimator={"mc": snk.EST_MC, "cv": snk.EST_MC_CV, "ray": snk.EST_RAY}[args.estimator])
    # the gradient magnitude (a3) only when the image term uses it
    P = pipeline.Pipeline(cfg.dim, cfg.n, p, spacing=cfg.spacing, gradmag=False, physical=args.physical)
    h_raw = torch.empty((cfg.n[2], cfg.n[1], cfg.n[0]), dtype=torch.uint16, pin_memory=True)
    t = time.perf_counter()
    synth.generate_into_ptr(cfg, h_raw.data_ptr())
    gen_s = time.perf_counter() - t
    P.upload(h_raw)
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()

    def step(ev=None):
        if ev is not None:
            ev[0].record(stream)
        P.preprocess()
        P.seed()
        if ev is not None:
            ev[1].record(stream)
        P.evolve()
        if ev is not None:
            ev[2].record(stream)
        P.cull()
        P.label()
        if ev is not None:
            ev[3].record(stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    l0 = snk.snk_launch_count()
    with ClockSampler(local_rank) as clk:
        torch.cuda.synchronize()
        start = torch.cuda.Event(enable_timing=True)
        end = torch.cuda.Event(enable_timing=True)
        start.record(stream)
        for k in range(args.steps):
            step(evs[k])
        end.record(stream)
        torch.cuda.synchronize()
    launches = snk.snk_launch_count() - l0
    evo_stats = snk.snk_evolve_stats(reset=True)
    total_ms = start.elapsed_time(end)
    evolve_ms = [e[1].elapsed_time(e[2]) for e in evs]
    n_cells = P.n_seeds
    n_iso_l, n_dets = list(P.n_iso), P.n_dets
    # ray-samples evaluated per step (with periodic culling: only the live cells' iterations)
    samples = P.cell_iters * cfg.n_samples
    value = samples * args.steps / (total_ms / 1e3)
    cells_per_s = n_cells * args.steps / (total_ms / 1e3)
    phase_lists = {"preprocess+seeds": [e[0].elapsed_time(e[1]) for e in evs], "evolve": evolve_ms,
                   "cull+label": [e[2].elapsed_time(e[3]) for e in evs]}
    phase = {k: statistics.median(v) for k, v in phase_lists.items()}
    clocks = clk.summary()
    # Roofline of the dominant kernel: (ii) the algorithmic gather
    # bytes (16 B per 3D sample, 8 B per 2D sample) per launch / its device time
    # against the measured HBM peak and the measured L2 peak; (i) the binding
    # units' SOL from the committed ncu capture of the same config; and the
    # instruction-issue model (lane-ops) for reference.
    ev_s = statistics.median(evolve_ms) / 1e3
    gbytes = GATHER_BYTES[cfg.dim]
    achieved = samples * gbytes / ev_s / 1e9
    hbm, hbm_src = hbm_peak()
    f_clk = (clocks["sm_max_mhz"] or 1965.0) * 1e6
    lane_peak = SMS * LANES_PER_SM * f_clk / 1e9            # G lane-ops/s
    ops = OPS_BY_ESTIMATOR[args.estimator] if cfg.dim == 3 else OPS_PER_SAMPLE_2D
    traffic, traffic_src = ncu_traffic(cfg.name) if not args.cull_every else (None, None)
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s",
                "frac": round(achieved / hbm, 4), "traffic": traffic,
                "peak_source": hbm_src,
                "l2": {"achieved": round(achieved, 1), "peak": L2_PEAK_GBPS, "unit": "GB/s",
                       "frac": round(achieved / L2_PEAK_GBPS, 4), "peak_source": L2_PEAK_SOURCE},
                "sol_ncu": ncu_sol(cfg.name) if not args.cull_every else None,
                "alu_model": {"achieved": round(samples * ops / ev_s / 1e9, 1), "peak": round(lane_peak, 1),
                              "unit": "Glane-op/s", "frac": round(samples * ops / ev_s / 1e9 / lane_peak, 4),
                              "ops_per_sample": ops,
                              "peak_source": f"{SMS} SMs x {LANES_PER_SM} FP32 lanes x sm_max_mhz"},
                "algorithmic_bytes_per_sample": gbytes,
                "algorithmic_gather_bytes_per_launch": samples * gbytes,
                "traffic_unit": "DRAM bytes per launch (ncu --set full)", "traffic_source": traffic_src,
                "kernel": "evolve_brick_kernel" if args.kernel_variant != 1 else "evolve_warp_kernel",
                "samples_per_s_kernel": samples / ev_s,
                "timing": "CUDA events around the evolve launch on its stream, median over the timed steps"}
    # end to end through the public host-buffer call (snk_run)
    e2e = None
    if not args.no_e2e and not args.physical:   # snk_run resamples anisotropic input (a1)
        niso = int(np.prod(n_iso_l))
        max_cells = P.max_cells
        del P
        torch.cuda.empty_cache()
        if args.e2e_mode == "batch":
            # the end-to-end call for a stream of volumes (snk_run_batch): each of
            # the K steps uploads its raw volume from pinned host memory and
            # downloads its detections + label map; the next upload and the
            # previous download overlap the current step's kernels
            br = pipeline.BatchRunner(cfg.dim, cfg.n, p, spacing=cfg.spacing, max_cells=max_cells)
            br.run([h_raw] * max(2, args.warmup))
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            nds = br.run([h_raw] * args.steps)
            e2e_s = time.perf_counter() - t0
            nd, k = nds[-1], 2
            del br
        else:
            # snk_run (one volume per call) from `inflight` host threads, each with
            # its own runner and a stream of distinct priority
            import concurrent.futures as cf
            k = max(1, min(args.e2e_inflight, args.steps))
            runners = [pipeline.HostRunner(cfg.dim, cfg.n, p, spacing=cfg.spacing, max_cells=max_cells)
                       for _ in range(k)]
            lo, hi = torch.cuda.Stream.priority_range()
            streams = [torch.cuda.Stream(priority=(hi if i == 0 else lo) if args.e2e_priorities else 0)
                       for i in range(k)]
            nds = [0] * k

            def work(i, nsteps, delay=0.0):
                torch.cuda.set_device(local_rank)
                time.sleep(delay)
                for _ in range(nsteps):
                    nds[i] = runners[i].run(h_raw, streams[i])

            for i in range(k):
                for _ in range(max(1, args.warmup // k)):
                    work(i, 1)
            torch.cuda.synchronize()
            share = [args.steps // k + (1 if i < args.steps % k else 0) for i in range(k)]
            delays = [i * (total_ms / args.steps) / 1e3 / k for i in range(k)]
            t0 = time.perf_counter()
            with cf.ThreadPoolExecutor(k) as ex:
                list(ex.map(work, range(k), share, delays))
            e2e_s = time.perf_counter() - t0
            nd = nds[0]
            del runners
        e2e = {"value": samples * args.steps / e2e_s, "unit": UNIT,
               "h2d_bytes_per_step": int(h_raw.numel() * 2),
               "d2h_bytes_per_step": int(nd * 64 + niso * 4),
               "cells_per_s": n_cells * args.steps / e2e_s, "inflight": k, "mode": args.e2e_mode}
    cpu = None
    if not args.no_cpu_baseline and cfg.dim == 3 and tuple(cfg.iso_n) == tuple(cfg.n):
        cpu = cpu_baseline_entry(cfg, raw=h_raw.numpy())
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": workload_config(cfg, 1, args.cull_every, args.estimator, args.physical),
        "cells": n_cells, "detections": n_dets, "cells_per_s": cells_per_s, "phase_ms": phase,
        "phase_ms_spread": {k: spread(v) for k, v in phase_lists.items()}, "gpu_launches": int(launches),
        "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks,
        "generate_s": round(gen_s, 2),
        "evolve_stats_per_step": {k: v / (args.steps + args.warmup) for k, v in evo_stats.items()},
    }
    return out


# ---------------------------------------------------------------- reference arm (the oracle)
def run_reference(args):
    """The oracle as it stands on the host cores, on our arm's workload and metric
    (the SURVEY 8(d) plan where it applies: every step re-times the slab volume
    passes and the 1% evolution subset, extrapolated; else the crop sample)."""
    rank, _, world = dist_env()
    if rank != 0:
        return None
    cfg = synth.CONFIGS[args.config]
    threads = os.cpu_count() or 1
    samples = secs = 0.0
    if plan_applies(cfg):
        plan = CpuPlan(cfg, threads)
        for k in range(args.warmup + args.steps):
            r = plan.step()
            if k >= args.warmup:
                samples += r["samples_full"]
                secs += r["seconds_full_extrapolated"]
        desc, extra = plan.describe(), {"extrapolated": True}
        cells = len(plan.seeds)
    else:
        part = None
        desc, cells = "", 0
        for k in range(args.warmup + args.steps):
            (s, dt, desc, cells), part = cpu_sample(cfg, threads, part)
            if k >= args.warmup:
                samples += s
                secs += dt
        extra = {}
    v = samples / secs
    return {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": max(world, args.gpus),
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": secs / args.steps * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": workload_config(cfg, max(world, args.gpus)),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "oracle", "sample": desc, **extra},
            "cells_per_s": cells * args.steps / secs,
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def _free_port() -> int:
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def launch_ranks(n: int) -> int:
    """`bench.py --gpus N` without a launcher: start N ranks (one process per
    GPU) through torch.distributed.run on 127.0.0.1 and return their exit code;
    rank 0 prints the JSON line."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def launch_check(args):
    """--launch-check: the rank plumbing alone (no kernels): every rank joins the
    process group (gloo), the ranks are all-gathered; rank 0 reports the world."""
    import torch
    import torch.distributed as tdist
    rank, _, world = dist_env()
    tdist.init_process_group("gloo")
    got = [None] * world
    tdist.all_gather_object(got, rank)
    tdist.destroy_process_group()
    assert world == args.gpus and got == list(range(world)), (world, got)
    return {"launch_check": True, "n_gpus": world, "ranks": got}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C4")
    ap.add_argument("--n-samples", type=int, default=0, help="override the config's N (sweeps only)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cta-warps", type=int, default=0, help="warps per cell (0: auto)")
    ap.add_argument("--kernel-variant", type=int, default=0, help="evolve kernel: 0 auto, 1 warp, 2 brick")
    ap.add_argument("--estimator", default="mc", choices=["mc", "cv", "ray"],
                    help="MC (the paper's), MC + control variate (G21) or stratified ray march (G27)")
    ap.add_argument("--physical", action="store_true",
                    help="anisotropic configs: sample the raw grid in physical coordinates, no resampling (G28)")
    ap.add_argument("--cull-every", type=int, default=0,
                    help="periodic culling every k iterations (P:326, G25); 0 = the paper's end-of-run cull")
    ap.add_argument("--e2e-mode", default="batch", choices=["batch", "threads"],
                    help="end to end through snk_run_batch (copies overlapped inside the call) or snk_run threads")
    ap.add_argument("--e2e-priorities", type=int, default=1, help="threads mode: distinct stream priorities")
    ap.add_argument("--e2e-inflight", type=int, default=2, help="steps in flight in the end-to-end run")
    ap.add_argument("--dist", action="store_true",
                    help="run through the z-slab driver (dist.py) even at N = 1 (NCCL world of one)")
    ap.add_argument("--launch-check", action="store_true", help="check the rank launch only (no kernels)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3   # contract: at least 3 warm-up steps
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        sys.exit(launch_ranks(args.gpus))
    if args.launch_check:
        out = launch_check(args)
    else:
        out = run_reference(args) if args.impl == "reference" else run_ours(args)
    rank, _, _ = dist_env()
    if out is not None and rank == 0:
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
