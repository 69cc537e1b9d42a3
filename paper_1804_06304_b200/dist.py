"""Multi-GPU z-slab driver: one process per GPU,
torch.distributed for the plumbing (NCCL on GPUs; gloo in the CPU tests).

Partition.  Rank r owns the isotropic planes [z0_r, z1_r) (equal split) and
holds raw planes [z0 - H - h, z1 + H + h) clipped to the volume, where
h = ceil(4 sigma) is the blur radius and H = ceil(leash + r_max + dR/2) + 2
bounds every voxel a cell seeded in [z0, z1) can read (leash per component,
sampled ball radius, trilinear +1) — so seeds, cells, detections and labels
are bit-identical to one GPU.

Exchange steps (the only ones the method has):
  N1  raw halo planes from the ranks that own them (P2P, once per step);
  N2  all_gather of per-rank seed counts -> global ids = exclusive prefix
      (slabs are contiguous in linear-index order, so ids equal one GPU's);
  N3  all_gather of the E0 candidates (64-byte snk_cell records); every rank
      then runs the identical deterministic cull (the overlap competition
      crosses slab boundaries);
  labels stay distributed (each rank labels its own planes).
Cells never interact during evolution, so nothing is exchanged per
iteration — except with periodic culling (cull_every = k > 0, G25):
  N6  at every checkpoint (after iterations k, 2k, ... < T) the E0 candidates
      are all-gathered, every rank runs the same cull, and each rank keeps the
      survivors it owns (its id range) — the per-checkpoint exchange of
      boundary-cell records, results still bit-identical to one GPU.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import torch
import torch.distributed as tdist

CELL_BYTES = 64   # sizeof(snk_cell) (include/snk.h); kept here so the driver imports without libsnk


@dataclass
class SlabPlan:
    n: tuple            # global isotropic dims (x, y, z)
    world: int
    rank: int
    own: tuple          # owned planes [z0, z1)
    halo: int           # H
    blur: int           # h
    buf: tuple          # raw / smoothed buffer planes [lo, hi)

    @property
    def nz_buf(self) -> int:
        return self.buf[1] - self.buf[0]


def slab_bounds(nz: int, world: int, r: int) -> tuple:
    base, rem = divmod(nz, world)
    z0 = r * base + min(r, rem)
    return z0, z0 + base + (1 if r < rem else 0)


def halo_planes(params) -> int:
    return int(math.ceil(params.leash + params.r_max + params.delta_R / 2.0)) + 2


def plan_slabs(n, world: int, rank: int, params) -> SlabPlan:
    n = tuple(int(a) for a in n)
    z0, z1 = slab_bounds(n[2], world, rank)
    H = max(halo_planes(params), int(getattr(params, "seed_window", 0)))
    h = int(math.ceil(4.0 * params.sigma)) if params.sigma > 0 else 0
    lo, hi = max(z0 - H - h, 0), min(z1 + H + h, n[2])
    return SlabPlan(n=n, world=world, rank=rank, own=(z0, z1), halo=H, blur=h, buf=(lo, hi))


def _staged(group) -> bool:
    """gloo moves host memory only: CUDA tensors are staged through the host
    (used when several ranks share one GPU, where NCCL refuses; GPU tests)."""
    return tdist.get_backend(group) == "gloo"


def exchange_halo(plan: SlabPlan, own_raw: torch.Tensor, group=None) -> torch.Tensor:
    """N1: assemble raw planes [buf) from this rank's own planes and the other
    ranks' (point-to-point; each rank sends exactly what the others need)."""
    if own_raw.is_cuda and _staged(group):
        return exchange_halo(plan, own_raw.cpu(), group).to(own_raw.device)
    nz = plan.n[2]
    lo, hi = plan.buf
    z0, z1 = plan.own
    plane_shape = own_raw.shape[1:]
    out = torch.empty((hi - lo,) + tuple(plane_shape), dtype=own_raw.dtype, device=own_raw.device)
    out[z0 - lo:z1 - lo].copy_(own_raw)
    ops = []
    recv = []
    for q in range(plan.world):
        if q == plan.rank:
            continue
        q0, q1 = slab_bounds(nz, plan.world, q)
        # what I need from q
        a, b = max(lo, q0), min(hi, q1)
        if a < b:
            buf = out[a - lo:b - lo]
            t = buf if buf.is_contiguous() else torch.empty_like(buf)
            ops.append(tdist.P2POp(tdist.irecv, _wire(t), q, group))
            recv.append((buf, t))
        # what q needs from me
        qp = plan_like(plan, q)
        a, b = max(qp.buf[0], z0), min(qp.buf[1], z1)
        if a < b:
            ops.append(tdist.P2POp(tdist.isend, _wire(own_raw[a - z0:b - z0].contiguous()), q, group))
    if ops:
        for r in tdist.batch_isend_irecv(ops):
            r.wait()
    for buf, t in recv:
        if t.data_ptr() != buf.data_ptr():
            buf.copy_(t)
    return out


def _wire(t: torch.Tensor) -> torch.Tensor:
    """u16 planes travel as bytes (NCCL has no 16-bit integer type; gloo no uint16)."""
    return t.view(torch.uint8) if t.dtype == torch.uint16 else t


def plan_like(plan: SlabPlan, rank: int) -> SlabPlan:
    z0, z1 = slab_bounds(plan.n[2], plan.world, rank)
    H, h = plan.halo, plan.blur
    return SlabPlan(n=plan.n, world=plan.world, rank=rank, own=(z0, z1), halo=H, blur=h,
                    buf=(max(z0 - H - h, 0), min(z1 + H + h, plan.n[2])))


def allgather_counts(count: int, device, group=None) -> list:
    """N2: every rank's count."""
    if _staged(group):
        device = torch.device("cpu")
    t = torch.tensor([count], dtype=torch.int64, device=device)
    outs = [torch.empty_like(t) for _ in range(tdist.get_world_size(group))]
    tdist.all_gather(outs, t, group=group)
    return [int(o.item()) for o in outs]


def allgather_records(rec: torch.Tensor, count: int, device, group=None, rec_bytes: int = CELL_BYTES, meta=None):
    """N3: concatenate every rank's `count` records (uint8, rec_bytes each) in rank order.
    meta: an optional host-side (gloo) group for the counts."""
    if _staged(group) and torch.device(device).type == "cuda":
        allrec, tot, counts = allgather_records(rec[:count * rec_bytes].cpu(), count, "cpu", group, rec_bytes)
        return allrec.to(device), tot, counts
    counts = allgather_counts(count, device, group if meta is None else meta)
    m = max(max(counts), 1)
    pad = torch.zeros(m * rec_bytes, dtype=torch.uint8, device=device)
    if count:
        pad[:count * rec_bytes].copy_(rec[:count * rec_bytes])
    outs = [torch.empty_like(pad) for _ in counts]
    tdist.all_gather(outs, pad, group=group)
    allrec = torch.cat([o[:c * rec_bytes] for o, c in zip(outs, counts)])
    return allrec, sum(counts), counts


def checkpoints(T: int, k: int) -> list:
    """Periodic-culling segments (G25): [1, k], [k+1, 2k], ..., the last one
    ending at T + 1; a checkpoint cull after each but the last."""
    if k <= 0 or k >= T:
        return [(1, T + 1)]
    ends = list(range(k, T, k)) + [T + 1]
    return list(zip([1] + [e + 1 for e in ends[:-1]], ends))


class SlabRun:
    """One rank's share of one step: N1 -> a2/a3 -> a4 -> N2 -> a5/a6 -> a7
    (compact, N3, cull) -> a8.  `backend` supplies the per-stage compute:
    CudaBackend (libsnk) in production; the tests plug in the CPU oracle to check
    the decomposition logic with gloo.  cull_every > 0: periodic culling with
    the N6 exchange at every checkpoint (T = max_iters)."""

    def __init__(self, plan: SlabPlan, backend, device, group=None, cull_every: int = 0,
                 max_iters: int = 0, meta_group=None):
        self.plan, self.be, self.device, self.group = plan, backend, device, group
        self.cull_every, self.T = cull_every, max_iters
        # meta_group (gloo): the per-rank counts travel host to host, so reading
        # them never waits behind a bulk device-to-host copy on the copy engine
        self.meta = meta_group

    def step(self, own_raw: torch.Tensor, ev=None) -> dict:
        """ev: optional pair of CUDA events recorded around a5/a6 (bench)."""
        pl = self.plan
        local = exchange_halo(pl, own_raw, self.group)                 # N1
        smooth = self.be.preprocess(pl, local)                          # a2/a3
        seeds, ns = self.be.seeds(pl, smooth)                           # a4
        counts = allgather_counts(ns, self.device, self.group if self.meta is None else self.meta)   # N2
        id_base = sum(counts[:pl.rank])
        if ev is not None:
            ev[0].record()
        live = ns
        cell_iters = ns * (self.T + 1)   # cell-iterations evolved by this rank (each N samples)
        if self.cull_every > 0:
            cells = self.be.init_cells(pl, seeds, ns, id_base)
            segs = checkpoints(self.T, self.cull_every)
            cell_iters = 0
            for i, (a, b) in enumerate(segs):
                cells = self.be.evolve_range(pl, smooth, cells, live, a, b)    # a5 segment
                cell_iters += live * (b - a + 1)
                if i + 1 < len(segs):                                           # checkpoint
                    cand, nc = self.be.compact(cells, live)
                    allc, ntot, _ = allgather_records(cand, nc, self.device, self.group, meta=self.meta)   # N6
                    surv, nsurv = self.be.cull(pl, allc, ntot)
                    cells, live = self.be.select_ids(surv, nsurv, id_base, id_base + ns)
        else:
            cells = self.be.evolve(pl, smooth, seeds, ns, id_base)      # a5/a6
        if ev is not None:
            ev[1].record()
        cand, nc = self.be.compact(cells, live)                         # a7: E0
        allc, ntot, _ = allgather_records(cand, nc, self.device, self.group, meta=self.meta)   # N3
        dets, nd = self.be.cull(pl, allc, ntot)                         # a7: overlap
        labels = self.be.label(pl, dets, nd)                            # a8
        return {"n_seeds": ns, "n_live": live, "id_base": id_base, "n_total": sum(counts), "cells": cells,
                "cell_iters": cell_iters,
                "seeds": seeds, "dets": dets, "n_dets": nd, "labels": labels, "smooth": smooth}


class CudaBackend:
    """libsnk on this rank's GPU; buffers are reused across steps."""

    def __init__(self, plan: SlabPlan, params, max_cells: int, gradmag: bool = True):
        from . import snk
        self.snk = snk
        self.p = params
        n, (lo, hi) = plan.n, plan.buf
        self.grid = snk.make_grid(3, n, z_lo=lo, nz_buf=hi - lo, own=plan.own)
        shape = (hi - lo, n[1], n[0])
        dev = torch.device("cuda", torch.cuda.current_device())
        self.smooth = torch.empty(shape, dtype=torch.uint16, device=dev)
        self.grad = torch.empty(shape, dtype=torch.uint16, device=dev) if gradmag else None
        self.max_cells = max_cells
        self.seeds_t = torch.empty((max_cells, 3), dtype=torch.float32, device=dev)
        self.cells = torch.empty(max_cells * CELL_BYTES, dtype=torch.uint8, device=dev)
        self.cand = torch.empty(max_cells * CELL_BYTES, dtype=torch.uint8, device=dev)
        self.total_cap = max_cells * plan.world
        self.dets = torch.empty(self.total_cap * CELL_BYTES, dtype=torch.uint8, device=dev)
        self.labels = torch.empty((plan.own[1] - plan.own[0], n[1], n[0]), dtype=torch.int32, device=dev)
        ws = max(snk.snk_workspace_bytes(self.grid, params, self.total_cap), 1)
        self.ws = torch.empty(ws, dtype=torch.uint8, device=dev)

    def preprocess(self, pl, local):
        self.snk.snk_preprocess(self.grid, self.p, local, self.smooth, self.grad, self.ws)
        return self.smooth

    def seeds(self, pl, smooth):
        n, _ = self.snk.snk_seeds(self.grid, self.p, smooth, self.seeds_t, self.max_cells, self.ws)
        return self.seeds_t, n

    def evolve(self, pl, smooth, seeds, n, id_base):
        img = self.grad if self.p.image_term == self.snk.IMAGE_GRADMAG else smooth
        if n:
            self.snk.snk_evolve(self.grid, self.p, img, seeds, None, id_base, n, self.cells, None)
        return self.cells

    def init_cells(self, pl, seeds, n, id_base):
        self.snk.snk_cells_init(self.p, seeds, None, id_base, n, self.cells)
        return self.cells

    def evolve_range(self, pl, smooth, cells, n, it0, it1):
        img = self.grad if self.p.image_term == self.snk.IMAGE_GRADMAG else smooth
        self.snk.snk_evolve_range(self.grid, self.p, img, cells, n, it0, it1, None)
        return cells

    def select_ids(self, recs, n, id_lo, id_hi):
        nl = self.snk.snk_select_ids(recs, n, id_lo, id_hi, self.cells, self.max_cells, self.ws)
        return self.cells, nl

    def compact(self, cells, n):
        return self.cand, self.snk.snk_compact_candidates(self.p, cells, n, self.cand, self.max_cells,
                                                          self.ws)

    def cull(self, pl, allc, ntot):
        nd = self.snk.snk_cull(self.grid, self.p, allc, ntot, self.dets, self.total_cap, self.ws)
        return self.dets, nd

    def label(self, pl, dets, nd):
        self.snk.snk_label(self.grid, self.p, dets, nd, self.labels, self.ws)
        return self.labels


def bench_rank(args, cfg):
    """bench.py for N > 1 ranks: z-slabs of one volume (strong scaling); timed on
    the device with CUDA events, max over ranks; rank 0 returns the JSON dict."""
    import os
    import statistics
    import time

    import numpy as np

    import synth
    from . import pipeline, snk

    rank, local_rank, world = (int(os.environ.get(k, d)) for k, d in
                               (("RANK", "0"), ("LOCAL_RANK", "0"), ("WORLD_SIZE", "1")))
    local_rank %= max(torch.cuda.device_count(), 1)   # ranks > GPUs: share (gloo tests only)
    torch.cuda.set_device(local_rank)
    # SNK_DIST_BACKEND=gloo: several ranks on one GPU (host-staged exchanges; tests only)
    backend = os.environ.get("SNK_DIST_BACKEND", "nccl")
    want = int(getattr(args, "gpus", world) or world)
    assert world == want, f"launched with WORLD_SIZE={world} but --gpus {want}"
    if backend == "nccl":
        # keep NCCL's communicator set-up lines (rank, device, transport) in the log
        # (images may preset NCCL_DEBUG=VERSION / WARN, which hides them)
        if os.environ.get("NCCL_DEBUG", "").upper() in ("", "VERSION", "WARN"):
            os.environ["NCCL_DEBUG"] = "INFO"
            os.environ["NCCL_DEBUG_SUBSYS"] = "INIT"
        # NCCL logs to stdout by default: keep stdout for the one JSON line
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        tdist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    else:
        tdist.init_process_group(backend)
    tdist.barrier()   # a collective over all ranks before the first point-to-point batch (NCCL)
    assert tuple(cfg.iso_n) == tuple(cfg.n), "the slab driver takes isotropic volumes"
    p = pipeline.params_for(cfg, image_term=snk.IMAGE_INTENSITY, cull_every=getattr(args, "cull_every", 0))
    plan = plan_slabs(cfg.n, world, rank, p)
    z0, z1 = plan.own
    nown = (z1 - z0) * cfg.n[0] * cfg.n[1]
    max_cells = max(4096, (plan.nz_buf * cfg.n[0] * cfg.n[1]) // (2 * cfg.window + 1) ** 3 + 4096)
    be = CudaBackend(plan, p, max_cells, gradmag=p.image_term == snk.IMAGE_GRADMAG)
    h_raw = torch.empty((z1 - z0, cfg.n[1], cfg.n[0]), dtype=torch.uint16, pin_memory=True)
    synth.generate_into_ptr(cfg, h_raw.data_ptr(), z0, z1)
    own = torch.empty(h_raw.shape, dtype=torch.uint16, device="cuda")
    own.copy_(h_raw)
    # the seed / candidate counts go host to host over gloo (a D2H read of an
    # NCCL-gathered count would queue behind the end-to-end loop's bulk copies)
    meta = tdist.new_group(backend="gloo") if backend == "nccl" else None
    run = SlabRun(plan, be, torch.device("cuda", local_rank), cull_every=p.cull_every,
                  max_iters=p.max_iters, meta_group=meta)
    for _ in range(args.warmup):
        r = run.step(own)
    torch.cuda.synchronize()
    tdist.barrier()
    l0 = snk.snk_launch_count()
    from bench import ClockSampler, GATHER_BYTES, L2_PEAK_GBPS, hbm_peak, workload_config  # noqa: E402
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(args.steps)]
    with ClockSampler(local_rank) as clk:
        torch.cuda.synchronize()
        tdist.barrier()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for k in range(args.steps):
            r = run.step(own, evs[k])
        e.record()
        torch.cuda.synchronize()
        tdist.barrier()
    red_dev = "cpu" if backend == "gloo" else "cuda"
    evolve_ms = statistics.median(a.elapsed_time(b) for a, b in evs)
    ms = torch.tensor([s.elapsed_time(e), evolve_ms], dtype=torch.float64, device=red_dev)
    tdist.all_reduce(ms, op=tdist.ReduceOp.MAX)
    total_ms, evolve_ms_max = float(ms[0].item()), float(ms[1].item())
    launches = snk.snk_launch_count() - l0
    n_total = r["n_total"]
    # ray-samples evaluated (with periodic culling only the live cells' iterations), all ranks
    ci = torch.tensor([r["cell_iters"]], dtype=torch.int64, device=red_dev)
    tdist.all_reduce(ci, op=tdist.ReduceOp.SUM)
    samples = int(ci.item()) * cfg.n_samples
    # this rank's evolve kernel: algorithmic gather bytes / its device time (SURVEY
    # 8(d)(ii)) against the per-GPU HBM and L2 peaks; the mean over ranks
    my_samples = r["cell_iters"] * cfg.n_samples
    clocks = clk.summary()
    hbm, hbm_src = hbm_peak()
    ach = torch.tensor([my_samples * GATHER_BYTES[cfg.dim] / (evolve_ms / 1e3) / 1e9], dtype=torch.float64,
                       device=red_dev)
    tdist.all_reduce(ach, op=tdist.ReduceOp.SUM)
    achieved = float(ach.item()) / world
    # end to end: each step copies this rank's raw planes in (pinned host -> device)
    # and its labels + the detections out, wall clock, max over ranks
    h_labels = torch.empty(tuple(be.labels.shape), dtype=torch.int32, pin_memory=True)
    h_dets = torch.empty(be.dets.numel(), dtype=torch.uint8, pin_memory=True)
    # double-buffered: step k+1's planes go up and step k's labels / detections
    # come down on two copy streams while the next step computes (each step's
    # outputs are first snapshotted on the compute stream, device to device)
    comp, cs, cd = torch.cuda.current_stream(), torch.cuda.Stream(), torch.cuda.Stream()   # compute, up, down
    owns = [own, torch.empty_like(own)]
    labs = [torch.empty_like(be.labels) for _ in range(2)]
    dsnap = [torch.empty_like(be.dets) for _ in range(2)]
    up = [torch.cuda.Event() for _ in range(2)]
    done = [torch.cuda.Event() for _ in range(2)]
    down = [torch.cuda.Event() for _ in range(2)]
    tdist.barrier()
    t0 = time.perf_counter()
    with torch.cuda.stream(cs):
        owns[0].copy_(h_raw, non_blocking=True)
        up[0].record(cs)
    for k in range(args.steps):
        b = k & 1
        if k + 1 < args.steps:   # step k+1's upload runs under step k (the driver syncs the host inside a step)
            with torch.cuda.stream(cs):
                if k >= 1:
                    cs.wait_event(done[b ^ 1])   # step k-1 has finished reading owns[b ^ 1]
                owns[b ^ 1].copy_(h_raw, non_blocking=True)
                up[b ^ 1].record(cs)
        comp.wait_event(up[b])
        r = run.step(owns[b])
        nb = r["n_dets"] * CELL_BYTES
        if k >= 2:
            comp.wait_event(down[b])   # step k-2's downloads are done with labs[b] / dsnap[b]
        labs[b].copy_(r["labels"])
        dsnap[b][:nb].copy_(r["dets"][:nb])
        done[b].record(comp)
        with torch.cuda.stream(cd):
            cd.wait_event(done[b])
            h_labels.copy_(labs[b], non_blocking=True)
            h_dets[:nb].copy_(dsnap[b][:nb], non_blocking=True)
            down[b].record(cd)
    torch.cuda.synchronize()
    del owns, labs, dsnap
    wall = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=red_dev)
    tdist.all_reduce(wall, op=tdist.ReduceOp.MAX)
    e2e_s = float(wall.item())
    # the oracle's bounded sample on rank 0's host cores (after the timed regions)
    cpu = None
    if rank == 0 and not getattr(args, "no_cpu_baseline", False):
        from bench import cpu_baseline_entry  # noqa: E402
        cpu = cpu_baseline_entry(cfg)   # the whole workload's plan (rank 0 generates the volume)
    out = None
    if rank == 0:
        out = {"metric": "contour ray-samples/sec and cells segmented/sec at 1/2/4/8 B200; HBM/L2 GB/s",
               "value": samples * args.steps / (total_ms / 1e3), "unit": "ray-samples/s",
               "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
               "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "strong",
               "vs_baseline": None, "dtype": "f32", "data": "synthetic",
               "config": workload_config(cfg, world, p.cull_every),
               "cells": n_total, "detections": r["n_dets"], "halo_planes": plan.halo, "backend": backend,
               "cells_per_s": n_total * args.steps / (total_ms / 1e3), "gpu_launches": int(launches),
               "phase_ms": {"evolve_max_over_ranks": evolve_ms_max},
               "clocks": clocks,
               "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s",
                            "frac": round(achieved / hbm, 4), "traffic": None, "peak_source": hbm_src,
                            "l2": {"peak": L2_PEAK_GBPS, "frac": round(achieved / L2_PEAK_GBPS, 4)},
                            "algorithmic_bytes_per_sample": GATHER_BYTES[cfg.dim],
                            "kernel": "evolve_brick_kernel (slab)", "per": "GPU, mean over ranks"},
               "cpu_baseline": cpu,
               "e2e": {"value": samples * args.steps / e2e_s, "unit": "ray-samples/s",
                       "h2d_bytes_per_step": int(nown * 2 * world),
                       "d2h_bytes_per_step": int(cfg.n[0] * cfg.n[1] * cfg.n[2] * 4 + r["n_dets"] * CELL_BYTES * world)}}
    tdist.barrier()
    tdist.destroy_process_group()
    return out
