"""Single-GPU driver: device buffers (PyTorch allocations) + the a1..a8 chain
of C-ABI calls.  PyTorch is used only for memory and streams; every step runs
in libsnk's kernels."""
from __future__ import annotations

import contextlib
import time
from dataclasses import dataclass

import numpy as np
import torch

from . import snk


def params_for(cfg, **over) -> snk.snk_params:
    """snk_params for a synth.Config-like object (r0, n_samples, max_iters, seed_mode,
    seed_window / window, seed_threshold, philox_seed, dim)."""
    mode = {"lattice": snk.SEED_LATTICE, "maxima": snk.SEED_MAXIMA}[getattr(cfg, "seed_mode", "maxima")]
    kw = dict(n_samples=cfg.n_samples, max_iters=cfg.max_iters, seed_mode=mode,
              seed_window=getattr(cfg, "window", 4), seed_threshold=cfg.seed_threshold,
              seed=cfg.philox_seed)
    kw.update(over)
    return snk.make_params(cfg.r0, **kw)


def as_cells(t: torch.Tensor, n: int) -> np.ndarray:
    """Device byte buffer of snk_cell records -> numpy record array (copies n records)."""
    return t[: n * snk.CELL_BYTES].cpu().numpy().view(snk.CELL_DTYPE).copy()


@dataclass
class StepResult:
    n_seeds: int
    first_id: int
    n_dets: int
    phase_ms: dict | None = None


class Pipeline:
    """Buffers and the call chain for one (isotropic or resampled) volume."""

    def __init__(self, dim: int, n_raw, params: snk.snk_params, spacing=(1.0, 1.0, 1.0),
                 max_cells: int | None = None, labels: bool = True, gradmag: bool | None = None,
                 device: str | torch.device = "cuda", physical: bool = False):
        """physical=True: an anisotropic volume is NOT resampled (a1); every stage
        works on the raw grid in physical coordinates (G28, snk_grid.scale)."""
        self.dim = dim
        self.n_raw = tuple(int(a) for a in n_raw)
        self.spacing = tuple(float(s) for s in spacing)
        self.params = params
        self.device = torch.device(device)
        smin = min(self.spacing[:dim])
        self.scale = tuple(s / smin if a < dim else 1.0 for a, s in enumerate(self.spacing))
        if physical:
            self.n_iso = self.n_raw
        else:
            self.n_iso = snk.snk_resample_dims(dim, self.n_raw, self.spacing)
            self.scale = (1.0, 1.0, 1.0)
        self.resample = tuple(self.n_iso) != self.n_raw
        self.grid = snk.make_grid(dim, self.n_iso, scale=self.scale)
        nvox = self.n_iso[0] * self.n_iso[1] * self.n_iso[2]
        if max_cells is None:
            # generous bound on seeds: one per (2w+1)^d box for MAXIMA, the lattice count otherwise
            max_cells = max(1024, nvox // max(1, (2 * max(params.seed_window, 1) + 1) ** dim) + 1024)
        self.max_cells = int(max_cells)
        self.gradmag = (params.image_term == snk.IMAGE_GRADMAG) if gradmag is None else gradmag
        dev = self.device
        shape_raw = (self.n_raw[2], self.n_raw[1], self.n_raw[0])
        shape_iso = (self.n_iso[2], self.n_iso[1], self.n_iso[0])
        self.raw = torch.empty(shape_raw, dtype=torch.uint16, device=dev)
        self.iso = torch.empty(shape_iso, dtype=torch.uint16, device=dev) if self.resample else self.raw
        self.smooth = torch.empty(shape_iso, dtype=torch.uint16, device=dev)
        self.grad = torch.empty(shape_iso, dtype=torch.uint16, device=dev) if self.gradmag else None
        self.seeds = torch.empty((self.max_cells, 3), dtype=torch.float32, device=dev)
        self.cells = torch.empty(self.max_cells * snk.CELL_BYTES, dtype=torch.uint8, device=dev)
        self.dets = torch.empty(self.max_cells * snk.CELL_BYTES, dtype=torch.uint8, device=dev)
        self.labels = torch.empty(shape_iso, dtype=torch.int32, device=dev) if labels else None
        ws = snk.snk_workspace_bytes(self.grid, params, self.max_cells)
        if self.resample:
            ws = max(ws, 2 * nvox * 2 + 4096)
        if physical:
            ws = max(ws, 2 * nvox * 2 + 4096)   # per-axis blur ping-pong
        self.ws = torch.empty(ws, dtype=torch.uint8, device=dev)
        self.n_seeds = 0
        self.n_live = 0       # records in self.cells after evolve (< n_seeds with periodic culling)
        self.cell_iters = 0   # cell-iterations evolved (each N samples)
        self.first_id = 0
        self.n_dets = 0

    # ------------------------------------------------------------------ steps
    def upload(self, raw) -> None:
        src = torch.from_numpy(np.ascontiguousarray(raw)) if isinstance(raw, np.ndarray) else raw
        self.raw.copy_(src.reshape(self.raw.shape), non_blocking=True)

    def image(self) -> torch.Tensor:
        return self.grad if self.params.image_term == snk.IMAGE_GRADMAG else self.smooth

    def preprocess(self, stream=None):
        if self.resample:
            snk.snk_resample(self.dim, self.n_raw, self.spacing, 0, self.n_raw[2], self.raw, 0,
                             self.n_iso[2], self.iso, self.ws, stream)
        snk.snk_preprocess(self.grid, self.params, self.iso, self.smooth, self.grad, self.ws, stream)

    def seed(self, stream=None) -> int:
        self.n_seeds, self.first_id = snk.snk_seeds(self.grid, self.params, self.smooth, self.seeds,
                                                    self.max_cells, self.ws, stream)
        return self.n_seeds

    def evolve(self, stream=None, n: int | None = None, ids=None, id_base: int | None = None):
        """a5 + a6; with params.cull_every > 0 the periodic-culling segments (G25)."""
        n = self.n_seeds if n is None else n
        base = self.first_id if id_base is None else id_base
        if self.params.cull_every > 0:
            return self.evolve_periodic(stream, n, ids, base)
        snk.snk_evolve(self.grid, self.params, self.image(), self.seeds, ids, base, n, self.cells, None,
                       stream)
        self.n_live = n
        self.cell_iters = n * (self.params.max_iters + 1)

    def evolve_periodic(self, stream=None, n=None, ids=None, id_base=0):
        """Evolution in segments with the a7 cull after each but the last (P:326,
        G25); afterwards self.cells holds the self.n_live surviving records."""
        snk.snk_cells_init(self.params, self.seeds, ids, id_base, n, self.cells, stream)
        live, cur, nxt = n, self.cells, self.dets
        segs = snk.checkpoints(self.params.max_iters, self.params.cull_every)
        self.cell_iters = 0
        for i, (a, b) in enumerate(segs):
            snk.snk_evolve_range(self.grid, self.params, self.image(), cur, live, a, b, None, stream)
            self.cell_iters += live * (b - a + 1)
            if i + 1 < len(segs):
                live = snk.snk_cull(self.grid, self.params, cur, live, nxt, self.max_cells, self.ws, stream)
                cur, nxt = nxt, cur
        if cur is not self.cells and live:
            # on the stream the last segment ran on (the copy must follow it)
            with torch.cuda.stream(stream) if stream is not None else contextlib.nullcontext():
                self.cells[: live * snk.CELL_BYTES].copy_(cur[: live * snk.CELL_BYTES])
        self.n_live = live

    def cull(self, stream=None) -> int:
        self.n_dets = snk.snk_cull(self.grid, self.params, self.cells, self.n_live, self.dets,
                                   self.max_cells, self.ws, stream)
        return self.n_dets

    def label(self, stream=None):
        if self.labels is not None:
            snk.snk_label(self.grid, self.params, self.dets, self.n_dets, self.labels, self.ws, stream)

    def step(self, stream=None, timing: bool = False) -> StepResult:
        """One pass of the whole hot path (a1..a8) on the resident raw volume."""
        ev = []

        def mark():
            if timing:
                e = torch.cuda.Event(enable_timing=True)
                e.record(stream if stream is not None else torch.cuda.current_stream())
                ev.append(e)

        mark()
        self.preprocess(stream)
        mark()
        self.seed(stream)
        mark()
        self.n_live = 0
        if self.n_seeds:
            self.evolve(stream)
        mark()
        self.cull(stream)
        mark()
        self.label(stream)
        mark()
        ms = None
        if timing:
            torch.cuda.synchronize()
            names = ["preprocess", "seeds", "evolve", "cull", "label"]
            ms = {k: ev[i].elapsed_time(ev[i + 1]) for i, k in enumerate(names)}
        return StepResult(self.n_seeds, self.first_id, self.n_dets, ms)

    # ------------------------------------------------------------------ results
    def cells_np(self) -> np.ndarray:
        return as_cells(self.cells, self.n_live)

    def dets_np(self) -> np.ndarray:
        return as_cells(self.dets, self.n_dets)

    def seeds_np(self) -> np.ndarray:
        return self.seeds[: self.n_seeds].cpu().numpy().copy()


class HostRunner:
    """The end-to-end call (snk_run): host raw volume in, host detections and
    labels out, host<->device copies inside the call."""

    def __init__(self, dim, n_raw, params, spacing=(1.0, 1.0, 1.0), max_cells=None, labels=True,
                 device="cuda"):
        self.dim, self.n_raw, self.spacing, self.params = dim, tuple(n_raw), tuple(spacing), params
        n_iso = snk.snk_resample_dims(dim, self.n_raw, self.spacing)
        nvox = n_iso[0] * n_iso[1] * n_iso[2]
        if max_cells is None:
            max_cells = max(1024, nvox // max(1, (2 * max(params.seed_window, 1) + 1) ** dim) + 1024)
        self.max_cells = int(max_cells)
        ws = snk.snk_run_workspace_bytes(dim, self.n_raw, self.spacing, params, self.max_cells)
        self.ws = torch.empty(ws, dtype=torch.uint8, device=device)
        self.h_dets = torch.empty(self.max_cells * snk.CELL_BYTES, dtype=torch.uint8, pin_memory=True)
        self.h_labels = (torch.empty((n_iso[2], n_iso[1], n_iso[0]), dtype=torch.int32, pin_memory=True)
                         if labels else None)
        self.n_iso = n_iso

    def run(self, h_raw: torch.Tensor, stream=None) -> int:
        """h_raw: u16 (snk_run) or u8 (snk_run_u8: promoted x257 on the device)."""
        f = snk.snk_run_u8 if h_raw.dtype == torch.uint8 else snk.snk_run
        return f(self.dim, self.n_raw, self.spacing, self.params, h_raw, self.h_dets,
                 self.max_cells, self.h_labels, self.max_cells, self.ws, stream)

    def dets_np(self, n) -> np.ndarray:
        return self.h_dets[: n * snk.CELL_BYTES].numpy().view(snk.CELL_DTYPE).copy()


class BatchRunner:
    """The end-to-end call for a stream of volumes (snk_run_batch): host raw
    volumes in, host detections and label maps out; the next volume's upload
    and the previous results' download overlap the current volume's kernels."""

    def __init__(self, dim, n_raw, params, spacing=(1.0, 1.0, 1.0), max_cells=None, labels=True,
                 device="cuda"):
        self.dim, self.n_raw, self.spacing, self.params = dim, tuple(n_raw), tuple(spacing), params
        n_iso = snk.snk_resample_dims(dim, self.n_raw, self.spacing)
        nvox = n_iso[0] * n_iso[1] * n_iso[2]
        if max_cells is None:
            max_cells = max(1024, nvox // max(1, (2 * max(params.seed_window, 1) + 1) ** dim) + 1024)
        self.max_cells = int(max_cells)
        ws = snk.snk_run_batch_workspace_bytes(dim, self.n_raw, self.spacing, params, self.max_cells)
        self.ws = torch.empty(ws, dtype=torch.uint8, device=device)
        # two result slots are in flight at a time; volumes alternate between them
        self.h_dets = [torch.empty(self.max_cells * snk.CELL_BYTES, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
        self.h_labels = ([torch.empty((n_iso[2], n_iso[1], n_iso[0]), dtype=torch.int32, pin_memory=True)
                          for _ in range(2)] if labels else None)
        self.n_iso = n_iso

    def run(self, h_raws, stream=None) -> list:
        k = len(h_raws)
        dets = [self.h_dets[i % 2] for i in range(k)]
        labs = [self.h_labels[i % 2] for i in range(k)] if self.h_labels is not None else None
        return snk.snk_run_batch(self.dim, self.n_raw, self.spacing, self.params, list(h_raws), dets,
                                 self.max_cells, labs, self.max_cells, self.ws, stream)

    def dets_np(self, slot, n) -> np.ndarray:
        return self.h_dets[slot][: n * snk.CELL_BYTES].numpy().view(snk.CELL_DTYPE).copy()


def wall(fn, *a, **k):
    t = time.perf_counter()
    r = fn(*a, **k)
    return r, time.perf_counter() - t
