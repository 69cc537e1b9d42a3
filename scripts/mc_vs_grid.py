"""MC vs uniform-grid integration on B200 (the paper's only
quantified speed-up of MC: "~4X gain in performance on average" in 3D, P:204,
Figs. 6-7).  Times snk_evolve alone (CUDA events on the launching stream,
warm-up first) with SNK_EST_MC and SNK_EST_GRID on the same seeds of one
config and prints one JSON line.

    python scripts/mc_vs_grid.py --config C3 [--steps 3] [--iters 400]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1804_06304_b200 import pipeline, snk  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C3")
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--warmup", type=int, default=1)
ap.add_argument("--iters", type=int, default=None)
a = ap.parse_args()
cfg = synth.CONFIGS[a.config]
if a.iters:
    cfg = cfg.with_(max_iters=a.iters)
p_mc = pipeline.params_for(cfg)
p_grid = pipeline.params_for(cfg, estimator=snk.EST_GRID)
P = pipeline.Pipeline(cfg.dim, cfg.n, p_mc, spacing=cfg.spacing, labels=False)
P.upload(synth.generate(cfg))
P.preprocess()
P.seed()
torch.cuda.synchronize()
st = torch.cuda.current_stream()
out = {"workload": cfg.name, "cells": P.n_seeds,
       "iters": cfg.max_iters, "n_samples": cfg.n_samples}
res = {}
for name, p in (("mc", p_mc), ("grid", p_grid)):
    P.params = p
    for _ in range(a.warmup):
        P.evolve()
    torch.cuda.synchronize()
    ms = []
    for _ in range(a.steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        P.evolve()
        e1.record(st)
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    cells = P.cells_np()
    P.cull()
    res[name] = {"evolve_ms": float(np.median(ms)), "evolve_ms_all": ms, "detections": int(P.n_dets),
                 "R_mean": float(cells["R"].mean()), "E_mean": float(cells["energy"].mean())}
out.update(res)
out["grid_over_mc_time"] = res["grid"]["evolve_ms"] / res["mc"]["evolve_ms"]
out["mc_speedup_paper_P204"] = "~4x (GTX 1070, their N and R)"
print(json.dumps(out), flush=True)
