"""Histogram of the contour radii R after T iterations on a config (brick sizing study).

    python scripts/r_hist.py --config C4 --iters 1 25 100 400
"""
import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from paper_1804_06304_b200 import pipeline  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4")
ap.add_argument("--iters", type=int, nargs="+", default=[1, 25, 100, 400])
a = ap.parse_args()
base = synth.CONFIGS[a.config]
raw = synth.generate(base)
for T in a.iters:
    cfg = base.with_(max_iters=T)
    P = pipeline.Pipeline(cfg.dim, cfg.n, pipeline.params_for(cfg), spacing=cfg.spacing)
    P.upload(raw)
    P.preprocess(); P.seed(); P.evolve()
    torch.cuda.synchronize()
    c = pipeline.as_cells(P.cells, P.n_seeds)
    R = c["R"].astype(np.float64)
    edges = np.arange(0, 28, 1.0)
    h, _ = np.histogram(R, edges)
    print(f"T={T} n={len(R)} mean={R.mean():.2f} p50={np.median(R):.2f} p90={np.percentile(R,90):.2f} "
          f"p99={np.percentile(R,99):.2f} frac(R>13.5)={np.mean(R>13.5):.3f} frac(R>=25.9)={np.mean(R>=25.9):.3f}")
    print("  hist", {int(e): int(v) for e, v in zip(edges[:-1], h) if v})
