"""Run `--steps` passes of the hot path on one config (for ncu / compute-sanitizer).

    python scripts/profile_step.py --config C3 --steps 1 [--warmup 1] [--cta-warps 0]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from paper_1804_06304_b200 import pipeline, snk  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C3")
ap.add_argument("--steps", type=int, default=1)
ap.add_argument("--warmup", type=int, default=1)
ap.add_argument("--cta-warps", type=int, default=0)
ap.add_argument("--iters", type=int, default=None)
ap.add_argument("--n-samples", type=int, default=None)
ap.add_argument("--maxima", action="store_true", help="MAXIMA seeds (C1 defaults to the lattice)")
a = ap.parse_args()
cfg = synth.CONFIGS[a.config]
if a.iters:
    cfg = cfg.with_(max_iters=a.iters)
if a.n_samples:
    cfg = cfg.with_(n_samples=a.n_samples)
if a.maxima:
    cfg = cfg.with_(seed_mode="maxima")
# the step bench.py times: intensity image term, no gradient magnitude (a3 only when used)
p = pipeline.params_for(cfg, cta_warps=a.cta_warps, image_term=snk.IMAGE_INTENSITY)
P = pipeline.Pipeline(cfg.dim, cfg.n, p, spacing=cfg.spacing, gradmag=False)
P.upload(synth.generate(cfg))
for _ in range(a.warmup + a.steps):
    r = P.step(timing=True)
torch.cuda.synchronize()
print(a.config, r)
