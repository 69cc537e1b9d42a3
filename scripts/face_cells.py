"""Evolve-kernel time of C4's face cells (balls crossing a volume face) against
interior cells of the same count (which cells cost what).

    python scripts/face_cells.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1804_06304_b200 import pipeline, snk  # noqa: E402

cfg = synth.CONFIGS["C4"]
p = pipeline.params_for(cfg, image_term=snk.IMAGE_INTENSITY)
P = pipeline.Pipeline(cfg.dim, cfg.n, p, spacing=cfg.spacing, gradmag=False)
P.upload(synth.generate(cfg))
P.preprocess()
P.seed()
torch.cuda.synchronize()
s = P.seeds_np()
n = np.array(cfg.n, dtype=np.float64)
m = 16.0   # a ball of radius ~15 around a seed within 16 of a face crosses it at some point
face = np.any((s < m) | (s > n - 1 - m), axis=1)
print(f"{len(s)} cells, {face.sum()} within {m} voxels of a face ({face.mean():.1%})")
ids_all = np.arange(len(s), dtype=np.int64)
k = int(face.sum())
groups = {"face": ids_all[face], "interior": ids_all[~face][np.linspace(0, (~face).sum() - 1, k).astype(np.int64)]}
seeds_all = P.seeds[: len(s)].clone()
for name, ids in groups.items():
    sel = torch.from_numpy(ids).cuda()
    P.seeds[:k].copy_(seeds_all[sel])
    idt = sel.clone()
    times = []
    for rep in range(4):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        snk.snk_evolve(P.grid, P.params, P.image(), P.seeds, idt, 0, k, P.cells, None, None)
        b.record()
        torch.cuda.synchronize()
        times.append(a.elapsed_time(b))
    print(f"{name:9s} {k} cells: evolve {np.median(times[1:]):.2f} ms")
