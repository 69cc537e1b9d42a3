"""Bit-identity of the brick kernel (default launch) vs the warp kernel, field by field."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from paper_1804_06304_b200 import pipeline, snk
for r0, N in ((10.0, 1024), (9.0, 512), (9.0, 256), (9.0, 128)):
    cfg = synth.CONFIGS["C1"].with_(r0=r0, n_samples=N, max_iters=120)
    p = pipeline.params_for(cfg, seed_mode=snk.SEED_LATTICE)
    P = pipeline.Pipeline(3, cfg.n, p)
    P.upload(synth.generate(cfg)); P.preprocess(); P.seed()
    P.evolve(); torch.cuda.synchronize(); a = P.cells_np()
    P.params = pipeline.params_for(cfg, seed_mode=snk.SEED_LATTICE, kernel_variant=1, cta_warps=4 if N >= 1024 else 1)
    P.evolve(); torch.cuda.synchronize(); b = P.cells_np()
    out = {f: int(np.sum(np.any((a[f] != b[f]).reshape(len(a), -1), axis=1))) for f in ("c", "R", "energy", "flags")}
    print(os.environ.get("SNK_LIB", "default"), r0, N, out, float(np.max(np.abs(a["energy"] - b["energy"]))))
