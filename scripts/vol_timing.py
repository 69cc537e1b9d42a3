"""Median / spread of the volume passes on a config (device-resident input):
preprocess (a2 [+ a3]), seeds (a4), label (a8) per call, CUDA events, 10 repeats."""
import json
import statistics
import sys

import torch

sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
import synth  # noqa: E402
from paper_1804_06304_b200 import pipeline, snk  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
cfg = synth.CONFIGS[name]
p = pipeline.params_for(cfg, image_term=snk.IMAGE_INTENSITY)
P = pipeline.Pipeline(cfg.dim, cfg.n, p, spacing=cfg.spacing, gradmag=False)
P.upload(synth.generate(cfg))
P.step()
torch.cuda.synchronize()
res = {}
for name_, fn in (("preprocess", P.preprocess), ("seeds", P.seed), ("label", P.label)):
    ts = []
    for _ in range(12):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts = ts[2:]
    res[name_] = {"median_ms": statistics.median(ts), "min_ms": min(ts), "max_ms": max(ts)}
nvox = P.n_iso[0] * P.n_iso[1] * P.n_iso[2]
res["blur_GBps_algorithmic"] = 4 * nvox / res["preprocess"]["median_ms"] / 1e6
res["label_GBps_algorithmic"] = 4 * nvox / res["label"]["median_ms"] / 1e6
res["n_seeds"], res["n_dets"] = P.n_seeds, P.n_dets
print(json.dumps(res))
