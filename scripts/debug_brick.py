"""Small brick-kernel check (for compute-sanitizer): C1, warp vs brick kernel."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from paper_1804_06304_b200 import pipeline  # noqa: E402

cfg = synth.CONFIGS["C1"].with_(max_iters=int(sys.argv[1]) if len(sys.argv) > 1 else 20)
P = pipeline.Pipeline(3, cfg.n, pipeline.params_for(cfg))
P.upload(synth.generate(cfg))
P.preprocess()
P.seed()
res = []
for v, w in ((1, 0), (2, 4), (2, 8)):
    P.params = pipeline.params_for(cfg, kernel_variant=v, cta_warps=w)
    P.evolve()
    torch.cuda.synchronize()
    res.append(P.cells_np())
    print("variant", v, "W", w, "R[:4]", res[-1]["R"][:4], flush=True)
print("identical:", all(r.tobytes() == res[0].tobytes() for r in res))
