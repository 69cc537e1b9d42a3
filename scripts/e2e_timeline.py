"""Per-step wall times of the end-to-end call (snk_run) with 1 and 2 steps in flight (C4)."""
import os, sys, time, threading
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_1804_06304_b200 import pipeline, snk
cfg = synth.CONFIGS["C4"]
p = pipeline.params_for(cfg)
h_raw = torch.empty((cfg.n[2], cfg.n[1], cfg.n[0]), dtype=torch.uint16, pin_memory=True)
synth.generate_into_ptr(cfg, h_raw.data_ptr())
runners = [pipeline.HostRunner(3, cfg.n, p, max_cells=600000) for _ in range(2)]
lo, hi = torch.cuda.Stream.priority_range()
streams = [torch.cuda.Stream(priority=hi), torch.cuda.Stream(priority=lo)]
log = []
t0 = time.perf_counter()
def work(i, n):
    torch.cuda.set_device(0)
    for _ in range(n):
        a = time.perf_counter()
        runners[i].run(h_raw, streams[i])
        log.append((i, a - t0, time.perf_counter() - t0))
work(0, 1)
# one in flight
log.clear(); t0 = time.perf_counter(); work(0, 3); t1 = time.perf_counter() - t0
print("k=1:", [(round(a, 3), round(b, 3)) for _, a, b in log], "per step", round(t1 / 3, 3))
log.clear(); t0 = time.perf_counter()
th = [threading.Thread(target=work, args=(i, 3)) for i in range(2)]
for t in th: t.start()
for t in th: t.join()
t2 = time.perf_counter() - t0
print("k=2:", sorted((i, round(a, 3), round(b, 3)) for i, a, b in log), "per step", round(t2 / 6, 3))
