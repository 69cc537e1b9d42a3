#!/bin/bash
# C5 (BASELINE.json configs[4]): MC sample-count sweep x cell-density sweep on the
# 512x512x128 anisotropic volume, plus the 2D config C2.  Usage: scripts/c5_sweep.sh TAG
TAG=${1:-c5}; O=gpurun_out; mkdir -p $O
for k in 0 1 2 3; do for N in 64 128 256 512 1024 2048 4096; do
  timeout 300 python bench.py --config C5_$k --steps 3 --no-cpu-baseline --no-e2e --n-samples $N > $O/${TAG}_C5_${k}_N${N}.json 2> $O/${TAG}_C5_${k}_N${N}.err
done; done
timeout 600 python bench.py --config C2 --steps 3 > $O/${TAG}_C2.json 2> $O/${TAG}_C2.err
