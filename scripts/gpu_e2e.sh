#!/bin/bash
TAG=${1:-e}; O=gpurun_out; mkdir -p $O
for pr in 1 0; do
  timeout 900 python bench.py --steps 6 --no-cpu-baseline --e2e-priorities $pr > $O/${TAG}_bench_c4_prio$pr.json 2> $O/${TAG}_bench_c4_prio$pr.err
done
timeout 900 python bench.py --steps 6 --no-cpu-baseline --e2e-inflight 3 > $O/${TAG}_bench_c4_prio1_k3.json 2> $O/${TAG}_bench_c4_prio1_k3.err
