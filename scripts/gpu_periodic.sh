#!/bin/bash
# periodic culling + grid: GPU tests and benches.  Usage: scripts/gpu_periodic.sh TAG
TAG=${1:-p}; O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -rf > $O/${TAG}_pytest_gpu.log 2>&1
echo "pytest exit $?" >> $O/${TAG}_pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > $O/${TAG}_smoke.log 2>&1
for k in 0 25 50 100; do
  timeout 600 python bench.py --config C3 --steps 3 --no-cpu-baseline --no-e2e --cull-every $k > $O/${TAG}_bench_c3_k$k.json 2> $O/${TAG}_bench_c3_k$k.err
done
for k in 50; do
  timeout 900 python bench.py --config C4 --steps 3 --no-cpu-baseline --cull-every $k > $O/${TAG}_bench_c4_k$k.json 2> $O/${TAG}_bench_c4_k$k.err
done
echo done
