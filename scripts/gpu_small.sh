#!/bin/bash
TAG=${1:-s}; O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -rf -k "small_n or c1_parity or sample_counts" > $O/${TAG}_pytest_gpu.log 2>&1
echo "pytest exit $?" >> $O/${TAG}_pytest_gpu.log
for k in 0 3; do for N in 64 128 256 512; do
  timeout 300 python bench.py --config C5_$k --steps 3 --no-cpu-baseline --no-e2e --n-samples $N > $O/${TAG}_C5_${k}_N${N}.json 2> $O/${TAG}_C5_${k}_N${N}.err
done; done
