#!/bin/bash
TAG=${1:-e}; O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -rf -k "estimator" > $O/${TAG}_pytest_gpu.log 2>&1
echo "pytest exit $?" >> $O/${TAG}_pytest_gpu.log
for e in ray cv; do for c in C3 C4; do
timeout 600 python bench.py --config $c --steps 3 --no-cpu-baseline --no-e2e --estimator $e > $O/${TAG}_bench_${c}_$e.json 2> $O/${TAG}_bench_${c}_$e.err
done; done
