#!/bin/bash
TAG=${1:-b}; O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -rf -k "run_batch or end_to_end or host or cull or seeds or label or periodic" > $O/${TAG}_pytest_gpu.log 2>&1
echo "pytest exit $?" >> $O/${TAG}_pytest_gpu.log
timeout 900 python bench.py --no-cpu-baseline > $O/${TAG}_bench_c4_batch.json 2> $O/${TAG}_bench_c4_batch.err
timeout 900 python bench.py --no-cpu-baseline --e2e-mode threads > $O/${TAG}_bench_c4_threads.json 2> $O/${TAG}_bench_c4_threads.err
timeout 600 python bench.py --config C3 --no-cpu-baseline > $O/${TAG}_bench_c3_batch.json 2> $O/${TAG}_bench_c3_batch.err
