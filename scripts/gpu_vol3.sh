#!/bin/bash
TAG=${1:-v}; O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -rf -k "seeds or label or full_size or end_to_end or anisotropic or cull" > $O/${TAG}_pytest_gpu.log 2>&1
echo "pytest exit $?" >> $O/${TAG}_pytest_gpu.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:"maxima|label_kernel|bits_" \
  --log-file $O/${TAG}_vol_c4.csv python scripts/profile_step.py --config C4 --steps 1 --warmup 0 --iters 2 > $O/${TAG}_vol_c4.log 2>&1
timeout 600 python bench.py --config C4 --steps 3 --no-cpu-baseline --no-e2e > $O/${TAG}_bench_c4.json 2> $O/${TAG}_bench_c4.err
