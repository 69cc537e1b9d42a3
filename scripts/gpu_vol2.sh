#!/bin/bash
TAG=${1:-v}; O=gpurun_out; mkdir -p $O
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:"zcol|sep8|maxima|gradmag|label_kernel|bits_|resample|lattice" \
  --log-file $O/${TAG}_vol_c4.csv python scripts/profile_step.py --config C4 --steps 1 --warmup 0 --iters 2 > $O/${TAG}_vol_c4.log 2>&1
timeout 600 python bench.py --config C3 --steps 3 --no-cpu-baseline --physical > $O/${TAG}_bench_c3_physical.json 2> $O/${TAG}_bench_c3_physical.err
timeout 600 python bench.py --config C3 --steps 3 --no-cpu-baseline --physical --estimator ray > $O/${TAG}_bench_c3_physical_ray.json 2> $O/${TAG}_bench_c3_physical_ray.err
