#!/bin/bash
TAG=${1:-v}; O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -rf -k "blur or seeds or full_size" > $O/${TAG}_pytest_gpu.log 2>&1
echo "pytest exit $?" >> $O/${TAG}_pytest_gpu.log
for lib in "" zonly; do
  L=""; [ -n "$lib" ] && L=paper_1804_06304_b200/libsnk_$lib.so
  SNK_LIB=$L timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:"zcol|sep8|maxima|gradmag|label_kernel|bits_" \
    --log-file $O/${TAG}_vol_c4_${lib:-default}.csv python scripts/profile_step.py --config C4 --steps 1 --warmup 0 --iters 2 > $O/${TAG}_vol_c4_${lib:-default}.log 2>&1
  SNK_LIB=$L timeout 600 python bench.py --config C4 --steps 3 --no-cpu-baseline --no-e2e > $O/${TAG}_bench_c4_${lib:-default}.json 2>&1
done
