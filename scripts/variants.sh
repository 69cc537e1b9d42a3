#!/bin/bash
# Tuning sweep over alternative builds: scripts/variants.sh TAG CFG "lib:warps ..."
# (libs built here with SNK_BUILD_TAG=<lib> SNK_NVCC_EXTRA=...; "-" = the default libsnk.so)
TAG=$1; CFG=${2:-C4}; O=gpurun_out; mkdir -p $O
for spec in $3; do
  lib=${spec%%:*}; w=${spec##*:}
  if [ "$lib" = "-" ]; then L=""; else L=paper_1804_06304_b200/libsnk_$lib.so; fi
  SNK_LIB=$L timeout 600 python bench.py --config $CFG --steps 3 --no-cpu-baseline --no-e2e --cta-warps $w \
    > $O/${TAG}_${CFG}_${lib}_w$w.json 2> $O/${TAG}_${CFG}_${lib}_w$w.err
done
echo done
