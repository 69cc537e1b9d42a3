#!/bin/bash
TAG=${1:-l}; O=gpurun_out; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"label_kernel|gradmag8" -c 2 -o $O/${TAG}_lg python scripts/profile_step.py --config C4 --steps 1 --warmup 0 --iters 2 > $O/${TAG}_lg.log 2>&1
ncu -i $O/${TAG}_lg.ncu-rep --page raw --csv > $O/${TAG}_lg_raw.csv 2>/dev/null
ncu -i $O/${TAG}_lg.ncu-rep --page source --csv -k regex:label_kernel > $O/${TAG}_label_source.csv 2>/dev/null
rm -f $O/${TAG}_lg.ncu-rep
