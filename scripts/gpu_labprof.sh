#!/bin/bash
cd "$GRAFT_REPO_ROOT"; O=gpurun_out; mkdir -p $O; TAG=${TAG:-r2q}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"label_kernel" -c 1 \
  -o $O/${TAG}_lab python scripts/profile_step.py --config C4 --steps 1 --warmup 0 --iters 10 > $O/${TAG}_lab.log 2>&1
ncu -i $O/${TAG}_lab.ncu-rep -k regex:label_kernel --page source --csv --print-source sass > $O/${TAG}_src_label.csv 2>/dev/null
python scripts/ncu_summary.py $O/${TAG}_lab.ncu-rep --title "${TAG}: label" --out $O/${TAG}_lab_summary.md
rm -f $O/${TAG}_lab.ncu-rep
