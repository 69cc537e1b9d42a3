#!/bin/bash
# ncu --set full of the C4 volume kernels (blur, MAXIMA, label): summaries + source-level csv
cd "$GRAFT_REPO_ROOT"; O=gpurun_out; mkdir -p $O; TAG=${TAG:-r2o}
python -c "import __graft_entry__ as g; g.build()" > $O/${TAG}_build.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"label_kernel|maxima_tma|blur_tma" -c 3 \
  -o $O/${TAG}_vol python scripts/profile_step.py --config C4 --steps 1 --warmup 0 --iters 10 > $O/${TAG}_vol.log 2>&1
python scripts/ncu_summary.py $O/${TAG}_vol.ncu-rep --title "${TAG}: C4 volume kernels" --out $O/${TAG}_vol_summary.md
ncu -i $O/${TAG}_vol.ncu-rep --page raw --csv > $O/${TAG}_vol_raw.csv 2>/dev/null
for k in label_kernel maxima_tma blur_tma; do
  ncu -i $O/${TAG}_vol.ncu-rep -k regex:$k --page source --csv --print-source sass > $O/${TAG}_src_$k.csv 2>/dev/null
done
rm -f $O/${TAG}_vol.ncu-rep
ls -la $O | tail -8
