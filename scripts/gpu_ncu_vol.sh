#!/bin/bash
# ncu --set full of the volume kernels on C4 (one launch each)
cd "$GRAFT_REPO_ROOT"
TAG=${TAG:-r2m}
KREGEX=${KREGEX:-blur_tma}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${KREGEX}" -s ${SKIP:-2} -c ${COUNT:-1} \
  -o gpurun_out/${TAG}_vol python scripts/vol_timing.py ${CFG:-C4} > gpurun_out/${TAG}_ncu.log 2>&1
python scripts/ncu_summary.py gpurun_out/${TAG}_vol.ncu-rep --title "${TAG}: ${KREGEX} on ${CFG:-C4}" --out gpurun_out/${TAG}_vol_summary.md
ncu -i gpurun_out/${TAG}_vol.ncu-rep --page raw --csv > gpurun_out/${TAG}_vol_raw.csv 2>/dev/null
ncu -i gpurun_out/${TAG}_vol.ncu-rep --page source --csv > gpurun_out/${TAG}_vol_source.csv 2>/dev/null
rm -f gpurun_out/${TAG}_vol.ncu-rep
cat gpurun_out/${TAG}_vol_summary.md | head -60
