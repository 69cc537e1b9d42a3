#!/bin/bash
# source-level stall samples of the C4 evolve kernel (which regions the time goes to)
cd "$GRAFT_REPO_ROOT"; O=gpurun_out; mkdir -p $O; TAG=${TAG:-s3q}
timeout 1500 ncu --section SourceCounters --section WarpStateStats --clock-control none --import-source on -k regex:evolve_ -s 1 -c 1 -o $O/${TAG}_evolve_c4 python scripts/profile_step.py --config C4 --steps 1 --warmup 1 > $O/${TAG}_evolve_c4.log 2>&1
ncu -i $O/${TAG}_evolve_c4.ncu-rep --page source --csv --print-source sass > $O/${TAG}_evolve_c4_source.csv 2>/dev/null
rm -f $O/${TAG}_evolve_c4.ncu-rep
ls -la $O/${TAG}_evolve_c4_source.csv
