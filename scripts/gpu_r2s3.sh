#!/bin/bash
# Session-3 check of the restored tree: GPU tests, C4 bench, ncu of the C3 evolve kernel (pipe counters)
cd "$GRAFT_REPO_ROOT"; O=gpurun_out; mkdir -p $O; TAG=${TAG:-s3a}
timeout 1500 python -m pytest tests -m gpu -x -q > $O/${TAG}_gputests.txt 2>&1; tail -3 $O/${TAG}_gputests.txt
timeout 600 python bench.py > $O/${TAG}_C4.json 2> $O/${TAG}_C4.err; tail -c 400 $O/${TAG}_C4.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:evolve_ -s 1 -c 1 -o $O/${TAG}_evolve_c3 python scripts/profile_step.py --config C3 --steps 1 --warmup 1 > $O/${TAG}_evolve_c3.log 2>&1
ncu -i $O/${TAG}_evolve_c3.ncu-rep --page raw --csv > $O/${TAG}_evolve_c3_raw.csv 2>/dev/null
ncu -i $O/${TAG}_evolve_c3.ncu-rep --page details --csv > $O/${TAG}_evolve_c3_details.csv 2>/dev/null
ncu -i $O/${TAG}_evolve_c3.ncu-rep --page source --csv --print-source sass > $O/${TAG}_evolve_c3_source.csv 2>/dev/null
rm -f $O/${TAG}_evolve_c3.ncu-rep
du -sh $O
