#!/bin/bash
# compaction rewrite: seeds tests, C4 bench, launch list; ncu source counters of label_kernel on C4
cd "$GRAFT_REPO_ROOT"; O=gpurun_out; mkdir -p $O; TAG=${TAG:-s3d}
timeout 900 python -m pytest tests -m gpu -x -q -k "seeds or maxima or end_to_end or run_batch or edge" > $O/${TAG}_tests.txt 2>&1; tail -2 $O/${TAG}_tests.txt
timeout 600 python bench.py --no-cpu-baseline --no-e2e > $O/${TAG}_C4.json 2> $O/${TAG}_C4.err
python -c "import json; d=json.loads(open('$O/${TAG}_C4.json').read().splitlines()[-1]); print('C4', d['ms_per_step'], d['phase_ms'], d['roofline']['frac'], d['detections'], d['cells'])"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${TAG}_launches_c4.csv python scripts/profile_step.py --config C4 --steps 1 --warmup 1 > $O/${TAG}_launches_c4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:label_kernel -s 1 -c 1 -o $O/${TAG}_label_c4 python scripts/profile_step.py --config C4 --steps 1 --warmup 1 > $O/${TAG}_label_c4.log 2>&1
ncu -i $O/${TAG}_label_c4.ncu-rep --page raw --csv > $O/${TAG}_label_c4_raw.csv 2>/dev/null
ncu -i $O/${TAG}_label_c4.ncu-rep --page source --csv --print-source sass > $O/${TAG}_label_c4_source.csv 2>/dev/null
rm -f $O/${TAG}_label_c4.ncu-rep
