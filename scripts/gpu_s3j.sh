#!/bin/bash
# MAXIMA predicate on a (x groups, y, z) grid: seeds tests (incl. full-size C4), C4 bench, launch list
cd "$GRAFT_REPO_ROOT"; O=gpurun_out; mkdir -p $O; TAG=${TAG:-s3j}
timeout 1500 python -m pytest tests -m gpu -x -q -k "seeds or maxima or end_to_end or run_batch or edge or scale or u8 or 2d or dist" > $O/${TAG}_tests.txt 2>&1; tail -1 $O/${TAG}_tests.txt
timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 > $O/${TAG}_C4.json 2> $O/${TAG}_C4.err
python -c "import json; d=json.loads(open('$O/${TAG}_C4.json').read().splitlines()[-1]); print('C4', d['ms_per_step'], d['phase_ms'], d['detections'], d['cells'])"
timeout 900 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum --clock-control none --csv -k regex:maxima_pred -c 2 --log-file $O/${TAG}_pred.csv python scripts/profile_step.py --config C4 --steps 1 --warmup 1 > $O/${TAG}_pred.log 2>&1
grep -o '"gpu__time_duration.sum","[a-z]*","[0-9.,]*"\|"smsp__inst_executed.sum","[a-z]*","[0-9.,]*"' $O/${TAG}_pred.csv
