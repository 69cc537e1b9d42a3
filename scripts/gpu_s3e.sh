#!/bin/bash
# row-tiled label kernel: label/cull/end-to-end tests (incl. the C4 scale checks), C4 + C3 benches, both label kernels timed
cd "$GRAFT_REPO_ROOT"; O=gpurun_out; mkdir -p $O; TAG=${TAG:-s3e}
timeout 1500 python -m pytest tests -m gpu -x -q -k "label or cull or end_to_end or host_call or run_batch or anisotropic or edge or scale" > $O/${TAG}_tests.txt 2>&1; tail -2 $O/${TAG}_tests.txt
for v in row column; do
  if [ $v = column ]; then export SNK_LABEL_COLUMN=1; fi
  for c in C4 C3; do
    timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 5 > $O/${TAG}_${v}_$c.json 2> $O/${TAG}_${v}_$c.err
    python -c "import json; d=json.loads(open('$O/${TAG}_${v}_$c.json').read().splitlines()[-1]); print('$v $c', d['phase_ms'], d['detections'])"
  done
done
unset SNK_LABEL_COLUMN
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none --csv -k regex:label -c 4 --log-file $O/${TAG}_label_ncu.csv python scripts/profile_step.py --config C4 --steps 1 --warmup 1 > $O/${TAG}_label_ncu.log 2>&1
grep -i "label" $O/${TAG}_label_ncu.csv | head -20
