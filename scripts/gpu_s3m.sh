#!/bin/bash
# group kernel default B = 4 at N = 64: group / small-N tests, C5 N = 64 benches
cd "$GRAFT_REPO_ROOT"; O=gpurun_out; mkdir -p $O; TAG=${TAG:-s3m}
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "group or small_n or sample_counts or c1_parity" > $O/${TAG}_tests.txt 2>&1; tail -1 $O/${TAG}_tests.txt
for c in C5_0 C5_3; do
  timeout 600 python bench.py --config $c --n-samples 64 --steps 3 --no-cpu-baseline --no-e2e > $O/${TAG}_${c}_N64.json 2> $O/${TAG}_${c}_N64.err
  python -c "import json; d=json.loads(open('$O/${TAG}_${c}_N64.json').read().splitlines()[-1]); print('$c N64', d['ms_per_step'], 'evolve', round(d['phase_ms']['evolve'],3), d['roofline']['frac'], 'dets', d['detections'])"
done
