#!/bin/bash
# slab driver counts over a gloo group: dist tests, C4 --dist (device + e2e)
cd "$GRAFT_REPO_ROOT"; O=gpurun_out; mkdir -p $O; TAG=${TAG:-s3o}
timeout 1200 python -m pytest tests/test_gpu_dist.py -m gpu -x -q > $O/${TAG}_tests.txt 2>&1; tail -1 $O/${TAG}_tests.txt
timeout 600 python bench.py --config C4 --dist --no-cpu-baseline > $O/${TAG}_C4_dist1.json 2> $O/${TAG}_C4_dist1.err
echo "stdout lines: $(grep -c . $O/${TAG}_C4_dist1.json)"
python -c "import json; d=json.loads(open('$O/${TAG}_C4_dist1.json').read().splitlines()[-1]); print('C4 dist1', d['ms_per_step'], d['value']/1e9, d['roofline']['frac'], d['detections'], 'e2e', d['e2e']['value']/1e9)"
