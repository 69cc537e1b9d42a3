#!/bin/bash
# NCCL log to stderr: dist tests; C2 bench with the 4-CTA 2D kernel; --dist C4 stdout check
cd "$GRAFT_REPO_ROOT"; O=gpurun_out; mkdir -p $O; TAG=${TAG:-s3g}
timeout 1200 python -m pytest tests/test_gpu_dist.py tests/test_gpu_parity.py -m gpu -x -q -k "dist or nccl or bench or slabs or 2d or bit_identical" > $O/${TAG}_tests.txt 2>&1; tail -2 $O/${TAG}_tests.txt
timeout 600 python bench.py --config C2 > $O/${TAG}_C2.json 2> $O/${TAG}_C2.err
python -c "import json; d=json.loads(open('$O/${TAG}_C2.json').read().splitlines()[-1]); print('C2', d['ms_per_step'], d['phase_ms'], d['roofline']['frac'], d['detections'], d['e2e']['value'])"
timeout 600 python bench.py --config C4 --dist --no-cpu-baseline --steps 5 > $O/${TAG}_C4_dist1.json 2> $O/${TAG}_C4_dist1.err
echo "stdout lines: $(grep -c . $O/${TAG}_C4_dist1.json), NCCL lines in stderr: $(grep -c 'NCCL INFO' $O/${TAG}_C4_dist1.err)"
python -c "import json; d=json.loads(open('$O/${TAG}_C4_dist1.json').read().splitlines()[-1]); print('C4 dist1', d['ms_per_step'], d['value']/1e9, d['roofline']['frac'], d['detections'], d['e2e']['value']/1e9)"
