#!/bin/bash
# overlapped slab-driver e2e (upload issued before the step) + the kBig update specialization A/B
cd "$GRAFT_REPO_ROOT"; O=gpurun_out; mkdir -p $O; TAG=${TAG:-s3i}
timeout 1200 python -m pytest tests/test_gpu_dist.py -m gpu -x -q > $O/${TAG}_tests.txt 2>&1; tail -1 $O/${TAG}_tests.txt
timeout 600 python bench.py --config C4 --dist --no-cpu-baseline --steps 5 > $O/${TAG}_C4_dist1.json 2> $O/${TAG}_C4_dist1.err
python -c "import json; d=json.loads(open('$O/${TAG}_C4_dist1.json').read().splitlines()[-1]); print('C4 dist1', d['ms_per_step'], d['value']/1e9, d['roofline']['frac'], d['detections'], 'e2e', d['e2e']['value']/1e9)"
VARIANTS="nb" CONFIGS="C4 C3 C2" STEPS=5 TESTS="bit_identical or c1_parity or brick_reload or 2d or slab or edge" TAG=${TAG}v bash scripts/gpu_variant.sh
