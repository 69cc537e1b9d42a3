#!/bin/bash
# fast containment test for balls crossing a face: evolve tests, C4 / C3 / C2
cd "$GRAFT_REPO_ROOT"; O=gpurun_out; mkdir -p $O; TAG=${TAG:-s3r}
timeout 1500 python -m pytest tests -m gpu -x -q -k "evolve or bit_identical or brick or parity or estimator or anisotropic or periodic or edge or scale or small" > $O/${TAG}_tests.txt 2>&1; tail -1 $O/${TAG}_tests.txt
for c in C4 C3 C2; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 5 > $O/${TAG}_$c.json 2> $O/${TAG}_$c.err
  python -c "import json; d=json.loads(open('$O/${TAG}_$c.json').read().splitlines()[-1]); print('$c', round(d['ms_per_step'],2), 'evolve', round(d['phase_ms']['evolve'],3), d['roofline']['frac'], 'dets', d['detections'], d.get('evolve_stats_per_step'))"
done
