#!/bin/bash
# small brick: warps per cell at N = 128 / 256 (SNK_SMALL_W)
cd "$GRAFT_REPO_ROOT"; O=gpurun_out; mkdir -p $O; TAG=${TAG:-s3n}
one() { local name=$1; local envs=$2; shift 2
  env $envs timeout 600 python bench.py "$@" --steps 3 --no-cpu-baseline --no-e2e > $O/${TAG}_$name.json 2> $O/${TAG}_$name.err
  python -c "import json; d=json.loads(open('$O/${TAG}_$name.json').read().splitlines()[-1]); print('$name', 'evolve', round(d['phase_ms']['evolve'],3), d['roofline']['frac'], 'dets', d['detections'])"
}
for c in C5_0 C5_3; do for N in 128 256; do for W in 1 2; do one ${c}_N${N}_W$W SNK_SMALL_W=$W --config $c --n-samples $N; done; done; done
