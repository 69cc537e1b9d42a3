#!/bin/bash
# small N: group-kernel lanes per cell (SNK_GROUP_B = samples per lane) vs cells in flight
cd "$GRAFT_REPO_ROOT"; O=gpurun_out; mkdir -p $O; TAG=${TAG:-s3l}
one() { # name env args
  local name=$1; local envs=$2; shift 2
  env $envs timeout 600 python bench.py "$@" --steps 3 --no-cpu-baseline --no-e2e > $O/${TAG}_$name.json 2> $O/${TAG}_$name.err
  python -c "import json; d=json.loads(open('$O/${TAG}_$name.json').read().splitlines()[-1]); print('$name', 'evolve', round(d['phase_ms']['evolve'],3), d['roofline']['frac'], 'dets', d['detections'])"
}
for c in C5_0 C5_3; do
  for B in 8 4; do one ${c}_N64_B$B SNK_GROUP_B=$B --config $c --n-samples 64; done
  one ${c}_N128_default X=1 --config $c --n-samples 128
  for B in 8 4; do one ${c}_N128_grp_B$B SNK_GROUP_B=$B --config $c --n-samples 128 --kernel-variant 3; done
  one ${c}_N256_default X=1 --config $c --n-samples 256
  for B in 8 16; do one ${c}_N256_grp_B$B SNK_GROUP_B=$B --config $c --n-samples 256 --kernel-variant 3; done
done
