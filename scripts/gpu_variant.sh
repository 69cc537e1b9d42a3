#!/bin/bash
# Benchmark tagged builds against the default: VARIANTS="p4 ..." (libsnk_<tag>.so), C4 and C3 evolve,
# plus the schedule bit-identity tests under each build.
cd "$GRAFT_REPO_ROOT"; O=gpurun_out; mkdir -p $O; TAG=${TAG:-var}
for v in default $VARIANTS; do
  if [ "$v" = default ]; then unset SNK_LIB; else export SNK_LIB=$PWD/paper_1804_06304_b200/libsnk_$v.so; fi
  if [ "$v" != default ]; then timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "bit_identical or c1_parity or brick_reload" > $O/${TAG}_${v}_tests.txt 2>&1; echo "$v tests: $(tail -1 $O/${TAG}_${v}_tests.txt)"; fi
  for c in ${CONFIGS:-C4 C3}; do
    timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e > $O/${TAG}_${v}_$c.json 2> $O/${TAG}_${v}_$c.err
    python -c "import json; d=json.loads(open('$O/${TAG}_${v}_$c.json').read().splitlines()[-1]); print('$v $c', round(d['ms_per_step'],2), 'evolve', round(d['phase_ms']['evolve'],2), d['roofline']['frac'], 'dets', d['detections'])"
  done
done
