#!/bin/bash
# Benchmark tagged builds against the default: VARIANTS="p4 ..." (libsnk_<tag>.so); CONFIGS="C4 C3 C5_0:64"
# (config[:n_samples]); the schedule bit-identity tests under each build.
cd "$GRAFT_REPO_ROOT"; O=gpurun_out; mkdir -p $O; TAG=${TAG:-var}
for v in default $VARIANTS; do
  if [ "$v" = default ]; then unset SNK_LIB; else export SNK_LIB=$PWD/paper_1804_06304_b200/libsnk_$v.so; fi
  if [ "$v" != default ]; then timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "${TESTS:-bit_identical or c1_parity or brick_reload}" > $O/${TAG}_${v}_tests.txt 2>&1; echo "$v tests: $(tail -1 $O/${TAG}_${v}_tests.txt)"; fi
  for cn in ${CONFIGS:-C4 C3}; do
    c=${cn%%:*}; n=""; [ "$c" != "$cn" ] && n="--n-samples ${cn##*:}"
    timeout 600 python bench.py --config $c $n --steps ${STEPS:-5} --no-cpu-baseline --no-e2e > $O/${TAG}_${v}_${cn/:/_}.json 2> $O/${TAG}_${v}_${cn/:/_}.err
    python -c "import json; d=json.loads(open('$O/${TAG}_${v}_${cn/:/_}.json').read().splitlines()[-1]); print('$v $cn', round(d['ms_per_step'],3), 'evolve', round(d['phase_ms']['evolve'],3), d['roofline']['frac'], 'dets', d['detections'])"
  done
done
