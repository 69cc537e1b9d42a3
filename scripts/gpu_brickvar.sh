#!/bin/bash
# brick geometry variants (SNK_LIB): evolve time on C3 / C4
cd "$GRAFT_REPO_ROOT"; O=gpurun_out; mkdir -p $O; TAG=${TAG:-r2z}
for c in C3 C4; do for lib in ${LIBS:-- s32 a4s32}; do
  if [ "$lib" = "-" ]; then L=""; else L=paper_1804_06304_b200/libsnk_$lib.so; fi
  SNK_LIB=$L timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/${TAG}_${c}_$lib.json 2> $O/${TAG}_${c}_$lib.err
  python -c "import json; d=json.loads(open('$O/${TAG}_${c}_$lib.json').read().splitlines()[-1]); print('$c $lib', round(d['phase_ms']['evolve'],2), d['detections'], d['evolve_stats_per_step'])"
done; done
