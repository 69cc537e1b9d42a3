#!/bin/bash
# C5 small-N: default build vs the S = 24 small brick (SNK_LIB)
cd "$GRAFT_REPO_ROOT"; O=gpurun_out; mkdir -p $O; TAG=${TAG:-r2t}
for k in 0 3; do for N in 64 128 256 512; do for lib in - s24; do
  if [ "$lib" = "-" ]; then L=""; else L=paper_1804_06304_b200/libsnk_$lib.so; fi
  SNK_LIB=$L timeout 300 python bench.py --config C5_$k --steps 3 --no-cpu-baseline --no-e2e --n-samples $N > $O/${TAG}_C5_${k}_N${N}_$lib.json 2> $O/${TAG}_C5_${k}_N${N}_$lib.err
  python -c "import json; d=json.loads(open('$O/${TAG}_C5_${k}_N${N}_$lib.json').read().splitlines()[-1]); r=d['roofline']; print('C5_$k N=$N $lib', round(d['phase_ms']['evolve'],3), 'hbm', r['frac'], 'alu', r['alu_model']['frac'], d['evolve_stats_per_step'])"
done; done; done
