#!/bin/bash
# diagnostic builds of the evolve kernel (wrong results on purpose): bounds for
# conflict-free gathers (dnc) and fewer Philox rounds (dp5); C3 and C4 evolve time
cd "$GRAFT_REPO_ROOT"; O=gpurun_out; mkdir -p $O; TAG=${TAG:-r2l}
for c in C3 C4; do for lib in - dnc dp5 dncp5; do
  if [ "$lib" = "-" ]; then L=""; else L=paper_1804_06304_b200/libsnk_$lib.so; fi
  SNK_LIB=$L timeout 600 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-e2e \
    > $O/${TAG}_${c}_${lib}.json 2> $O/${TAG}_${c}_${lib}.err
  python -c "import json,sys; d=json.loads(open('$O/${TAG}_${c}_${lib}.json').read().splitlines()[-1]); print('$c', '$lib', d['phase_ms'], d['roofline']['samples_per_s_kernel']/1e9)"
done; done
timeout 900 python -m pytest tests/test_gpu_dist.py -q -x > $O/${TAG}_dist.log 2>&1; tail -2 $O/${TAG}_dist.log
