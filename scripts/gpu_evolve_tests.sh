#!/bin/bash
# evolve-path change check: every evolve / pipeline GPU test + the scale tests + C3/C4 timing
cd "$GRAFT_REPO_ROOT"; O=gpurun_out; mkdir -p $O; TAG=${TAG:-r3a}
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -q -x -k "not blur and not gradmag and not maxima and not resample and not lattice_bitexact" > $O/${TAG}_pytest.log 2>&1
echo "rc=$?" >> $O/${TAG}_pytest.log; tail -4 $O/${TAG}_pytest.log
timeout 1500 python -m pytest tests/test_gpu_parity_scale.py -q -x > $O/${TAG}_scale.log 2>&1
echo "rc=$?" >> $O/${TAG}_scale.log; tail -3 $O/${TAG}_scale.log
for c in C3 C4; do
  timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/${TAG}_${c}.json 2> $O/${TAG}_${c}.err
  python -c "import json; d=json.loads(open('$O/${TAG}_${c}.json').read().splitlines()[-1]); print('$c', d['phase_ms'], d['detections'], d['roofline']['frac'], d['evolve_stats_per_step'])"
done
