#!/bin/bash
# evolve change check: schedule bit-identity + evolve parity tests, C3/C4 evolve timing
cd "$GRAFT_REPO_ROOT"; O=gpurun_out; mkdir -p $O; TAG=${TAG:-r2m}
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -k "schedules or bit_identical or sample_counts or small_n or reload or 2d_parity or estimator_variants or range_resumes or full_size_sampled" > $O/${TAG}_pytest.log 2>&1
echo "rc=$?" >> $O/${TAG}_pytest.log; tail -5 $O/${TAG}_pytest.log
for c in C3 C4; do
  timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/${TAG}_${c}.json 2> $O/${TAG}_${c}.err
  python -c "import json; d=json.loads(open('$O/${TAG}_${c}.json').read().splitlines()[-1]); print('$c', d['phase_ms'], d['roofline']['samples_per_s_kernel']/1e9)"
done
timeout 900 python -m pytest tests/test_gpu_dist.py -q -x > $O/${TAG}_dist.log 2>&1; tail -2 $O/${TAG}_dist.log
