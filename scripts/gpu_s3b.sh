#!/bin/bash
# loader rewrite: GPU tests + C4 / C3 benches
cd "$GRAFT_REPO_ROOT"; O=gpurun_out; mkdir -p $O; TAG=${TAG:-s3b}
timeout 1500 python -m pytest tests -m gpu -x -q > $O/${TAG}_gputests.txt 2>&1; tail -3 $O/${TAG}_gputests.txt
for c in C4 C3; do
timeout 600 python bench.py --config $c --no-cpu-baseline > $O/${TAG}_$c.json 2> $O/${TAG}_$c.err
python -c "import json; d=json.loads(open('$O/${TAG}_$c.json').read().splitlines()[-1]); print('$c', d['ms_per_step'], d['phase_ms'], d['roofline']['frac'], d['evolve_stats_per_step'])"
done
