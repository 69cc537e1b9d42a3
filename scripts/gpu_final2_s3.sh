#!/bin/bash
# Final check of the last tree (kBig update, overlapped slab e2e): all GPU tests + smoke, the lines it changes
cd "$GRAFT_REPO_ROOT"; O=gpurun_out; mkdir -p $O; TAG=${TAG:-fin2}
timeout 1500 python -m pytest tests -m gpu -q > $O/${TAG}_gputests.txt 2>&1; tail -1 $O/${TAG}_gputests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${TAG}_smoke.txt 2>&1; tail -1 $O/${TAG}_smoke.txt
run() { # name, args...
  local name=$1; shift
  timeout 900 python bench.py "$@" > $O/${TAG}_$name.json 2> $O/${TAG}_$name.err
  python -c "import json; d=json.loads(open('$O/${TAG}_$name.json').read().splitlines()[-1]); r=d['roofline']; print('$name', round(d['ms_per_step'],2), 'ms', '%.1f G' % (d['value']/1e9), 'phases', {k: round(v,2) for k,v in d.get('phase_ms',{}).items()}, 'hbm', r.get('frac'), 'dets', d.get('detections'), 'e2e', (d.get('e2e') or {}).get('value'))" 2>&1 | tail -1
}
run C4
run C3 --config C3
run C2 --config C2
run C3_cull100 --config C3 --cull-every 100 --no-e2e --no-cpu-baseline
run C4_cull50 --config C4 --cull-every 50 --no-e2e --no-cpu-baseline --steps 5
run C5_0_N1024 --config C5_0 --n-samples 1024 --steps 3 --no-e2e --no-cpu-baseline
run C5_3_N1024 --config C5_3 --n-samples 1024 --steps 3 --no-e2e --no-cpu-baseline
run C4_dist1 --config C4 --dist --no-cpu-baseline
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${TAG}_launches_c4.csv python scripts/profile_step.py --config C4 --steps 1 --warmup 1 > $O/${TAG}_launches_c4.log 2>&1
