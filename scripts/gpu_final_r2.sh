#!/bin/bash
# Round-2 final numbers: benches of every config / variant, C5 subset, ncu evidence
cd "$GRAFT_REPO_ROOT"; O=gpurun_out; mkdir -p $O; TAG=${TAG:-r3f}
python -c "import __graft_entry__ as g; g.build()" > $O/${TAG}_build.log 2>&1
run() { # name, args...
  local name=$1; shift
  timeout 900 python bench.py "$@" > $O/${TAG}_$name.json 2> $O/${TAG}_$name.err
  python -c "import json; d=json.loads(open('$O/${TAG}_$name.json').read().splitlines()[-1]); r=d['roofline']; print('$name', round(d['ms_per_step'],2), 'ms', '%.1f G' % (d['value']/1e9), 'evolve', round(d['phase_ms']['evolve'],2), 'hbm', r['frac'], 'dets', d['detections'], 'e2e', (d['e2e'] or {}).get('value'))" 2>&1 | tail -1
}
run C4 
run C3 --config C3
run C2 --config C2
run C3_ray --config C3 --estimator ray --no-e2e --no-cpu-baseline
run C3_cv --config C3 --estimator cv --no-e2e --no-cpu-baseline
run C3_cull100 --config C3 --cull-every 100 --no-e2e --no-cpu-baseline
run C3_physical --config C3 --physical --no-cpu-baseline
run C4_ray --config C4 --estimator ray --no-e2e --no-cpu-baseline --steps 5
run C4_cull50 --config C4 --cull-every 50 --no-e2e --no-cpu-baseline --steps 5
timeout 900 python scripts/mc_vs_grid.py --config C3 > $O/${TAG}_mc_vs_grid_c3.json 2> $O/${TAG}_mc_vs_grid_c3.err; tail -c 600 $O/${TAG}_mc_vs_grid_c3.json
for k in 0 3; do for N in 64 128 256 512 1024 4096; do
  run C5_${k}_N$N --config C5_$k --n-samples $N --steps 3 --no-e2e --no-cpu-baseline
done; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${TAG}_launches_c4.csv python scripts/profile_step.py --config C4 --steps 1 --warmup 1 > $O/${TAG}_launches_c4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:evolve_ -s 1 -c 1 -o $O/${TAG}_evolve_c3 python scripts/profile_step.py --config C3 --steps 1 --warmup 1 > $O/${TAG}_evolve_c3.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:evolve_ -s 1 -c 1 -o $O/${TAG}_evolve_c4 python scripts/profile_step.py --config C4 --steps 1 --warmup 1 > $O/${TAG}_evolve_c4.log 2>&1
python scripts/ncu_summary.py $O/${TAG}_evolve_c3.ncu-rep $O/${TAG}_evolve_c4.ncu-rep --launches $O/${TAG}_launches_c4.csv --title "${TAG}: evolve kernel + C4 launch list" --out $O/${TAG}_evolve_summary.md
ncu -i $O/${TAG}_evolve_c3.ncu-rep --page raw --csv > $O/${TAG}_evolve_c3_raw.csv 2>/dev/null
ncu -i $O/${TAG}_evolve_c4.ncu-rep --page raw --csv > $O/${TAG}_evolve_c4_raw.csv 2>/dev/null
ncu -i $O/${TAG}_evolve_c4.ncu-rep --page source --csv --print-source sass > $O/${TAG}_evolve_c4_source.csv 2>/dev/null
rm -f $O/${TAG}_evolve_c3.ncu-rep $O/${TAG}_evolve_c4.ncu-rep
du -sh $O
