#!/bin/bash
# Round-2 final numbers (last session): GPU tests + smoke, benches of every config / variant, C5 subset,
# reference arm, launch list and ncu of the evolve and label kernels
cd "$GRAFT_REPO_ROOT"; O=gpurun_out; mkdir -p $O; TAG=${TAG:-fin4}
timeout 1500 python -m pytest tests -m gpu -q > $O/${TAG}_gputests.txt 2>&1; tail -2 $O/${TAG}_gputests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/${TAG}_smoke.txt 2>&1; tail -1 $O/${TAG}_smoke.txt
run() { # name, args...
  local name=$1; shift
  timeout 900 python bench.py "$@" > $O/${TAG}_$name.json 2> $O/${TAG}_$name.err
  python -c "import json; d=json.loads(open('$O/${TAG}_$name.json').read().splitlines()[-1]); r=d['roofline']; print('$name', round(d['ms_per_step'],2), 'ms', '%.1f G' % (d['value']/1e9), 'phases', {k: round(v,2) for k,v in d.get('phase_ms',{}).items()}, 'hbm', r.get('frac'), 'dets', d.get('detections'), 'e2e', (d.get('e2e') or {}).get('value'))" 2>&1 | tail -1
}
run C4
timeout 900 python bench.py --impl reference > $O/${TAG}_ref_C4.json 2> $O/${TAG}_ref_C4.err; tail -c 300 $O/${TAG}_ref_C4.json; echo
run C3 --config C3
run C2 --config C2
run C3_ray --config C3 --estimator ray --no-e2e --no-cpu-baseline
run C3_cv --config C3 --estimator cv --no-e2e --no-cpu-baseline
run C3_cull100 --config C3 --cull-every 100 --no-e2e --no-cpu-baseline
run C3_physical --config C3 --physical --no-cpu-baseline
run C4_ray --config C4 --estimator ray --no-e2e --no-cpu-baseline --steps 5
run C4_cull50 --config C4 --cull-every 50 --no-e2e --no-cpu-baseline --steps 5
run C4_dist1 --config C4 --dist --no-cpu-baseline --steps 5
for k in 0 3; do for N in 64 128 256 1024 4096; do
  run C5_${k}_N$N --config C5_$k --n-samples $N --steps 3 --no-e2e --no-cpu-baseline
done; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${TAG}_launches_c4.csv python scripts/profile_step.py --config C4 --steps 1 --warmup 1 > $O/${TAG}_launches_c4.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:evolve_ -s 1 -c 1 -o $O/${TAG}_evolve_c4 python scripts/profile_step.py --config C4 --steps 1 --warmup 1 > $O/${TAG}_evolve_c4.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"label_kernel|blur_tma|maxima_pred|bits_" -s 5 -c 5 -o $O/${TAG}_volume_c4 python scripts/profile_step.py --config C4 --steps 1 --warmup 1 > $O/${TAG}_volume_c4.log 2>&1
python scripts/ncu_summary.py $O/${TAG}_evolve_c4.ncu-rep --launches $O/${TAG}_launches_c4.csv --title "${TAG}: evolve kernel (C4) + C4 launch list" --out $O/${TAG}_evolve_summary.md
python scripts/ncu_summary.py $O/${TAG}_volume_c4.ncu-rep --title "${TAG}: volume passes and label map on C4" --out $O/${TAG}_volume_summary.md
ncu -i $O/${TAG}_evolve_c4.ncu-rep --page raw --csv > $O/${TAG}_evolve_c4_raw.csv 2>/dev/null
ncu -i $O/${TAG}_volume_c4.ncu-rep --page raw --csv > $O/${TAG}_volume_c4_raw.csv 2>/dev/null
rm -f $O/${TAG}_evolve_c4.ncu-rep $O/${TAG}_volume_c4.ncu-rep
du -sh $O
