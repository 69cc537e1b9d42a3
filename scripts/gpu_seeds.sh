#!/bin/bash
# a4 MAXIMA check: bit-exact seed tests + C3/C4 preprocess+seeds timing (TMA pass vs the 4-pass path)
cd "$GRAFT_REPO_ROOT"; O=gpurun_out; mkdir -p $O; TAG=${TAG:-r2n}
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -k "seeds or maxima or cull_and_label or end_to_end or edge" > $O/${TAG}_pytest.log 2>&1
echo "rc=$?" >> $O/${TAG}_pytest.log; tail -4 $O/${TAG}_pytest.log
timeout 1500 python -m pytest tests/test_gpu_parity_scale.py -q -x > $O/${TAG}_scale.log 2>&1
echo "rc=$?" >> $O/${TAG}_scale.log; tail -4 $O/${TAG}_scale.log
for c in C3 C4; do
  for v in tma old; do
    if [ $v = tma ]; then export SNK_TMA_MAXIMA=1; else unset SNK_TMA_MAXIMA; fi
    timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/${TAG}_${c}_$v.json 2> $O/${TAG}_${c}_$v.err
    python -c "import json; d=json.loads(open('$O/${TAG}_${c}_$v.json').read().splitlines()[-1]); print('$c $v', d['phase_ms'], d['cells'])"
  done
done
unset SNK_TMA_MAXIMA
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"blur|maxima|bits_|label_kernel|zcol|sep8" --csv python scripts/profile_step.py --config C4 --steps 1 --warmup 1 --iters 10 > $O/${TAG}_vol_c4.csv 2> $O/${TAG}_vol_c4.err
python - <<'PY'
import csv, io, collections
rows = list(csv.reader(open("gpurun_out/r2n_vol_c4.csv".replace("r2n", __import__("os").environ.get("TAG", "r2n")))))
h = None; agg = collections.defaultdict(dict)
for r in rows:
    if r and r[0] == "ID": h = r; continue
    if h and len(r) == len(h):
        d = dict(zip(h, r)); agg[(d["ID"], d["Kernel Name"][:60])][d["Metric Name"]] = d["Metric Value"] + " " + d["Metric Unit"]
for k, v in agg.items(): print(k, v)
PY
