#!/bin/bash
# a8 check: label tests (crafted, stage-isolated, end to end, C4 stagewise) + C4 timing
cd "$GRAFT_REPO_ROOT"; O=gpurun_out; mkdir -p $O; TAG=${TAG:-r2p}
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -k "label or end_to_end or edge or anisotropic or host_call or run_batch" > $O/${TAG}_pytest.log 2>&1
echo "rc=$?" >> $O/${TAG}_pytest.log; tail -4 $O/${TAG}_pytest.log
timeout 1500 python -m pytest tests/test_gpu_parity_scale.py -q -x > $O/${TAG}_scale.log 2>&1
echo "rc=$?" >> $O/${TAG}_scale.log; tail -3 $O/${TAG}_scale.log
for c in C3 C4 C2; do
  timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/${TAG}_${c}.json 2> $O/${TAG}_${c}.err
  python -c "import json; d=json.loads(open('$O/${TAG}_${c}.json').read().splitlines()[-1]); print('$c', d['phase_ms'], d['detections'])"
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum --clock-control none -k regex:"label_kernel|maxima_tma" --csv python scripts/profile_step.py --config C4 --steps 1 --warmup 0 --iters 10 > $O/${TAG}_lab_c4.csv 2> $O/${TAG}_lab_c4.err
grep -E "label_kernel|maxima_tma" $O/${TAG}_lab_c4.csv | awk -F'","' '{print $5, $(NF-2), $(NF-1), $NF}' | head -12
