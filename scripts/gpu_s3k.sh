#!/bin/bash
# label store stride + sanitizer pass over the last tree: label / cull tests, C4 phases, compute-sanitizer
# (memcheck, racecheck, synccheck) on C1 with the default MAXIMA chain, the group kernel and the small brick
cd "$GRAFT_REPO_ROOT"; O=gpurun_out; mkdir -p $O; TAG=${TAG:-s3k}
timeout 1500 python -m pytest tests -m gpu -x -q -k "label or cull or end_to_end or host_call or scale or anisotropic" > $O/${TAG}_tests.txt 2>&1; tail -1 $O/${TAG}_tests.txt
timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 > $O/${TAG}_C4.json 2> $O/${TAG}_C4.err
python -c "import json; d=json.loads(open('$O/${TAG}_C4.json').read().splitlines()[-1]); print('C4', d['ms_per_step'], d['phase_ms'], d['detections'])"
for tool in memcheck racecheck synccheck; do
  for spec in "C1:1024:m" "C1:64:l" "C1:256:l"; do
    cfg=${spec%%:*}; rest=${spec#*:}; n=${rest%%:*}; mx=${rest##*:}
    timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python scripts/profile_step.py --config $cfg --steps 1 --warmup 0 --iters 12 --n-samples $n $([ "$mx" = m ] && echo --maxima) > $O/${TAG}_${tool}_${cfg}_N${n}.log 2>&1
    echo "$tool $spec rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $O/${TAG}_${tool}_${cfg}_N${n}.log | tail -1)"
  done
done
