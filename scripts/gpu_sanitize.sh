#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck) over every kernel family on C1-sized inputs:
# brick kernel (N = 1024), group kernel (N = 64), small brick (N = 256, r0 9), TMA MAXIMA, label, cull, u8 ingest
cd "$GRAFT_REPO_ROOT"; O=gpurun_out; mkdir -p $O; TAG=${TAG:-r2v}
for tool in memcheck racecheck synccheck; do
  for spec in "C1:1024:0" "C1:64:0" "C1:256:1"; do
    cfg=${spec%%:*}; rest=${spec#*:}; n=${rest%%:*}; tma=${rest##*:}
    SNK_TMA_MAXIMA=$tma timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python scripts/profile_step.py --config $cfg --steps 1 --warmup 0 --iters 12 --n-samples $n $([ "$tma" = 1 ] && echo --maxima) > $O/${TAG}_${tool}_${cfg}_N${n}.log 2>&1
    echo "$tool $spec rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $O/${TAG}_${tool}_${cfg}_N${n}.log | tail -1)"
  done
done
