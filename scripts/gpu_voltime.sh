#!/bin/bash
# volume-pass timing (scripts/vol_timing.py) for alternative builds: SNK_LIB=<lib> ; "tma" = the one-pass TMA MAXIMA
cd "$GRAFT_REPO_ROOT"; O=gpurun_out; mkdir -p $O; TAG=${TAG:-r2r}
for spec in ${SPECS:-"-"}; do
  lib=${spec%%:*}; mode=${spec##*:}
  if [ "$lib" = "-" ]; then L=""; else L=paper_1804_06304_b200/libsnk_$lib.so; fi
  if [ "$mode" = "tma" ]; then export SNK_TMA_MAXIMA=1; else unset SNK_TMA_MAXIMA; fi
  echo "$spec $(SNK_LIB=$L timeout 600 python scripts/vol_timing.py ${CFG:-C4} 2>&1 | tail -1)"
done
