#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r2h_tma.txt; : > $O
for xy in "0 0" "8 0" "0 7" "8 7" "5 0" "2 3" "-8 0"; do set -- $xy; echo "== x=$1 y=$2" >> $O; TX=$1 TY=$2 timeout 60 ./scripts/micro/tma2 >> $O 2>&1; echo "rc=$?" >> $O; done
cat $O
