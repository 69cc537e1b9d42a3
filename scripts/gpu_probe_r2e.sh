#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r2e_tma.txt; : > $O
for cl in 1 2 4; do echo "== cluster $cl" >> $O; CL=$cl timeout 60 ./scripts/micro/tma4 >> $O 2>&1; echo "rc=$?" >> $O; done
cat $O
