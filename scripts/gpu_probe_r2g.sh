#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r2g_tma.txt; : > $O
for b in tma5 tma6; do echo "== $b" >> $O; timeout 60 ./scripts/micro/$b >> $O 2>&1; echo "rc=$?" >> $O; done
cat $O
