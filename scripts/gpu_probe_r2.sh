#!/bin/bash
# round 2: TMA probe (fresh) + L2/HBM bandwidth microbenchmark
cd "$GRAFT_REPO_ROOT"
nvidia-smi --query-gpu=name,driver_version,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2a_smi.txt 2>&1
timeout 60 ./scripts/micro/tma2 > gpurun_out/r2a_tma2.txt 2>&1; echo "rc=$?" >> gpurun_out/r2a_tma2.txt
timeout 120 ./scripts/micro/l2bw > gpurun_out/r2a_l2bw.txt 2>&1; echo "rc=$?" >> gpurun_out/r2a_l2bw.txt
cat gpurun_out/r2a_tma2.txt gpurun_out/r2a_l2bw.txt
