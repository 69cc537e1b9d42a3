#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 300 python scripts/micro/tma_after_cublas.py > gpurun_out/r2d_tma.txt 2>&1; echo "rc=$?" >> gpurun_out/r2d_tma.txt
env | sort > gpurun_out/r2d_env.txt
cat /proc/self/maps | grep -v "\.so\b" | head -3 >> gpurun_out/r2d_env.txt
cat gpurun_out/r2d_tma.txt
