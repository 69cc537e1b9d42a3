#!/bin/bash
# round 2: the full-size parity tests (C4 stagewise, C4 crop / C3 / C2 end to end)
cd "$GRAFT_REPO_ROOT"
nproc > gpurun_out/r2i_nproc.txt; free -g >> gpurun_out/r2i_nproc.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2i_build.log 2>&1
timeout 2400 python -m pytest tests/test_gpu_parity_scale.py -m gpu -x -q -s --durations=0 > gpurun_out/r2i_scale.log 2>&1
echo "rc=$?" >> gpurun_out/r2i_scale.log
tail -40 gpurun_out/r2i_scale.log
