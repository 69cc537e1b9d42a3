#!/bin/bash
# round 2 re-entry: full GPU tests, smoke, C4 bench (state at session start)
cd "$GRAFT_REPO_ROOT"
TAG=${TAG:-r2k}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x --durations=20 > gpurun_out/${TAG}_pytest_gpu.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/${TAG}_bench_c4.json 2> gpurun_out/${TAG}_bench_c4.err
tail -3 gpurun_out/${TAG}_pytest_gpu.log; tail -2 gpurun_out/${TAG}_smoke.log; cat gpurun_out/${TAG}_bench_c4.json
