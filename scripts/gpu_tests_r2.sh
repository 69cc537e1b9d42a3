#!/bin/bash
# round 2: full GPU test suite (+ the full-size parity tests) and smoke
cd "$GRAFT_REPO_ROOT"
TAG=${TAG:-r2j}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
timeout 3000 python -m pytest tests -m gpu -q -s --durations=15 ${PYTEST_ARGS} > gpurun_out/${TAG}_pytest_gpu.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_smoke.log
grep -E "passed|failed|error" gpurun_out/${TAG}_pytest_gpu.log | tail -5
grep -E "cells, max|differences|end to end" gpurun_out/${TAG}_pytest_gpu.log | head -30
tail -3 gpurun_out/${TAG}_smoke.log
