#!/bin/bash
cd "$GRAFT_REPO_ROOT"
TAG=${TAG:-r2l}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "blur or seeds or resample or edge or small_n or c1" > gpurun_out/${TAG}_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
tail -3 gpurun_out/${TAG}_pytest.log
timeout 600 python scripts/vol_timing.py C4 > gpurun_out/${TAG}_vol_c4.json 2>&1; cat gpurun_out/${TAG}_vol_c4.json
timeout 300 python scripts/vol_timing.py C2 > gpurun_out/${TAG}_vol_c2.json 2>&1; cat gpurun_out/${TAG}_vol_c2.json
${EXTRA_CMD}
