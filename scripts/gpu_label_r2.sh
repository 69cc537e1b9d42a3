#!/bin/bash
cd "$GRAFT_REPO_ROOT"
TAG=${TAG:-r2n}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_scale.py -m gpu -q -x -k "label or cull or c1 or aniso or end_to_end or c2_full or c4_full" > gpurun_out/${TAG}_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
tail -3 gpurun_out/${TAG}_pytest.log
timeout 600 python scripts/vol_timing.py C4 > gpurun_out/${TAG}_vol_c4.json 2>&1; cat gpurun_out/${TAG}_vol_c4.json
