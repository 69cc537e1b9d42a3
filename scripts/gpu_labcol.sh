#!/bin/bash
# column label kernel: every label test + the scale tests + C4 timing vs the tile kernel (libsnk_oldlab)
cd "$GRAFT_REPO_ROOT"; O=gpurun_out; mkdir -p $O; TAG=${TAG:-r3i}
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -q -x -k "label or end_to_end or anisotropic or edge or host_call or run_batch or slab or periodic or u8" > $O/${TAG}_pytest.log 2>&1
echo "rc=$?" >> $O/${TAG}_pytest.log; tail -3 $O/${TAG}_pytest.log
timeout 1500 python -m pytest tests/test_gpu_parity_scale.py -q -x > $O/${TAG}_scale.log 2>&1
echo "rc=$?" >> $O/${TAG}_scale.log; tail -2 $O/${TAG}_scale.log
SPECS="- oldlab" TAG=$TAG bash scripts/gpu_voltime.sh
