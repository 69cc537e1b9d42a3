#!/bin/bash
# grid estimator tests + MC/grid timing + one-barrier variant sweep.  Usage: scripts/gpu_grid.sh TAG
TAG=${1:-g}; O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -rf -k "grid or c1_parity or reload or slab" > $O/${TAG}_pytest_gpu.log 2>&1
echo "pytest exit $?" >> $O/${TAG}_pytest_gpu.log
timeout 600 python scripts/mc_vs_grid.py --config C3 > $O/${TAG}_mc_vs_grid_c3.json 2> $O/${TAG}_mc_vs_grid_c3.err
bash scripts/variants.sh ${TAG}v C3 "-:4 pipe2:4"
bash scripts/variants.sh ${TAG}v C4 "-:4 pipe2:4"
