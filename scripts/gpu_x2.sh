#!/bin/bash
# f32x2 fast path: evolve tests + C3/C4 bench vs the scalar build.  Usage: scripts/gpu_x2.sh TAG
TAG=${1:-x}; O=gpurun_out; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 -rf -k "evolve or smoke or end_to_end or periodic or full_size" > $O/${TAG}_pytest_gpu.log 2>&1
echo "pytest exit $?" >> $O/${TAG}_pytest_gpu.log
bash scripts/variants.sh ${TAG}v C3 "-:4 scalar:4"
bash scripts/variants.sh ${TAG}v C4 "-:4 scalar:4"
echo done
