#!/bin/bash
TAG=${1:-pp}; O=gpurun_out; mkdir -p $O
SNK_LIB=paper_1804_06304_b200/libsnk_pipe3.so timeout 900 python -m pytest tests -m gpu -q --timeout 600 -rf -k "c1_parity or periodic or estimator or evolve_range" > $O/${TAG}_pytest_gpu.log 2>&1
echo "pytest exit $?" >> $O/${TAG}_pytest_gpu.log
bash scripts/variants.sh ${TAG}v C3 "-:4 pipe3:4"
bash scripts/variants.sh ${TAG}v C4 "-:4 pipe3:4"
