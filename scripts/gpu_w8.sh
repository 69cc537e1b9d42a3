#!/bin/bash
TAG=${1:-w}; O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -rf -k "c1_parity or sample_counts or reload" > $O/${TAG}_pytest_gpu.log 2>&1
echo "pytest exit $?" >> $O/${TAG}_pytest_gpu.log
bash scripts/variants.sh ${TAG}v C3 "-:4 -:8 w8b3:8"
bash scripts/variants.sh ${TAG}v C4 "-:4 w8b3:8"
echo done
