#!/bin/bash
# One GPU session: build check, GPU tests, smoke, benches.  Usage: scripts/gpu_round.sh [tag]
TAG=${1:-r}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi > $OUT/${TAG}_nvidia_smi.txt 2>&1
nproc > $OUT/${TAG}_nproc.txt; lscpu | grep 'Model name' >> $OUT/${TAG}_nproc.txt
python -c "import __graft_entry__ as g; g.build()" > $OUT/${TAG}_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -rf > $OUT/${TAG}_pytest_gpu.log 2>&1
echo "pytest exit $?" >> $OUT/${TAG}_pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > $OUT/${TAG}_smoke.log 2>&1
echo "smoke exit $?" >> $OUT/${TAG}_smoke.log
timeout 600 python bench.py --config C3 --steps 3 --no-cpu-baseline > $OUT/${TAG}_bench_c3.json 2> $OUT/${TAG}_bench_c3.err
timeout 900 python bench.py > $OUT/${TAG}_bench_c4.json 2> $OUT/${TAG}_bench_c4.err
echo done
timeout 900 python bench.py --impl reference > $OUT/${TAG}_bench_ref.json 2> $OUT/${TAG}_bench_ref.err
echo done-ref
