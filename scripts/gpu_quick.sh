#!/bin/bash
# quick GPU iteration: tests + short benches.  Usage: scripts/gpu_quick.sh TAG [pytest -k expr]
TAG=${1:-q}; K=${2:-}
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/${TAG}_build.log 2>&1
if [ -n "$K" ]; then timeout 1200 python -m pytest tests -m gpu -q --timeout 900 -rf -k "$K" > $O/${TAG}_pytest_gpu.log 2>&1;
else timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -rf > $O/${TAG}_pytest_gpu.log 2>&1; fi
echo "pytest exit $?" >> $O/${TAG}_pytest_gpu.log
for cfg in C3 C4; do
 for v in ${VARIANTS:-0_4}; do set -- ${v/_/ }
  timeout 600 python bench.py --config $cfg --steps 3 --no-cpu-baseline --no-e2e --kernel-variant $1 --cta-warps $2 > $O/${TAG}_bench_${cfg}_v$1w$2.json 2> $O/${TAG}_bench_${cfg}_v$1w$2.err
 done
done
echo done
