#!/bin/bash
TAG=${1:-f}; O=gpurun_out; mkdir -p $O
for e in ray cv; do for c in C3 C4; do
  timeout 600 python bench.py --config $c --steps 3 --no-cpu-baseline --no-e2e --estimator $e > $O/${TAG}_bench_${c}_est_$e.json 2> $O/${TAG}_bench_${c}_est_$e.err
done; done
timeout 600 python bench.py --config C4 --steps 3 --no-cpu-baseline --no-e2e --cull-every 50 > $O/${TAG}_bench_C4_cull50.json 2> $O/${TAG}_bench_C4_cull50.err
timeout 600 python bench.py --config C3 --steps 3 --no-cpu-baseline --no-e2e --cull-every 100 > $O/${TAG}_bench_C3_cull100.json 2> $O/${TAG}_bench_C3_cull100.err
timeout 600 python bench.py --config C3 --steps 3 --no-cpu-baseline --physical > $O/${TAG}_bench_C3_physical.json 2> $O/${TAG}_bench_C3_physical.err
timeout 600 python bench.py --config C2 --steps 3 --no-cpu-baseline > $O/${TAG}_bench_C2.json 2> $O/${TAG}_bench_C2.err
timeout 600 python scripts/mc_vs_grid.py --config C3 > $O/${TAG}_mc_vs_grid_c3.json 2> $O/${TAG}_mc_vs_grid_c3.err
SNK_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 3 > $O/${TAG}_bench_c4_n2_gloo.json 2> $O/${TAG}_bench_c4_n2_gloo.err
