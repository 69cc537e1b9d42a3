#!/bin/bash
TAG=${1:-d}; O=gpurun_out; mkdir -p $O
SNK_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 3 > $O/${TAG}_bench_c4_n2_gloo.json 2> $O/${TAG}_bench_c4_n2_gloo.err
