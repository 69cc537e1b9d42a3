#!/bin/bash
# --dist (NCCL world of one) on C3 / C4 with tracebacks on timeout; then the occupancy variants
cd "$GRAFT_REPO_ROOT"; O=gpurun_out; mkdir -p $O; TAG=${TAG:-s3f}
for c in C1 C3 C4; do
  timeout -s ABRT 300 python -X faulthandler bench.py --config $c --dist --no-cpu-baseline --steps 3 --warmup 3 > $O/${TAG}_dist_$c.json 2> $O/${TAG}_dist_$c.err
  echo "dist $c rc=$? $(tail -c 300 $O/${TAG}_dist_$c.json)"
  grep -v "NCCL INFO" $O/${TAG}_dist_$c.err | tail -30
done
VARIANTS="m4 m5 g6" CONFIGS="C2 C5_0:64 C5_3:64" TESTS="bit_identical or c1_parity or brick_reload or 2d or small_n" TAG=${TAG}v bash scripts/gpu_variant.sh
