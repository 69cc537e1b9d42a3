#!/bin/bash
cd "$GRAFT_REPO_ROOT"
D=/opt/prime-rl/.venv/lib/python3.12/site-packages/flashinfer/data/cutlass/examples/python/CuTeDSL
mkdir -p gpurun_out/r2f_cute
O=gpurun_out/r2f.txt; : > $O
export CUTE_DSL_KEEP_PTX=1 CUTE_DSL_KEEP_CUBIN=1 CUTE_DSL_DUMP_DIR=$GRAFT_REPO_ROOT/gpurun_out/r2f_cute
timeout 600 python $D/blackwell/dense_gemm.py --mnkl 512,512,256,1 >> $O 2>&1; echo "rc=$?" >> $O
timeout 600 python $D/blackwell/dense_gemm.py --mnkl 512,512,256,1 --use_tma_store >> $O 2>&1; echo "rc=$?" >> $O
ls -la gpurun_out/r2f_cute >> $O
cat $O | tail -40
