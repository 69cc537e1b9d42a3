#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r2c_tma.txt
: > $O
for b in tma2_sm100 tma2_ptx90 tma2_ptx100a tma2_ptx100; do echo "== $b" >> $O; timeout 120 ./scripts/micro/$b >> $O 2>&1; echo "rc=$?" >> $O; done
python -c "import cutlass; print('cutlass dsl', cutlass.__version__ if hasattr(cutlass,'__version__') else '?')" >> $O 2>&1
cat $O
