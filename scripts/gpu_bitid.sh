#!/bin/bash
O=gpurun_out; mkdir -p $O
for lib in paper_1804_06304_b200/libsnk_xp2.so paper_1804_06304_b200/libsnk_xp3.so; do
  SNK_LIB=$lib timeout 300 python scripts/debug_bitid.py >> $O/bitid2.txt 2>&1
done
