#!/bin/bash
# round 2: TMA descriptor-source variants, plain bulk copy, cuBLAS bf16 GEMM (TMA inside cuBLAS), sanitizer view
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r2b_tma.txt
: > $O
for v in 0 1 2; do echo "== tma3 $v" >> $O; timeout 60 ./scripts/micro/tma3 $v >> $O 2>&1; echo "rc=$?" >> $O; done
echo "== bulk" >> $O; timeout 60 ./scripts/micro/bulk >> $O 2>&1; echo "rc=$?" >> $O
echo "== sanitizer tma3 0" >> $O; timeout 120 compute-sanitizer --tool memcheck ./scripts/micro/tma3 0 >> $O 2>&1; echo "rc=$?" >> $O
echo "== cublas bf16" >> $O
timeout 300 python - >> $O 2>&1 <<'PY'
import torch
a = torch.randn(4096, 4096, device="cuda", dtype=torch.bfloat16)
b = torch.randn(4096, 4096, device="cuda", dtype=torch.bfloat16)
c = a @ b
torch.cuda.synchronize()
print("matmul ok", float((c.float() - a.float() @ b.float()).abs().max()))
PY
echo "rc=$?" >> $O
timeout 300 ncu --metrics gpu__time_duration.sum --csv python -c "
import torch
a = torch.randn(4096, 4096, device='cuda', dtype=torch.bfloat16); c = a @ a; torch.cuda.synchronize()" >> $O 2>&1
cat $O
