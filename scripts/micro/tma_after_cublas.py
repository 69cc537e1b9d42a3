"""TMA probe inside a process that has already run a cuBLAS bf16 GEMM (whose
nvjet kernels use TMA): loads scripts/micro/tma2.cubin through the driver API
and launches tma_load<2> on the same (primary) context."""
import ctypes
import os
import sys

import numpy as np
import torch
from cuda.bindings import driver as cu

print({k: v for k, v in os.environ.items() if "CUDA" in k or "NV" in k or "LD_" in k})
a = torch.randn(2048, 2048, device="cuda", dtype=torch.bfloat16)
c = a @ a
torch.cuda.synchronize()
print("cuBLAS GEMM ok")


def ck(r):
    err = r[0] if isinstance(r, tuple) else r
    if err != cu.CUresult.CUDA_SUCCESS:
        raise RuntimeError(str(err))
    return r[1] if isinstance(r, tuple) and len(r) == 2 else r


here = os.path.dirname(os.path.abspath(__file__))
mod = ck(cu.cuModuleLoadData(open(os.path.join(here, "tma2.cubin"), "rb").read()))
fn = ck(cu.cuModuleGetFunction(mod, b"_Z8tma_loadILi2EEv14CUtensorMap_stPtiiii"))
n = 96
src = torch.arange(n * n, device="cuda", dtype=torch.int32).to(torch.int16).view(n, n)
out = torch.zeros(1 << 16, device="cuda", dtype=torch.int16)
tm = ck(cu.cuTensorMapEncodeTiled(cu.CUtensorMapDataType.CU_TENSOR_MAP_DATA_TYPE_UINT16, cu.cuuint32_t(2), src.data_ptr(),
                                  [cu.cuuint64_t(n), cu.cuuint64_t(n)], [cu.cuuint64_t(n * 2)],
                                  [cu.cuuint32_t(32), cu.cuuint32_t(16)], [cu.cuuint32_t(1), cu.cuuint32_t(1)],
                                  cu.CUtensorMapInterleave.CU_TENSOR_MAP_INTERLEAVE_NONE,
                                  cu.CUtensorMapSwizzle.CU_TENSOR_MAP_SWIZZLE_NONE,
                                  cu.CUtensorMapL2promotion.CU_TENSOR_MAP_L2_PROMOTION_NONE,
                                  cu.CUtensorMapFloatOOBfill.CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE))
raw = bytes((ctypes.c_char * 128).from_address(tm.getPtr()))
# kernel params: CUtensorMap (128 B, by value), uint16_t* out, int x, y, z, bytes
buf = (ctypes.c_uint8 * 160)()
ctypes.memmove(buf, raw, 128)
ctypes.c_uint64.from_buffer(buf, 128).value = out.data_ptr()
for i, v in enumerate([5, 7, 0, 1024]):
    ctypes.c_int32.from_buffer(buf, 136 + 4 * i).value = v
ptrs = [ctypes.addressof(buf), ctypes.addressof(buf) + 128] + [ctypes.addressof(buf) + 136 + 4 * i for i in range(4)]
arr = (ctypes.c_void_p * 6)(*ptrs)
ck(cu.cuFuncSetAttribute(fn, cu.CUfunction_attribute.CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, 65536))
r = cu.cuLaunchKernel(fn, 1, 1, 1, 128, 1, 1, 2048, 0, ctypes.addressof(arr), 0)
print("launch", r)
r = cu.cuCtxSynchronize()
print("sync", r)
if r[0] == cu.CUresult.CUDA_SUCCESS:
    g = out[:512].cpu().numpy().reshape(16, 32)
    e = src[7:23, 5:37].cpu().numpy()
    print("mismatches", int((g != e).sum()))
sys.exit(0 if r[0] == cu.CUresult.CUDA_SUCCESS else 1)
