import torch, triton, triton.language as tl
from triton.tools.tensor_descriptor import TensorDescriptor

@triton.jit
def copy3(in_desc, out_ptr, BZ: tl.constexpr, BY: tl.constexpr, BX: tl.constexpr):
    t = in_desc.load([9, 7, 5])
    offs = (tl.arange(0, BZ)[:, None, None] * BY + tl.arange(0, BY)[None, :, None]) * BX + tl.arange(0, BX)[None, None, :]
    tl.store(out_ptr + offs, t)

import sys
bz, by, bx = (int(v) for v in sys.argv[1:4])
dt = {"f32": torch.float32, "i16": torch.int16}[sys.argv[4]]
x = (torch.arange(64 ** 3, device="cuda") % 30000).to(dt).reshape(64, 64, 64)
out = torch.empty(bz * by * bx, dtype=dt, device="cuda")
desc = TensorDescriptor.from_tensor(x, [bz, by, bx])
copy3[(1,)](desc, out, bz, by, bx)
torch.cuda.synchronize()
print(sys.argv[1:], "triton 3D TMA ok:", torch.equal(out.reshape(bz, by, bx), x[9:9+bz, 7:7+by, 5:5+bx]), flush=True)
