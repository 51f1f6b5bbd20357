# Does TMA work on this box at all?  (Triton host-side tensor descriptor.)
import torch, triton, triton.language as tl
from triton.tools.tensor_descriptor import TensorDescriptor

@triton.jit
def k(desc, out_ptr, BM: tl.constexpr, BN: tl.constexpr):
    x = desc.load([0, 0])
    offs = tl.arange(0, BM)[:, None] * BN + tl.arange(0, BN)[None, :]
    tl.store(out_ptr + offs, x)

a = torch.arange(64 * 256, dtype=torch.float32, device="cuda").reshape(64, 256)
out = torch.empty(16, 64, dtype=torch.float32, device="cuda")
d = TensorDescriptor.from_tensor(a, [16, 64])
k[(1,)](d, out, 16, 64)
torch.cuda.synchronize()
print("triton TMA ok:", torch.equal(out, a[:16, :64]))
import subprocess
src = k.cache[0] if hasattr(k, "cache") else None
