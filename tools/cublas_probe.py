"""cuBLAS (torch.matmul) on the LLaMA-7B GEMM shapes, for side-by-side ncu comparison."""
import sys
import torch
which = sys.argv[1] if len(sys.argv) > 1 else "gemm1"
g = torch.Generator(device="cuda").manual_seed(0)
if which == "gemm1":
    A = torch.randn(8192, 4096, device="cuda", generator=g).bfloat16()
    B = torch.randn(22016, 4096, device="cuda", generator=g).bfloat16()
else:
    A = torch.randn(8192, 11008, device="cuda", generator=g).bfloat16()
    B = torch.randn(4096, 11008, device="cuda", generator=g).bfloat16()
for _ in range(6):
    C = A @ B.T
torch.cuda.synchronize()
print("ok", C.shape)
