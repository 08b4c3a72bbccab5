"""One tl_mlp_forward layer (W = 1) per call, repeated, for ncu captures of the bench's kernels:
python tools/mlp_probe.py llama70b|llama7b|mixtral [calls]"""
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2503_20313_b200 as tl  # noqa: E402

SHAPES = {"llama70b": (8192, 8192, 28672), "llama7b": (8192, 4096, 11008), "mixtral": (16384, 4096, 14336)}
M, H, I = SHAPES[sys.argv[1] if len(sys.argv) > 1 else "llama70b"]
calls = int(sys.argv[2]) if len(sys.argv) > 2 else 3
c = tl.Comm.single(0, max_M=M, max_H=H)
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.randn(M, H, device="cuda", generator=g).bfloat16()
w1 = (torch.randn(2 * I, H, device="cuda", generator=g) * H ** -0.5).bfloat16()
w2 = (torch.randn(H, I, device="cuda", generator=g) * I ** -0.5).bfloat16()
out = torch.empty(M, H, device="cuda", dtype=torch.bfloat16)
for _ in range(calls):
    c.mlp_forward(x, w1, w2, out, act=tl.ACT_SILU_MUL)
torch.cuda.synchronize()
st, diag = c.check()
print("status", st, "mlp_launches", c.get_option("mlp_launches"))
