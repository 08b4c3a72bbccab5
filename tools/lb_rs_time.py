import sys, torch
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2503_20313_b200 as tl
W, M, N, K = 8, 8192, 4096, 1376
c = tl.Comm.loopback(W, 0, max_M=M, max_H=N)
As = [torch.randn(M, K, device="cuda").bfloat16() for _ in range(W)]
Bs = [torch.randn(N, K, device="cuda").bfloat16() for _ in range(W)]
Cs = [torch.empty(M // W, N, device="cuda", dtype=torch.bfloat16) for _ in range(W)]
for _ in range(3): c.gemm_rs_lb(As, Bs, Cs)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): c.gemm_rs_lb(As, Bs, Cs)
e1.record(); torch.cuda.synchronize()
print("loopback rs W=8 ms", e0.elapsed_time(e1) / 10, c.check()[0])
