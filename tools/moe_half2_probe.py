import sys, torch
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2503_20313_b200 as tl
import tl_inputs as TI
S, H, I, E, topk = 8192, 4096, int(sys.argv[1]) if len(sys.argv) > 1 else 2048, 8, 2
il = I
X = TI._randn((S, H), 0, 0).cuda()
Wt = TI.moe_weights(E, 2 * il, H, 1, seed=1)[0].cuda()
ids = TI.moe_routing(S, E, topk, seed=2).cuda()
c = tl.Comm.single(0, max_M=S, max_H=H, max_topk=topk)
R = tl.moe_capacity(c, S, topk, E)
Y = torch.empty(R, il, device="cuda", dtype=torch.bfloat16)
rows = torch.empty(R, device="cuda", dtype=torch.int32)
offs = torch.empty(E + 1, device="cuda", dtype=torch.int32)
W2t = TI.moe_down_weights(E, H, il, 1, seed=3)[0].cuda()
wts = TI.moe_topk_weights(S, topk, seed=4).cuda()
out = torch.empty(S, H, device="cuda", dtype=torch.bfloat16)
for _ in range(4):
    tl.moe_ag_gemm(c, X, ids, Wt, Y, rows, offs, act=tl.ACT_SILU_MUL)
    tl.moe_gemm_rs(c, Y, rows, offs, wts, W2t, out)
torch.cuda.synchronize()
print("ok")
