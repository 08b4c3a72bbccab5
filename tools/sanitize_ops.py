"""Run one small call of every fused op (both resource bindings) so `compute-sanitizer --tool memcheck`
can check every kernel for out-of-bounds / misaligned global accesses:
    compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_ops.py
Results are compared with torch fp32 so a sanitizer-perturbed run that computes garbage also fails."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2503_20313_b200 as tl  # noqa: E402
import tl_inputs as TI  # noqa: E402

tl.lib()
cu = lambda L: [t.cuda().contiguous() for t in L]


def rel(a, b):
    a, b = a.float(), b.float()
    return ((a - b).norm() / b.norm().clamp_min(1e-30)).item()


def check(c, name):
    st, diag = c.check()
    assert st == 0, (name, diag)


def mlp(W, binding, fused=1, pull=0):
    M, H, I = 512, 256, 768
    X, G, U, W2 = TI.mlp_full(M, H, I, seed=1)
    Xs, W1s, W2s = (cu(L) for L in TI.shard_mlp(X, G, U, W2, W, TI.ACT_SILU_MUL))
    c = tl.Comm.loopback(W, 0, max_M=M, max_H=H)
    c.set_option("timeout_ms", 600000)   # the sanitizer slows the spin-waits down
    if binding:
        c.set_option("ag_binding", 1)
        c.set_option("rs_binding", 1)
        c.set_option("rs_dma_rows", 128)
    c.set_option("mlp_fused", fused)     # 2: the one-launch layer kernel, 0: two launches
    c.set_option("ag_mode", pull)        # 1: AllGather pull mode
    outs = [torch.empty(M // W, H, device="cuda", dtype=torch.bfloat16) for _ in range(W)]
    c.mlp_forward_lb(Xs, W1s, W2s, outs, act=TI.ACT_SILU_MUL)
    check(c, "mlp")
    Xf = X.cuda().float()
    h = torch.nn.functional.silu(Xf @ G.cuda().float().t()) * (Xf @ U.cuda().float().t())
    ref = h.bfloat16().float() @ W2.cuda().float().t()
    e = rel(torch.cat(outs, 0), ref)
    print(f"mlp W={W} binding={binding} fused={fused} pull={pull} launches={c.get_option('mlp_launches')}: rel {e:.2e}")
    assert e < 1e-2
    c.close()


def ag_rs(W, binding):
    M, N, K = 512, 384, 256
    As, Bs = (cu(L) for L in TI.ag_gemm_inputs(M, N, K, W, seed=2))
    c = tl.Comm.loopback(W, 0, max_M=M, max_H=max(K, N))
    c.set_option("timeout_ms", 600000)   # the sanitizer slows the spin-waits down
    c.set_option("ag_binding", binding)
    Cs = [torch.empty(M, N, device="cuda", dtype=torch.bfloat16) for _ in range(W)]
    c.ag_gemm_lb(As, Bs, Cs)
    check(c, "ag")
    Af = torch.cat(As, 0).float()
    for r in range(W):
        assert rel(Cs[r], Af @ Bs[r].float().t()) < 1e-2
    c.set_option("rs_binding", binding)
    if binding:
        c.set_option("rs_dma_rows", 128)
    Zs = [torch.randn(M, K, device="cuda").bfloat16() for _ in range(W)]
    Ws = [torch.randn(N, K, device="cuda").bfloat16() for _ in range(W)]
    Ps = [torch.empty(M // W, N, device="cuda", dtype=torch.bfloat16) for _ in range(W)]
    c.gemm_rs_lb(Zs, Ws, Ps)
    check(c, "rs")
    ref = sum(Zs[r].float() @ Ws[r].float().t() for r in range(W))
    e = rel(torch.cat(Ps, 0), ref)
    print(f"ag/rs W={W} binding={binding}: rel {e:.2e}")
    assert e < 1e-2
    c.close()


def moe(W, binding):
    M, H, I, E, topk = 512, 256, 512, 8, 2
    il = I // W
    X = TI._randn((M, H), 3, 0)
    Xs = cu(TI.shard_rows(X, W))
    W1s, W2s = cu(TI.moe_weights(E, 2 * il, H, W, seed=4)), cu(TI.moe_down_weights(E, H, il, W, seed=5))
    ids = TI.moe_routing(M, E, topk, seed=6, skew=1.0)
    wts = TI.moe_topk_weights(M, topk, seed=7)
    c = tl.Comm.loopback(W, 0, max_M=M, max_H=H, max_topk=topk)
    c.set_option("timeout_ms", 600000)   # the sanitizer slows the spin-waits down
    c.set_option("ag_binding", binding)
    c.set_option("rs_binding", binding)
    R = tl.moe_capacity(c, M, topk, E)
    Zg = [torch.empty(R, il, device="cuda", dtype=torch.bfloat16) for _ in range(W)]
    rows = [torch.empty(R, device="cuda", dtype=torch.int32) for _ in range(W)]
    offs = [torch.empty(E + 1, device="cuda", dtype=torch.int32) for _ in range(W)]
    outs = [torch.empty(M // W, H, device="cuda", dtype=torch.bfloat16) for _ in range(W)]
    idd, wtd = [ids.cuda() for _ in range(W)], [wts.cuda() for _ in range(W)]
    tl.moe_ag_gemm_lb(c, Xs, idd, W1s, Zg, rows, offs, act=TI.ACT_SILU_MUL)
    tl.moe_gemm_rs_lb(c, Zg, rows, offs, wtd, W2s, outs)
    check(c, "moe")
    assert torch.isfinite(torch.cat(outs, 0).float()).all()
    print(f"moe W={W} binding={binding}: ok")
    c.close()


def attn(W, binding, pull=0):
    S, heads = 256 * W, 2
    Qs, Ks, Vs = (cu(L) for L in TI.attention_inputs(S, heads, 128, W, seed=8))
    c = tl.Comm.loopback(W, 0, max_M=S, max_H=2 * heads * 128)
    c.set_option("timeout_ms", 600000)   # the sanitizer slows the spin-waits down
    c.set_option("ag_binding", binding)
    c.set_option("ag_mode", pull)
    outs = [torch.empty_like(q) for q in Qs]
    tl.sp_attention_lb(c, Qs, Ks, Vs, outs)
    check(c, "attn")
    K, V = torch.cat(Ks, 0).float(), torch.cat(Vs, 0).float()
    for r in range(W):
        q = Qs[r].float()
        s = torch.einsum("qhd,khd->hqk", q, K) / 128 ** 0.5
        ref = torch.einsum("hqk,khd->qhd", s.softmax(-1), V)
        assert rel(outs[r], ref) < 1e-2
    print(f"attn W={W} binding={binding}: ok")
    c.close()


if __name__ == "__main__":
    worlds = [int(w) for w in sys.argv[1].split(",")] if len(sys.argv) > 1 else [2, 4]
    for W in worlds:
        for fused, pull in ((2, 0), (0, 0), (2, 1), (0, 1)):
            mlp(W, 0, fused, pull)
        for b in (0, 1):
            mlp(W, b)
            ag_rs(W, b)
            moe(W, b)
            attn(W, b)
        attn(W, 0, pull=1)
    torch.cuda.synchronize()
    print("SANITIZE_OPS_DONE")
