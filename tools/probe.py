"""First-contact probe of the CUDA path on a B200 (one step per process; see tools/probe.sh)."""
import sys
import time

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2503_20313_b200 as tl  # noqa: E402


def rel(a, b):
    a, b = a.float(), b.float()
    return ((a - b).norm() / b.norm().clamp_min(1e-30)).item()


def gemm(pair, M, N, K, act=0):
    c = tl.Comm.single(0, max_M=M, max_H=K)
    c.set_option("cta_pair", pair)
    g = torch.Generator(device="cuda").manual_seed(0)
    A = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    if act:
        B = (torch.randn(2 * N, K, device="cuda", generator=g) / K ** 0.5).bfloat16()
    else:
        B = (torch.randn(N, K, device="cuda", generator=g) / K ** 0.5).bfloat16()
    C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    c.ag_gemm(A, B, C, act=act)
    torch.cuda.synchronize()
    Y = A.float() @ B.float().T
    if act == 1:
        ref = torch.nn.functional.silu(Y[:, :N]) * Y[:, N:]
    else:
        ref = Y
    e = rel(C, ref)
    # timing
    for _ in range(3):
        c.ag_gemm(A, B, C, act=act)
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    n = 10
    t0.record()
    for _ in range(n):
        c.ag_gemm(A, B, C, act=act)
    t1.record()
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / n
    fl = 2 * M * K * (2 * N if act else N)
    print(f"gemm pair={pair} M={M} N={N} K={K} act={act}: rel={e:.3e}  {ms*1e3:.1f} us  {fl/ms/1e9:.1f} TFLOPS",
          flush=True)
    c.close()
    return e


def loop_ag(W, M, N, K, act=0):
    c = tl.Comm.loopback(W, 0, max_M=M, max_H=K)
    g = torch.Generator(device="cuda").manual_seed(1)
    A = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    Bs = [(torch.randn((2 if act else 1) * N, K, device="cuda", generator=g) / K ** 0.5).bfloat16() for _ in range(W)]
    Cs = [torch.empty(M, N, device="cuda", dtype=torch.bfloat16) for _ in range(W)]
    Ag = [torch.empty(M, K, device="cuda", dtype=torch.bfloat16) for _ in range(W)]
    shards = list(A.chunk(W, 0))
    shards = [s.contiguous() for s in shards]
    c.ag_gemm_lb(shards, Bs, Cs, Ag, act=act)
    st, d = c.check()
    errs = []
    for r in range(W):
        Y = A.float() @ Bs[r].float().T
        ref = torch.nn.functional.silu(Y[:, :N]) * Y[:, N:] if act == 1 else Y
        errs.append(rel(Cs[r], ref))
        assert torch.equal(Ag[r], A), f"gathered A mismatch on rank {r}"
    print(f"loopback AG W={W} M={M} N={N} K={K} act={act}: status={st} diag={d} rel={max(errs):.3e}", flush=True)


def loop_rs(W, M, N, K, ring=0):
    c = tl.Comm.loopback(W, 0, max_M=M, max_H=N)
    c.set_option("rs_order", ring)
    g = torch.Generator(device="cuda").manual_seed(2)
    As = [torch.randn(M, K, device="cuda", generator=g).bfloat16() for _ in range(W)]
    Bs = [(torch.randn(N, K, device="cuda", generator=g) / (W * K) ** 0.5).bfloat16() for _ in range(W)]
    Cs = [torch.empty(M // W, N, device="cuda", dtype=torch.bfloat16) for _ in range(W)]
    c.gemm_rs_lb(As, Bs, Cs)
    st, d = c.check()
    P = sum(As[s].double() @ Bs[s].double().T for s in range(W))
    errs = [rel(Cs[r], P[r * (M // W):(r + 1) * (M // W)]) for r in range(W)]
    print(f"loopback RS W={W} M={M} N={N} K={K} ring={ring}: status={st} diag={d} rel={max(errs):.3e}", flush=True)


if __name__ == "__main__":
    what = sys.argv[1]
    args = [int(x) for x in sys.argv[2:]]
    {"gemm": gemm, "ag": loop_ag, "rs": loop_rs}[what](*args)
