"""Attention timing probe: tl_sp_attention vs torch SDPA (flash / cuDNN backends) on
the paper's Attn-1/2 head shapes.  W = 1 (one GPU's whole sequence) and the per-rank shape of a TP-8
run (S_r = S/8 queries over the full S keys, K/V gathered by the loopback comm in the same launch).
Prints one JSON object per config; CUDA events on the launching stream, L2 flushed between reps."""
import json
import sys

import torch
import torch.nn.functional as F

sys.path.insert(0, ".")
import paper_2503_20313_b200 as tl  # noqa: E402


def timeit(fn, reps=10, warm=3):
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(warm):
        fn()
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


def main():
    configs = [(1, 4096, 32), (1, 16384, 32), (1, 16384, 64), (8, 16384, 32), (8, 32768, 32)]
    if len(sys.argv) > 1:
        configs = [tuple(int(x) for x in a.split(",")) for a in sys.argv[1:]]
    D = 128
    for W, S, heads in configs:
        S_r = S // W
        g = torch.Generator(device="cuda").manual_seed(0)
        Q = torch.randn(S_r, heads, D, device="cuda", generator=g).to(torch.bfloat16)
        Ks = [torch.randn(S_r, heads, D, device="cuda", generator=g).to(torch.bfloat16) for _ in range(W)]
        Vs = [torch.randn(S_r, heads, D, device="cuda", generator=g).to(torch.bfloat16) for _ in range(W)]
        need = 2 * S * heads * D
        comm = (tl.Comm.loopback(W, 0, max_M=need // 4096 + 128, max_H=4096) if W > 1
                else tl.Comm.single(0, max_M=128, max_H=128))
        flops_rank = 4.0 * S_r * S * heads * D
        if W == 1:
            O = torch.empty_like(Q)
            ms = timeit(lambda: tl.sp_attention(comm, Q, Ks[0], Vs[0], O))
            total = flops_rank
        else:
            Qs = [Q] + [torch.randn_like(Q) for _ in range(W - 1)]
            Os = [torch.empty_like(Q) for _ in range(W)]
            ms = timeit(lambda: tl.sp_attention_lb(comm, Qs, Ks, Vs, Os))
            total = flops_rank * W
        # library baseline: SDPA over the gathered K/V (one rank's shape, no communication)
        Kf, Vf = torch.cat(Ks, 0), torch.cat(Vs, 0)
        q4, k4, v4 = (t.transpose(0, 1).unsqueeze(0) for t in (Q, Kf, Vf))
        res = {"W": W, "S": S, "heads": heads, "tl_ms": round(ms, 4), "tl_tflops": round(total / ms / 1e9, 1)}
        for name, be in (("flash", torch.nn.attention.SDPBackend.FLASH_ATTENTION),
                         ("cudnn", torch.nn.attention.SDPBackend.CUDNN_ATTENTION)):
            try:
                with torch.nn.attention.sdpa_kernel(be):
                    ms_b = timeit(lambda: F.scaled_dot_product_attention(q4, k4, v4))
                res[f"{name}_rank_ms"] = round(ms_b, 4)
                res[f"{name}_tflops"] = round(flops_rank / ms_b / 1e9, 1)
            except Exception as e:  # backend not available for this shape
                res[f"{name}_err"] = str(e)[:80]
        print(json.dumps(res), flush=True)
        del comm


if __name__ == "__main__":
    main()
