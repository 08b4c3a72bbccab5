"""MoE first half (AG + Gather + GroupGEMM + SiLU*up) on the paper's MoE shapes, one GPU:
W = 1 (whole layer) against a torch baseline (index gather + per-expert cuBLAS matmul + silu*mul),
and the TP-8 rank's local work; sampled-row oracle check."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2503_20313_b200 as tl  # noqa: E402
import tl_inputs as TI  # noqa: E402
from oracle import tl_oracle as O  # noqa: E402

SHAPES = {"MoE-1": (8192, 2048, 1536, 8, 2), "MoE-2": (8192, 2048, 1536, 32, 2), "MoE-3": (8192, 2048, 1536, 32, 5),
          "MoE-4": (8192, 4096, 2048, 8, 2), "MoE-5": (8192, 4096, 2048, 32, 2), "MoE-6": (8192, 4096, 2048, 32, 5)}


def timeit(fn, n=10, w=3):
    for _ in range(w):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


def run(name, S, H, I, E, topk, W=1):
    il = I // W
    X = TI._randn((S, H), 0, 0).cuda()
    Wt = TI.moe_weights(E, 2 * il, H, 1, seed=1)[0].cuda()
    ids = TI.moe_routing(S, E, topk, seed=2).cuda()
    c = tl.Comm.single(0, max_M=S, max_H=H)
    R = tl.moe_capacity(c, S, topk, E)
    Y = torch.empty(R, il, device="cuda", dtype=torch.bfloat16)
    rows = torch.empty(R, device="cuda", dtype=torch.int32)
    offs = torch.empty(E + 1, device="cuda", dtype=torch.int32)
    ms = timeit(lambda: tl.moe_ag_gemm(c, X, ids, Wt, Y, rows, offs, act=tl.ACT_SILU_MUL))

    flat = ids.flatten().long()
    order = torch.argsort(flat, stable=True)
    tok = order // topk
    counts = torch.bincount(flat, minlength=E).tolist()

    def base():
        xs = X.index_select(0, tok)                       # gather (not fused)
        outs, o = [], 0
        for e in range(E):
            n = counts[e]
            y = xs[o:o + n] @ Wt[e].T
            outs.append(torch.nn.functional.silu(y[:, :il]) * y[:, il:])
            o += n
        return torch.cat(outs)
    bms = timeit(base)
    fl = 2.0 * S * topk * H * 2 * il
    rid = rows.cpu().numpy()
    valid = np.nonzero(rid[:offs[-1].item()] >= 0)[0]
    samp = valid[np.linspace(0, len(valid) - 1, 8).astype(int)]
    Xd = TI.to_f64(X.cpu())
    Wd = TI.to_f64(Wt.cpu())
    err_num = err_den = 0.0
    for g in samp:
        t, k = divmod(int(rid[g]), topk)
        e = int(ids[t, k])
        ref = O.activation(Xd[t][None, :] @ Wd[e].T, O.ACT_SILU_MUL)[0]
        got = Y[g].float().cpu().double().numpy()
        err_num += float(((got - ref) ** 2).sum())
        err_den += float((ref ** 2).sum())
    # second half: GroupGEMM + Scatter + TopK reduce (+RS, W = 1 here) on the grouped output
    c2 = tl.Comm.single(0, max_M=S, max_H=H, max_topk=topk)
    W2t = TI.moe_down_weights(E, H, il, 1, seed=3)[0].cuda()
    wts = TI.moe_topk_weights(S, topk, seed=4).cuda()
    out = torch.empty(S, H, device="cuda", dtype=torch.bfloat16)
    ms2 = timeit(lambda: tl.moe_gemm_rs(c2, Y, rows, offs, wts, W2t, out))
    fl2 = 2.0 * S * topk * il * H

    def base2():
        z = Y[:S * topk]                                   # same amount of grouped work
        outs, o = [], 0
        for e in range(E):
            n = counts[e]
            outs.append(z[o:o + n] @ W2t[e].T)
            o += n
        p = torch.cat(outs) * wts.flatten()[order].unsqueeze(1).to(torch.bfloat16)
        res = torch.zeros(S, H, device="cuda", dtype=torch.float32)
        res.index_add_(0, tok, p.float())
        return res
    bms2 = timeit(base2)
    r = {"name": name, "S": S, "H": H, "I": I, "E": E, "topk": topk, "W": W, "ms": round(ms, 4),
         "second_half_ms": round(ms2, 4), "second_half_tflops": round(fl2 / ms2 / 1e9, 1),
         "torch_second_half_ms": round(bms2, 4), "layer_ms": round(ms + ms2, 4),
         "layer_speedup_vs_torch": round((bms + bms2) / (ms + ms2), 3),
         "tflops": round(fl / ms / 1e9, 1), "torch_gather_cublas_ms": round(bms, 4),
         "speedup": round(bms / ms, 3), "padding_rows": int(R - S * topk),
         "parity_rel_fro_sampled": (err_num / err_den) ** 0.5}
    print(json.dumps(r), flush=True)
    return r


if __name__ == "__main__":
    only = set(sys.argv[1:])          # e.g. MoE-4 MoE-1_rank_of_tp8 (default: all)
    out = []
    for n, (S, H, I, E, k) in SHAPES.items():
        for name, W in ((n, 1), (n + "_rank_of_tp8", 8)):
            if not only or name in only:
                out.append(run(name, S, H, I, E, k, W=W))
    if not only:
        json.dump(out, open("gpurun_out/moe_bench.json", "w"), indent=1)
