"""Single-GPU sweep over BASELINE.json's workloads: the full layer at W = 1 and the per-rank
compute of the W = 2/4/8 configs (the local GEMM shapes an 8-GPU rank runs once the AG/RS bytes
are hidden), against cuBLAS (+ silu*mul) on the same inputs, with a sampled-row oracle check."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2503_20313_b200 as tl  # noqa: E402
import tl_inputs as TI  # noqa: E402
from oracle import tl_oracle as O  # noqa: E402

P_BURST = 1638.8


def timeit(fn, steps=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def layer(name, M, H, I, W=1, check=True):
    """Per-rank layer of a TP-W config computed at W = 1 on this GPU (W = 1: the whole layer)."""
    il = I // W
    g = torch.Generator(device="cuda").manual_seed(M + H + I + W)
    if check:
        X, G, U, W2f = TI.mlp_full(M, H, I, seed=1)
        Xs, W1s, W2s = TI.shard_mlp(X, G, U, W2f, W, TI.ACT_SILU_MUL)
        x = X.cuda()                                  # the gathered activation of every rank
        w1, w2 = W1s[0].cuda(), W2s[0].cuda()
    else:
        x = torch.randn(M, H, device="cuda", generator=g).bfloat16()
        w1 = (torch.randn(2 * il, H, device="cuda", generator=g) * H ** -0.5).bfloat16()
        w2 = (torch.randn(H, il, device="cuda", generator=g) * I ** -0.5).bfloat16()
    c = tl.Comm.single(0, max_M=M, max_H=H)
    Z = torch.empty(M, il, device="cuda", dtype=torch.bfloat16)
    out = torch.empty(M, H, device="cuda", dtype=torch.bfloat16)
    t1 = timeit(lambda: c.ag_gemm(x, w1, Z, act=tl.ACT_SILU_MUL))
    t2 = timeit(lambda: c.gemm_rs(Z, w2, out))
    tl_ms = timeit(lambda: (c.ag_gemm(x, w1, Z, act=tl.ACT_SILU_MUL), c.gemm_rs(Z, w2, out)))

    def base():
        y = x @ w1.T
        z = torch.nn.functional.silu(y[:, :il]) * y[:, il:]
        return z @ w2.T
    b_ms = timeit(base)
    f = 2 * M * H * 2 * il + 2 * M * il * H
    r = {"name": name, "M": M, "H": H, "I": I, "W": W, "gemm1_ms": round(t1, 4), "gemm2_ms": round(t2, 4),
         "layer_ms": round(tl_ms, 4), "tflops": round(f / tl_ms / 1e9, 1),
         "frac_of_burst": round(f / tl_ms / 1e9 / P_BURST, 4), "cublas_ms": round(b_ms, 4),
         "speedup_vs_cublas": round(b_ms / tl_ms, 3)}
    if check and W == 1:
        rows = [0, M // 3, M - 1]
        ref = O.mlp_forward_rows([TI.to_f64(t) for t in Xs], [TI.to_f64(t) for t in W1s],
                                 [TI.to_f64(t) for t in W2s], TI.ACT_SILU_MUL, rows)
        got = out.float().cpu().double().numpy()
        r["parity_rel_fro"] = O.rel_frobenius(np.stack([got[i] for i in rows]), np.stack([ref[i] for i in rows]))
    c.close()
    print(json.dumps(r), flush=True)
    return r


if __name__ == "__main__":
    res = []
    res.append(layer("llama7b", 8192, 4096, 11008))
    res.append(layer("llama70b", 8192, 8192, 28672))
    res.append(layer("mixtral_ffn", 16384, 4096, 14336))
    for M in (1024, 2048, 4096, 16384, 32768):
        res.append(layer(f"llama7b_M{M}", M, 4096, 11008, check=(M <= 16384)))
    for W in (2, 4, 8):
        res.append(layer(f"llama7b_rank_of_tp{W}", 8192, 4096, 11008, W=W, check=False))
        res.append(layer(f"llama70b_rank_of_tp{W}", 8192, 8192, 28672, W=W, check=False))
        res.append(layer(f"mixtral_rank_of_tp{W}", 16384, 4096, 14336, W=W, check=False))
    json.dump(res, open("gpurun_out/sweep.json", "w"), indent=1)
