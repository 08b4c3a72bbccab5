"""Attention: fraction of exp2 on the FMA pipe (option attn_poly = every n-th pair; 0 = all MUFU).
W = 1, Attn-1 head shape; CUDA events, L2 flushed, median of 10 (tools/attn_bench.timeit)."""
import json
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2503_20313_b200 as tl  # noqa: E402
from tools.attn_bench import timeit  # noqa: E402

polys = [int(a) for a in sys.argv[1:]] or [0, 2, 3, 4, 6, 8]
for S, heads in ((16384, 32), (4096, 32)):
    g = torch.Generator(device="cuda").manual_seed(0)
    Q, K, V = (torch.randn(S, heads, 128, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
    O = torch.empty_like(Q)
    comm = tl.Comm.single(0, max_M=128, max_H=128)
    ref = None
    res = {pm: [] for pm in polys}
    for rnd in range(4):                      # round-robin: clock / power drift hits every variant alike
        for pm in polys:
            comm.set_option("attn_poly", pm)
            res[pm].append(timeit(lambda: tl.sp_attention(comm, Q, K, V, O)))
            if ref is None:
                ref = O.float().clone()
    for pm in polys:
        ms = sorted(res[pm])[len(res[pm]) // 2]
        print(json.dumps({"S": S, "heads": heads, "attn_poly": pm, "ms_median_of_rounds": round(ms, 4),
                          "tflops": round(4.0 * S * S * heads * 128 / ms / 1e9, 1),
                          "all_ms": [round(x, 4) for x in res[pm]]}), flush=True)
    del comm
