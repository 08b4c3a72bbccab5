"""Programmatic dependent launch on/off (option pdl) for the two-kernel MLP layer and the MoE layer on
small (TP-8 rank) and full shapes: round-robin medians, bitwise-equal outputs."""
import json
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2503_20313_b200 as tl  # noqa: E402
import tl_inputs as TI  # noqa: E402
from tools.sweep import timeit  # noqa: E402

for name, M, H, I, W in (("llama7b_rank_of_tp8", 8192, 4096, 11008, 8), ("llama7b_M1024", 1024, 4096, 11008, 1),
                         ("llama7b", 8192, 4096, 11008, 1)):
    il = I // W
    g = torch.Generator(device="cuda").manual_seed(1)
    x = torch.randn(M, H, device="cuda", generator=g).bfloat16()
    w1 = (torch.randn(2 * il, H, device="cuda", generator=g) * H ** -0.5).bfloat16()
    w2 = (torch.randn(H, il, device="cuda", generator=g) * I ** -0.5).bfloat16()
    c = tl.Comm.single(0, max_M=M, max_H=H)
    Z = torch.empty(M, il, device="cuda", dtype=torch.bfloat16)
    outs = {0: torch.empty(M, H, device="cuda", dtype=torch.bfloat16), 1: torch.empty(M, H, device="cuda", dtype=torch.bfloat16)}
    res = {0: [], 1: []}
    for rnd in range(5):
        for pdl in (0, 1):
            c.set_option("pdl", pdl)
            res[pdl].append(timeit(lambda: c.mlp_forward(x, w1, w2, outs[pdl], act=tl.ACT_SILU_MUL, Z=Z), steps=20))
    med = {k: sorted(v)[2] for k, v in res.items()}
    print(json.dumps({"name": name, "pdl0_ms": round(med[0], 4), "pdl1_ms": round(med[1], 4),
                      "gain": round(med[0] / med[1], 4), "equal": bool(torch.equal(outs[0], outs[1]))}), flush=True)
