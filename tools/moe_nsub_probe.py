"""MoE second half: n_sub = 1 (256x256 tiles, double-buffered TMEM: the scatter epilogue overlaps the
next tile's MMAs) vs n_sub = 2 (256x512 tiles, one accumulator) on the paper's MoE shapes."""
import json
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2503_20313_b200 as tl  # noqa: E402
import tl_inputs as TI  # noqa: E402
from tools.moe_bench import SHAPES, timeit  # noqa: E402

for name, (S, H, I, E, topk) in SHAPES.items():
    for W in (1, 8):
        il = I // W
        X = TI._randn((S, H), 0, 0).cuda()
        Wt = TI.moe_weights(E, 2 * il, H, 1, seed=1)[0].cuda()
        ids = TI.moe_routing(S, E, topk, seed=2).cuda()
        c = tl.Comm.single(0, max_M=S, max_H=H, max_topk=topk)
        R = tl.moe_capacity(c, S, topk, E)
        Y = torch.empty(R, il, device="cuda", dtype=torch.bfloat16)
        rows = torch.empty(R, device="cuda", dtype=torch.int32)
        offs = torch.empty(E + 1, device="cuda", dtype=torch.int32)
        res0 = {}
        Ys = {}
        for ns in (1, 2):
            c.set_option("n_sub", ns)
            Yn = torch.empty_like(Y)
            res0[f"first_nsub{ns}_ms"] = round(timeit(lambda: tl.moe_ag_gemm(c, X, ids, Wt, Yn, rows, offs,
                                                                             act=tl.ACT_SILU_MUL)), 4)
            Ys[ns] = Yn
        valid = (rows >= 0) & (torch.arange(R, device="cuda") < offs[-1])   # rows past offs[E] are unwritten
        res0["first_equal"] = bool(torch.equal(Ys[1][valid], Ys[2][valid]))
        Y = Ys[1]
        W2t = TI.moe_down_weights(E, H, il, 1, seed=3)[0].cuda()
        wts = TI.moe_topk_weights(S, topk, seed=4).cuda()
        res = {"name": name, "W": W, **res0}
        outs = {}
        for ns in (1, 2):
            c.set_option("n_sub", ns)
            out = torch.empty(S, H, device="cuda", dtype=torch.bfloat16)
            res[f"nsub{ns}_ms"] = round(timeit(lambda: tl.moe_gemm_rs(c, Y, rows, offs, wts, W2t, out)), 4)
            outs[ns] = out
        res["equal"] = bool(torch.equal(outs[1], outs[2]))
        print(json.dumps(res), flush=True)
