"""MoE layer vs vLLM's fused MoE kernel (the paper's MoE baseline: TileLink 1.51x / 1.31x /
1.14x over vLLM for part 1 / part 2 / the layer on H800) on the paper's MoE shapes, one GPU: the whole
layer (W = 1) and a TP-8 rank's local compute (expert weights sharded along I; vLLM's TP MoE runs
fused_experts on every token with the shard, then an all-reduce that is not timed here)."""
import json
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2503_20313_b200 as tl  # noqa: E402
import tl_inputs as TI  # noqa: E402
from tools.moe_bench import SHAPES, timeit  # noqa: E402

from vllm.model_executor.layers.fused_moe import fused_experts  # noqa: E402

only = set(sys.argv[1:])
for name, (S, H, I, E, topk) in SHAPES.items():
    for W in (1, 8):
        tag = name if W == 1 else name + "_rank_of_tp8"
        if only and tag not in only:
            continue
        il = I // W
        X = TI._randn((S, H), 0, 0).cuda()
        W1 = TI.moe_weights(E, 2 * il, H, 1, seed=1)[0].cuda()
        W2 = TI.moe_down_weights(E, H, il, 1, seed=3)[0].cuda()
        ids = TI.moe_routing(S, E, topk, seed=2).cuda()
        wts = TI.moe_topk_weights(S, topk, seed=4).cuda()
        c = tl.Comm.single(0, max_M=S, max_H=H, max_topk=topk)
        R = tl.moe_capacity(c, S, topk, E)
        Y = torch.empty(R, il, device="cuda", dtype=torch.bfloat16)
        rows = torch.empty(R, device="cuda", dtype=torch.int32)
        offs = torch.empty(E + 1, device="cuda", dtype=torch.int32)
        out = torch.empty(S, H, device="cuda", dtype=torch.bfloat16)

        def ours():
            tl.moe_ag_gemm(c, X, ids, W1, Y, rows, offs, act=tl.ACT_SILU_MUL)
            tl.moe_gemm_rs(c, Y, rows, offs, wts, W2, out)

        def vllm():
            return fused_experts(X, W1, W2, wts, ids)
        t_ours, t_vllm = timeit(ours), timeit(vllm)
        ref = vllm().float()
        ours()
        err = float((out.float() - ref).norm() / ref.norm())
        fl = 2.0 * S * topk * H * 3 * il
        print(json.dumps({"name": tag, "ours_ms": round(t_ours, 4), "vllm_fused_moe_ms": round(t_vllm, 4),
                          "speedup_vs_vllm": round(t_vllm / t_ours, 3), "ours_tflops": round(fl / t_ours / 1e9, 1),
                          "vllm_tflops": round(fl / t_vllm / 1e9, 1), "rel_diff_vs_vllm": round(err, 5)}),
              flush=True)
        c.close()
