"""A/B of option moe_split (MoE gather GroupGEMM split tail) on the paper's MoE shapes, W = 1 and the TP-8
rank's local shape (I/8): tl_moe_ag_gemm time per call, round robin; outputs must be bitwise equal."""
import json
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2503_20313_b200 as tl  # noqa: E402
import tl_inputs as TI  # noqa: E402

SHAPES = {"MoE-1": (8192, 2048, 1536, 8, 2), "MoE-2": (8192, 2048, 1536, 32, 2), "MoE-3": (8192, 2048, 1536, 32, 5),
          "MoE-4": (8192, 4096, 2048, 8, 2), "MoE-5": (8192, 4096, 2048, 32, 2), "MoE-6": (8192, 4096, 2048, 32, 5)}


def run(name, tp):
    M, H, I, E, topk = SHAPES[name]
    Il = I // tp
    X = TI._randn((M, H), 0, 0).cuda()
    W1 = TI.moe_weights(E, 2 * Il, H, 1, seed=1)[0].cuda()
    ids = TI.moe_routing(M, E, topk, seed=2).cuda()
    res, outs = {}, {}
    comms = {}
    for split in (0, 1):
        c = tl.Comm.single(0, max_M=M, max_H=H)
        c.set_option("moe_split", split)
        comms[split] = c
    R = tl.moe_capacity(comms[0], M, topk, E)
    bufs = {s: (torch.empty(R, Il, device="cuda", dtype=torch.bfloat16), torch.empty(R, device="cuda", dtype=torch.int32),
                torch.empty(E + 1, device="cuda", dtype=torch.int32)) for s in (0, 1)}
    call = lambda s: tl.moe_ag_gemm(comms[s], X, ids, W1, *bufs[s], act=tl.ACT_SILU_MUL)
    for s in (0, 1):
        for _ in range(3):
            call(s)
    torch.cuda.synchronize()
    for rnd in range(6):
        for s in (0, 1):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(20):
                call(s)
            b.record()
            torch.cuda.synchronize()
            res.setdefault(s, []).append(a.elapsed_time(b) / 20)
    n = int(bufs[0][2][-1].item())
    eq = torch.equal(bufs[0][0][:n], bufs[1][0][:n])
    flop = 2 * M * topk * H * 2 * Il
    out = {"shape": name, "tp": tp, "equal": bool(eq)}
    for s in (0, 1):
        ms = sorted(res[s])[len(res[s]) // 2]
        out[f"split{s}_ms"] = round(ms, 4)
        out[f"split{s}_tflops"] = round(flop / ms / 1e9, 1)
    print(json.dumps(out), flush=True)


for name in SHAPES:
    for tp in (1, 8):
        run(name, tp)
