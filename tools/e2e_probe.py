"""End-to-end pipeline probe (bench.py's e2e leg): the LLaMA-7B MLP layer with the X shard copied in
from pinned host memory and the output copied back every step, vs compute alone and vs one copy
direction alone, for pipeline depths 2 and 3 (paper_2503_20313_b200.pipeline.MLPPipeline)."""
import json
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2503_20313_b200 as tl  # noqa: E402
import tl_inputs as TI  # noqa: E402
from paper_2503_20313_b200.pipeline import MLPPipeline  # noqa: E402

M, H, I = 8192, 4096, 11008
X, G, U, W2 = TI.mlp_full(M, H, I, seed=0)
Xs, W1s, W2s = TI.shard_mlp(X, G, U, W2, 1, TI.ACT_SILU_MUL)
w1, w2 = W1s[0].cuda(), W2s[0].cuda()
comm = tl.Comm.single(0, M, H)
steps = 20
hx = [Xs[0].pin_memory(), (Xs[0].float() * -1).to(torch.bfloat16).pin_memory()]
hin = [hx[i % 2] for i in range(steps)]
hout = [torch.empty(M, H, dtype=torch.bfloat16).pin_memory() for _ in range(steps)]


def timed(fn):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / steps


res = {}
x = Xs[0].cuda()
out = torch.empty(M, H, device="cuda", dtype=torch.bfloat16)
Z = torch.empty(M, I, device="cuda", dtype=torch.bfloat16)
res["compute_only_ms"] = timed(lambda: [comm.mlp_forward(x, w1, w2, out, act=tl.ACT_SILU_MUL, Z=Z) for _ in range(steps)])
for depth in (2, 3):
    pipe = MLPPipeline(comm, w1, w2, tl.ACT_SILU_MUL, M, H, depth=depth)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    pipe.run(hin[:3], hout[:3])
    torch.cuda.synchronize()
    pipe.run(hin, hout, e0, e1)
    torch.cuda.synchronize()
    res[f"pipeline_depth{depth}_ms"] = e0.elapsed_time(e1) / steps
s2 = torch.cuda.Stream()


def h2d_and_compute():
    for i in range(steps):
        with torch.cuda.stream(s2):
            pipe.x[i % 2].copy_(hin[i], non_blocking=True)
        comm.mlp_forward(x, w1, w2, out, act=tl.ACT_SILU_MUL, Z=Z)
    torch.cuda.current_stream().wait_stream(s2)


def d2h_and_compute():
    for i in range(steps):
        with torch.cuda.stream(s2):
            hout[i].copy_(pipe.out[i % 2], non_blocking=True)
        comm.mlp_forward(x, w1, w2, out, act=tl.ACT_SILU_MUL, Z=Z)
    torch.cuda.current_stream().wait_stream(s2)


res["h2d_overlapping_compute_ms"] = timed(h2d_and_compute)
res["d2h_overlapping_compute_ms"] = timed(d2h_and_compute)
res["h2d_alone_ms"] = timed(lambda: [pipe.x[i % 2].copy_(hin[i], non_blocking=True) for i in range(steps)])
res["d2h_alone_ms"] = timed(lambda: [hout[i].copy_(pipe.out[i % 2], non_blocking=True) for i in range(steps)])
print(json.dumps({k: round(v, 4) for k, v in res.items()}))
