"""Tile-width choice (option n_sub: 1 = 256-wide + double-buffered accumulator, 2 = 512-wide, 0 = the
library's time model) per GEMM of the per-rank TP-W MLP shapes; round-robin, median of rounds."""
import json
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2503_20313_b200 as tl  # noqa: E402
from tools.sweep import timeit  # noqa: E402

SHAPES = [("llama7b", 8192, 4096, 11008), ("llama70b", 8192, 8192, 28672), ("mixtral", 16384, 4096, 14336)]
for name, M, H, I in SHAPES:
    for W in (1, 2, 4, 8):
        il = I // W
        g = torch.Generator(device="cuda").manual_seed(W)
        x = torch.randn(M, H, device="cuda", generator=g).bfloat16()
        w1 = (torch.randn(2 * il, H, device="cuda", generator=g) * H ** -0.5).bfloat16()
        w2 = (torch.randn(H, il, device="cuda", generator=g) * I ** -0.5).bfloat16()
        c = tl.Comm.single(0, max_M=M, max_H=H)
        Z = torch.empty(M, il, device="cuda", dtype=torch.bfloat16)
        out = torch.empty(M, H, device="cuda", dtype=torch.bfloat16)
        res = {}
        for rnd in range(3):
            for ns in (0, 1, 2):
                c.set_option("n_sub", ns)
                res.setdefault(("g1", ns), []).append(timeit(lambda: c.ag_gemm(x, w1, Z, act=tl.ACT_SILU_MUL)))
                res.setdefault(("g2", ns), []).append(timeit(lambda: c.gemm_rs(Z, w2, out)))
        f1, f2 = 2 * M * H * 2 * il, 2 * M * il * H
        row = {"name": name, "W": W}
        for (g_, ns), v in res.items():
            ms = sorted(v)[1]
            row[f"{g_}_ns{ns}_tf"] = round((f1 if g_ == "g1" else f2) / ms / 1e9, 1)
        print(json.dumps(row), flush=True)
        c.close()
