"""Per-GEMM timing probe of the per-rank MLP shapes (W=1 layer or the local GEMMs of a TP-W rank),
ours vs cuBLAS, with nvidia-smi clock samples.  Inputs drawn on the GPU (timing only, no parity).

  python tools/r02_probe.py [name ...]      names: 7b 70b mix 7b_tp2 7b_tp4 7b_tp8 70b_tp2 ... mix_tp8
  env TL_PROBE_OPTS="n_sub=2,raster_group=8"  comm options applied before timing
"""
import json
import os
import subprocess
import sys
import time

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2503_20313_b200 as tl  # noqa: E402

SHAPES = {"7b": (8192, 4096, 11008), "70b": (8192, 8192, 28672), "mix": (16384, 4096, 14336)}


def timeit(fn, steps=20, warm=5):
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


def run(name, steps):
    base, _, tp = name.partition("_tp")
    W = int(tp) if tp else 1
    M, H, I = SHAPES[base]
    il = I // W
    g = torch.Generator(device="cuda").manual_seed(1)
    x = torch.randn(M, H, device="cuda", generator=g).bfloat16()
    w1 = (torch.randn(2 * il, H, device="cuda", generator=g) * H ** -0.5).bfloat16()
    w2 = (torch.randn(H, il, device="cuda", generator=g) * I ** -0.5).bfloat16()
    c = tl.Comm.single(0, max_M=M, max_H=H)
    for kv in filter(None, os.environ.get("TL_PROBE_OPTS", "").split(",")):
        k, v = kv.split("=")
        c.set_option(k, int(v))
    Z = torch.empty(M, il, device="cuda", dtype=torch.bfloat16)
    out = torch.empty(M, H, device="cuda", dtype=torch.bfloat16)
    f1, f2 = 2 * M * H * 2 * il, 2 * M * il * H
    r = {"name": name, "M": M, "H": H, "I_l": il}
    r["g1_ms"] = timeit(lambda: c.ag_gemm(x, w1, Z, act=tl.ACT_SILU_MUL), steps)
    r["g2_ms"] = timeit(lambda: c.gemm_rs(Z, w2, out), steps)
    r["layer_ms"] = timeit(lambda: (c.ag_gemm(x, w1, Z, act=tl.ACT_SILU_MUL), c.gemm_rs(Z, w2, out)), steps)
    y = torch.empty(M, 2 * il, device="cuda", dtype=torch.bfloat16)
    r["cublas_g1_ms"] = timeit(lambda: torch.matmul(x, w1.T, out=y), steps)
    r["cublas_g2_ms"] = timeit(lambda: torch.matmul(Z, w2.T, out=out), steps)
    r["g1_tf"] = f1 / r["g1_ms"] / 1e9
    r["g2_tf"] = f2 / r["g2_ms"] / 1e9
    r["layer_tf"] = (f1 + f2) / r["layer_ms"] / 1e9
    r["cublas_g1_tf"] = f1 / r["cublas_g1_ms"] / 1e9
    r["cublas_g2_tf"] = f2 / r["cublas_g2_ms"] / 1e9
    r["opts"] = {k: c.get_option(k) for k in ("n_sub", "raster_group")}
    c.close()
    return {k: (round(v, 4) if isinstance(v, float) else v) for k, v in r.items()}


if __name__ == "__main__":
    names = sys.argv[1:] or ["70b", "mix", "7b", "7b_tp4", "7b_tp8", "70b_tp8", "mix_tp8"]
    steps = int(os.environ.get("TL_PROBE_STEPS", "20"))
    smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.active",
                            "--format=csv,noheader,nounits", "-lms", "200"], stdout=subprocess.PIPE, text=True)
    for n in names:
        t0 = time.time()
        print(json.dumps(run(n, steps)), flush=True)
    smi.terminate()
    lines = [ln.strip() for ln in smi.stdout.read().splitlines() if ln.strip()]
    clk = [float(ln.split(",")[0]) for ln in lines if ln.split(",")[0].strip().replace(".", "").isdigit()]
    pw = [float(ln.split(",")[1]) for ln in lines if len(ln.split(",")) > 1 and ln.split(",")[1].strip().replace(".", "").isdigit()]
    load = sorted(x for x in clk if x > 600)
    print(json.dumps({"clock_median_load": load[len(load) // 2] if load else None, "power_max": max(pw) if pw else None,
                      "samples": len(clk)}))
