"""Interleaved A/B of comm options on one per-rank MLP shape: time (CUDA events) and energy (NVML total
energy counter) per call, round-robin over the configurations so thermal / power-cap drift hits all
alike.  Under the 1 kW cap the energy per call is the quantity a kernel change must lower.

  python tools/ab.py SHAPE OP "optsA" "optsB" ...   SHAPE: 70b | 7b | mix [ _tpW ]   OP: g1 | g2 | layer
  opts: "n_sub=2,raster_group=8" (empty string = defaults);  env AB_ROUNDS, AB_ITERS, AB_LIB=path (B build)
"""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2503_20313_b200 as tl  # noqa: E402

SHAPES = {"7b": (8192, 4096, 11008), "70b": (8192, 8192, 28672), "mix": (16384, 4096, 14336)}


def main():
    shape, op, *cfgs = sys.argv[1:]
    base, _, tp = shape.partition("_tp")
    W = int(tp) if tp else 1
    M, H, I = SHAPES[base]
    if "_M" in base:
        pass
    il = I // W
    g = torch.Generator(device="cuda").manual_seed(1)
    x = torch.randn(M, H, device="cuda", generator=g).bfloat16()
    w1 = (torch.randn(2 * il, H, device="cuda", generator=g) * H ** -0.5).bfloat16()
    w2 = (torch.randn(H, il, device="cuda", generator=g) * I ** -0.5).bfloat16()
    Z = torch.empty(M, il, device="cuda", dtype=torch.bfloat16)
    out = torch.empty(M, H, device="cuda", dtype=torch.bfloat16)
    f1, f2 = 2 * M * H * 2 * il, 2 * M * il * H
    flops = {"g1": f1, "g2": f2, "layer": f1 + f2, "mlp": f1 + f2}[op]
    comms = []
    for cfg in cfgs:
        c = tl.Comm.single(0, max_M=M, max_H=H)
        for kv in filter(None, cfg.split(",") if cfg != "cublas" else []):
            k, v = kv.split("=")
            c.set_option(k, int(v))
        comms.append(c)
    y = torch.empty(M, 2 * il, device="cuda", dtype=torch.bfloat16)

    def run(ci):
        c = comms[ci]
        if cfgs[ci] == "cublas":
            if op in ("g1", "layer", "mlp"):
                torch.matmul(x, w1.T, out=y)
            if op in ("g2", "layer", "mlp"):
                torch.matmul(Z, w2.T, out=out)
            return
        if op == "mlp":      # tl_mlp_forward (one fused launch unless mlp_fused = 0)
            c.mlp_forward(x, w1, w2, out, act=tl.ACT_SILU_MUL, Z=Z)
            return
        if op in ("g1", "layer"):
            c.ag_gemm(x, w1, Z, act=tl.ACT_SILU_MUL)
        if op in ("g2", "layer"):
            c.gemm_rs(Z, w2, out)

    import threading
    import time
    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
    samples = []          # (t, watts, sm MHz) every ~10 ms (the energy counter is too coarse here)
    stop = [False]

    def sampler():
        while not stop[0]:
            try:
                samples.append((time.perf_counter(), pynvml.nvmlDeviceGetPowerUsage(h) / 1e3,
                                pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)))
            except Exception:
                pass
            time.sleep(0.01)
    th = threading.Thread(target=sampler, daemon=True)
    th.start()
    rounds, iters = int(os.environ.get("AB_ROUNDS", "6")), int(os.environ.get("AB_ITERS", "20"))
    for ci in range(len(cfgs)):
        for _ in range(3):
            run(ci)
    torch.cuda.synchronize()
    res = {ci: {"ms": [], "mj": [], "mhz": []} for ci in range(len(cfgs))}
    for r in range(rounds):
        order = list(range(len(cfgs))) if r % 2 == 0 else list(reversed(range(len(cfgs))))
        for ci in order:
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(iters):
                run(ci)
            b.record()
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            ms = a.elapsed_time(b) / iters
            win = [s for s in samples if t0 + 0.2 * (t1 - t0) <= s[0] <= t1]   # skip the ramp
            pw = statistics.mean(s[1] for s in win) if win else float("nan")
            res[ci]["ms"].append(ms)
            res[ci]["mj"].append(pw * ms)             # W x ms = mJ
            res[ci]["mhz"].append(statistics.median(s[2] for s in win) if win else float("nan"))
    stop[0] = True
    for ci, cfg in enumerate(cfgs):
        ms = statistics.median(res[ci]["ms"])
        mj = statistics.median(res[ci]["mj"])
        print(json.dumps({"shape": shape, "op": op, "cfg": cfg or "default", "ms": round(ms, 4),
                          "tflops": round(flops / ms / 1e9, 1), "mJ_per_call": round(mj, 2),
                          "tflop_per_J": round(flops / 1e12 / (mj / 1e3), 3), "mhz_med": statistics.median(res[ci]["mhz"]),
                          "ms_all": [round(v, 4) for v in res[ci]["ms"]]}), flush=True)


if __name__ == "__main__":
    main()
