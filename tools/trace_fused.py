"""Device event trace of the fused TP-MLP layer (AG-GEMM1 + SiLU*up, GEMM2 + RS) with W ranks emulated
on one GPU (loopback): writes the SPEC-format JSONL trace and prints the analyze_trace summary plus
timeline evidence of tile-level overlap (GEMM tiles computing while AllGather tiles are still in
flight; RS partial tiles pushed while later GEMM2 tiles compute).

  python tools/trace_fused.py [W] [M] [H] [I]      (default 8 8192 4096 11008: the LLaMA-7B layer)"""
import json
import os
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2503_20313_b200 as tl  # noqa: E402
import tl_inputs as TI  # noqa: E402
from paper_2503_20313_b200 import trace as T  # noqa: E402

W, M, H, I = (int(a) for a in (sys.argv[1:] + ["8", "8192", "4096", "11008"][len(sys.argv) - 1:])[:4])
X, G, U, W2 = TI.mlp_full(M, H, I, seed=0)
Xs, W1s, W2s = TI.shard_mlp(X, G, U, W2, W, TI.ACT_SILU_MUL)
xs, w1s, w2s = ([t.cuda() for t in L] for L in (Xs, W1s, W2s))
c = tl.Comm.loopback(W, 0, max_M=M, max_H=H)
Zs = [torch.empty(M, I // W, device="cuda", dtype=torch.bfloat16) for _ in range(W)]
outs = [torch.empty(M // W, H, device="cuda", dtype=torch.bfloat16) for _ in range(W)]
for _ in range(2):                                          # warm-up (untraced)
    c.ag_gemm_lb(xs, w1s, Zs, act=tl.ACT_SILU_MUL)
    c.gemm_rs_lb(Zs, w2s, outs)
torch.cuda.synchronize()
c.set_option("trace_events", 1 << 20)
summary = {}
for name, fn in (("ag_gemm", lambda: c.ag_gemm_lb(xs, w1s, Zs, act=tl.ACT_SILU_MUL)),
                 ("gemm_rs", lambda: c.gemm_rs_lb(Zs, w2s, outs))):
    fn()
    ev = T.read_events(c)
    os.makedirs("gpurun_out", exist_ok=True)
    T.to_jsonl(ev, f"gpurun_out/trace_{name}_w{W}.jsonl")
    rep = T.analyze_trace(ev)
    t0 = min(e["t_ns"] for e in ev)
    comp = [e for e in ev if e["unit"] == "compute"]
    s = {"events": len(ev), "span_us": rep["span_ns"] / 1e3, "diagnostics": rep["diagnostics"][:5],
         "n_diagnostics": len(rep["diagnostics"])}
    if name == "ag_gemm":
        copy_end = [e["t_ns"] - t0 for e in ev if e["kind"] == "copy_end"]
        tile_start = sorted(e["t_ns"] - t0 for e in comp if e["kind"] == "tile_start")
        last_copy = max(copy_end)
        s.update({"copy_spans": len(copy_end), "last_copy_end_us": last_copy / 1e3,
                  "gemm_tiles": len(tile_start),
                  "gemm_tiles_started_before_last_copy_end": sum(t < last_copy for t in tile_start),
                  "first_tile_start_us": tile_start[0] / 1e3,
                  "consumer_wait_total_us_per_rank": {k: v["wait_ns"] / 1e3 for k, v in rep["per_unit"].items()
                                                       if k.endswith("compute")},
                  "copy_time_under_compute_frac": {r: round(v["copy_under_compute_ns"] / max(1, v["copy_ns"]), 3)
                                                   for r, v in rep["overlap"].items()}})
    else:
        notif = sorted(e["t_ns"] - t0 for e in comp if e["kind"] == "notify")
        tile_end = sorted(e["t_ns"] - t0 for e in comp if e["kind"] == "tile_end")
        s.update({"rs_pushes": len(notif), "first_push_us": notif[0] / 1e3 if notif else None,
                  "last_tile_end_us": tile_end[-1] / 1e3,
                  "pushes_before_half_of_tiles_done": sum(n < tile_end[len(tile_end) // 2] for n in notif),
                  "owner_wait_total_us_per_rank": {k: v["wait_ns"] / 1e3 for k, v in rep["per_unit"].items()}})
    summary[name] = s
st, diag = c.check()
summary["status"] = st
summary["config"] = {"W": W, "M": M, "H": H, "I": I, "mode": "loopback (W ranks on one GPU)"}
print(json.dumps(summary, indent=1))
