#!/usr/bin/env python
"""Benchmark of the TileLink B200 TP-MLP layer (BASELINE.json metric: TP-MLP layer TFLOPS & ms at
1/2/4/8 B200, vs non-overlapped NCCL + cuBLAS, % of roofline).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config llama70b|llama7b|mixtral] [--M M] [--act silu_mul|none]
                  [--rank-shape-of W] [--msweep] [--workload mlp|moe|attention] [--dry-run]

Workload (`--config`, default llama70b = LLaMA-70B MLP-5: M = 8192 tokens, H = 8192,
I = 28672, gated SiLU): the same fixed layer at every N (strong scaling), tensor parallel W = N.
  N = 1 : the whole layer on one B200 (W = 1: AG and RS degenerate to identities) -- the
          largest single-GPU configuration of BASELINE.json's list (11.5 TFLOP per layer).
  N > 1 : one process per GPU, W = N over NVLink (IPC symmetric workspace bootstrapped over NCCL).
          Without torchrun in the environment, `--gpus N` re-executes itself under
          `python -m torch.distributed.run --nproc-per-node N` (127.0.0.1), so `bench.py --gpus 8`
          and the driver's torchrun launch time the same thing.
--rank-shape-of W : (N = 1 only) the local compute of ONE rank of a TP-W layer (M x H x 2I/W and
          M x I/W x H GEMMs, no AG / RS bytes) -- labelled `<config>_rank_of_tpW`, not a layer number.
--msweep : one line per M in 1024 .. 32768 (BASELINE.json configs[4]) instead of the single line.
--impl reference : the fp64 CPU oracle (oracle/tl_oracle.py) timed on the host cores on a bounded
          row sample of the same workload (rank 0 only; other ranks exit 0).
--dry-run : no CUDA; gloo process group; checks the launch / rank / max-over-ranks / JSON plumbing.
One JSON line is printed by rank 0 (one per M with --msweep).
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {   # BASELINE.json configs[1..3] (P:550-560 MLP-1 / MLP-5; Mixtral expert FFN as a dense TP MLP)
    "llama7b": {"M": 8192, "H": 4096, "I": 11008, "paper": "MLP-1 (P:552)"},
    "llama70b": {"M": 8192, "H": 8192, "I": 28672, "paper": "MLP-5 (P:556)"},
    "mixtral": {"M": 16384, "H": 4096, "I": 14336, "paper": "Mixtral-8x7B expert FFN as dense TP MLP"},
}
DEFAULT_CONFIG = "llama70b"
MSWEEP = (1024, 2048, 4096, 8192, 16384, 32768)
METRIC = "TP-MLP layer TFLOPS"
PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
B_NVL_MEASURED = 770.0    # GB/s per direction per GPU, peer copy (B200_PROFILING.md, this pool)
B_NVL_NOMINAL = 900.0     # GB/s per direction, NVLink 5


def layer_flops(M, H, I, W, gated=True):
    """Algorithmic FLOPs per rank: GEMM1 2*M*H*N1 (N1 = 2I/W gated, I/W plain) + GEMM2 2*M*(I/W)*H."""
    il = I // W
    return 2 * M * H * (2 * il if gated else il), 2 * M * il * H


def nvlink_bytes(M, H, W):
    """Bytes per direction per rank that must cross NVLink: V_AG = V_RS = (W-1)/W * M * H * 2 (bf16)."""
    v = (W - 1) * (M // W) * H * 2
    return v, v


def bench_config(W, name=DEFAULT_CONFIG, M=None, act="silu_mul", rank_shape_of=None):
    """The workload description shared by both arms (identical `config` in both JSON lines)."""
    c = CONFIGS[name]
    M = M or c["M"]
    H, I = c["H"], c["I"]
    Wl = rank_shape_of or W
    il = I // Wl
    n1 = 2 * il if act == "silu_mul" else il
    wl = f"{name}_mlp_w{W}" if not rank_shape_of else f"{name}_rank_of_tp{rank_shape_of}"
    if M != c["M"]:
        wl += f"_M{M}"
    if act != "silu_mul":
        wl += f"_{act}"
    w1b, w2b, xb = n1 * H * 2, H * il * 2, M * H * 2
    cfg = {"workload": wl, "paper_shape": c["paper"], "M": M, "H": H, "I": I, "world": W, "act": act,
           "gemm1": f"[{M}x{H}] x [{n1}x{H}]^T", "gemm2": f"[{M}x{il}] x [{H}x{il}]^T",
           "parallelism": f"tp{W}",
           "l2": f"inputs larger than L2 per rank (W1_r {w1b / 2**20:.0f} MiB + W2_r {w2b / 2**20:.0f} MiB + "
                 f"X {xb / 2**20:.0f} MiB > 126 MB)" if w1b + w2b + xb > 126e6 else
                 "L2 flushed between steps (256 MiB write)"}
    if rank_shape_of:
        cfg["note"] = (f"local compute of one rank of a TP-{rank_shape_of} layer on one GPU (the per-rank GEMMs "
                       f"of tl_mlp_forward at W={rank_shape_of}; no AllGather / ReduceScatter bytes move)")
    return cfg


def peaks():
    try:
        with open(PEAKS_PATH) as f:
            d = json.load(f)
        return float(d["bf16_tflops"]), float(d.get("bf16_tflops_sustained", d["bf16_tflops"])), "measured"
    except Exception:
        return 1590.0, 1400.0, "fallback"


def cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.lower().startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def self_launch(argv, n):
    """`--gpus N > 1` outside torchrun: re-execute this script under torch.distributed.run with N ranks
    (one per GPU, rendezvous on 127.0.0.1) and return its exit code.  Rank 0's JSON line is the output."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__), *argv]
    env = dict(os.environ)
    env.setdefault("OMP_NUM_THREADS", "4")
    return subprocess.run(cmd, env=env).returncode


# ----------------------------------------------------------------------------- clocks sampler
class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index, self.proc, self.lines = index, None, []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, pw, reasons = [], None, [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
                pw.append(float(f[3]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        load = [s for s in sm if mx and s > 0.3 * mx] or sm
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "power_w_max": max(pw) if pw else None, "samples": len(sm)}


class NvlinkCounters:
    """NVLink data bytes sent / received by this GPU, from NVML field counters (read before and after a
    region).  Best effort: returns None where the driver or sandbox does not expose them."""
    FIELDS = ((138, 139, 1024, "NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX/RX (KiB)"),
              (202, 204, 1, "NVML_FI_DEV_NVLINK_COUNT_XMIT/RCV_BYTES"))

    def __init__(self, index):
        self.h, self.why = None, None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
        except Exception as e:
            self.why = f"nvml: {e!r}"[:120]

    def read(self):
        if self.h is None:
            return None
        for tx, rx, scale, name in self.FIELDS:
            try:
                vals = self.nv.nvmlDeviceGetFieldValues(self.h, [(tx, 0xFFFFFFFF), (rx, 0xFFFFFFFF)])
                if all(v.nvmlReturn == 0 for v in vals):
                    return name, [int(vals[0].value.ullVal) * scale, int(vals[1].value.ullVal) * scale]
            except Exception as e:
                self.why = f"{name}: {e!r}"[:120]
        return None

    @staticmethod
    def delta(a, b):
        if a is None or b is None or a[0] != b[0]:
            return None
        return a[0], b[1][0] - a[1][0], b[1][1] - a[1][1]


# ----------------------------------------------------------------------------- reference arm (oracle)
def run_reference(args):
    import numpy as np
    import tl_inputs as TI
    from oracle import tl_oracle as O
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    W = max(1, args.gpus)
    c = CONFIGS[args.config]
    M, H, I = args.M or c["M"], c["H"], c["I"]
    act = TI.ACT_SILU_MUL if args.act == "silu_mul" else TI.ACT_NONE
    Wl = args.rank_shape_of or W
    X, G, U, W2 = TI.mlp_full(M, H, I, seed=0)
    Xs, W1s, W2s = TI.shard_mlp(X, G, U, W2, Wl, act)
    if args.rank_shape_of:   # the local compute of rank 0 of a TP-W layer over all M rows (no AG/RS)
        Xs, W1s, W2s = [X], W1s[:1], W2s[:1]
    f = lambda L: [TI.to_f64(t) for t in L]
    Xs, W1s, W2s = f(Xs), f(W1s), f(W2s)
    del X, G, U, W2
    rows_per_step = args.ref_rows
    rng = np.random.default_rng(0)
    g1, g2 = layer_flops(M, H, I, Wl, act != TI.ACT_NONE)
    flops_per_row = (g1 + g2) * (1 if args.rank_shape_of else Wl) / M
    for _ in range(args.warmup):
        O.mlp_forward_rows(Xs, W1s, W2s, act, rng.choice(M, rows_per_step, replace=False))
    t0 = time.perf_counter()
    for _ in range(args.steps):
        O.mlp_forward_rows(Xs, W1s, W2s, act, rng.choice(M, rows_per_step, replace=False))
    dt = time.perf_counter() - t0
    tflops = flops_per_row * rows_per_step * args.steps / dt / 1e12
    cores = os.cpu_count()
    line = {
        "impl": "reference", "metric": METRIC, "value": round(tflops, 6), "unit": "TFLOPS", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt / args.steps * 1e3, 3),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": bench_config(W, args.config, args.M, args.act, args.rank_shape_of),
        "cpu_baseline": {"value": round(tflops, 6), "unit": "TFLOPS", "cores": cores, "cpu_model": cpu_model(),
                         "kind": "oracle",
                         "sample": f"{rows_per_step} random token rows of the M={M} layer per step (rows are "
                                   f"independent, so the row-sampled oracle is exact for them); fp64 numpy"},
        "e2e": {"value": round(tflops, 6), "unit": "TFLOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline_leg(Xs64, W1s64, W2s64, act, flops_per_row, M, seconds):
    """The oracle as it stands, timed on this host on a bounded row sample (~`seconds`)."""
    import numpy as np
    from oracle import tl_oracle as O
    rng = np.random.default_rng(1)
    rows, batch = 0, 32
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < seconds:
        O.mlp_forward_rows(Xs64, W1s64, W2s64, act, rng.choice(M, batch, replace=False))
        rows += batch
    dt = time.perf_counter() - t0
    return {"value": round(flops_per_row * rows / dt / 1e12, 6), "unit": "TFLOPS", "cores": os.cpu_count(),
            "cpu_model": cpu_model(), "kind": "oracle",
            "sample": f"{rows} token rows of the M={M} layer (row-sampled fp64 oracle, {dt:.1f} s; rows are "
                      f"independent, so the sample is exact for them)"}


# ----------------------------------------------------------------------------- dry run (no CUDA)
def run_dry(args):
    """The multi-rank plumbing without a GPU: gloo group, per-rank config, max over ranks, one line."""
    import torch.distributed as dist
    from paper_2503_20313_b200.bootstrap import max_over_ranks
    W = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if W > 1:
        dist.init_process_group("gloo")
        dist.barrier()
    t = max_over_ranks(1.0 + rank)
    line = {"metric": METRIC, "value": None, "unit": "TFLOPS", "n_gpus": W, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": None, "higher_is_better": True, "scaling": "strong",
            "dry_run": True, "ranks_seen": int(round(t)),
            "config": bench_config(W, args.config, args.M, args.act, args.rank_shape_of)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if W > 1:
        dist.destroy_process_group()


# ----------------------------------------------------------------------------- our arm
def check_rows(got, ref, tol=5e-3):
    """Element-wise and per-row parity of sampled output rows against the oracle:
    rel-Frobenius over the sample, max per-row rel-Frobenius, and the per-element bound of
    tests/parity.py (|g - o| <= 2^-7 |o| + 2^-5 rms_row(o))."""
    import numpy as np
    from oracle import tl_oracle as O
    d = got - ref
    rms = np.sqrt((ref ** 2).mean(axis=1, keepdims=True))
    row = np.sqrt((d ** 2).sum(1) / np.maximum((ref ** 2).sum(1), 1e-300))
    bound = 2.0 ** -7 * np.abs(ref) + 2.0 ** -5 * rms
    return {"rows": int(got.shape[0]), "rel_fro": float(O.rel_frobenius(got, ref)), "max_row_rel_fro": float(row.max()),
            "elements_over_bound": int((np.abs(d) > bound).sum()), "tol": tol}


def run_layer(args, ctx, M, emit=True):
    """Time one layer configuration (M rows) on this rank; returns the JSON line (rank 0) or None."""
    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_2503_20313_b200 as tl
    import tl_inputs as TI
    from paper_2503_20313_b200.bootstrap import max_over_ranks

    rank, W, distributed, dev = ctx["rank"], ctx["W"], ctx["distributed"], ctx["dev"]
    P_burst, P_sust, peak_src = peaks()
    c = CONFIGS[args.config]
    H, I = c["H"], c["I"]
    act = tl.ACT_SILU_MUL if args.act == "silu_mul" else tl.ACT_NONE
    gated = act != tl.ACT_NONE
    Wl = args.rank_shape_of or W          # tensor-parallel width the shards are cut for
    Mr, Il = M // W, I // Wl
    cfg = bench_config(W, args.config, M if M != c["M"] else None, args.act, args.rank_shape_of)

    # ---- inputs: the full problem drawn on the device with a seeded generator (identical on every
    # rank), this rank's shards kept resident in HBM; rank 0 keeps host copies for the oracle
    X, G, U, W2f = TI.mlp_full(M, H, I, seed=0, device=torch.device("cuda", dev))
    Xs, W1s, W2s = TI.shard_mlp(X, G, U, W2f, Wl, act)
    if args.rank_shape_of:
        x, w1, w2 = X.contiguous(), W1s[0], W2s[0]
    else:
        x, w1, w2 = Xs[rank], W1s[rank], W2s[rank]
    host = None
    if rank == 0:
        if args.rank_shape_of:
            host = ([X.cpu()], [W1s[0].cpu()], [W2s[0].cpu()])
        else:
            host = ([t.cpu() for t in Xs], [t.cpu() for t in W1s], [t.cpu() for t in W2s])
    del X, G, U, W2f, Xs, W1s, W2s
    torch.cuda.empty_cache()
    out = torch.empty(Mr if not args.rank_shape_of else M, H, device="cuda", dtype=torch.bfloat16)
    Z = torch.empty(M, Il, device="cuda", dtype=torch.bfloat16)
    if distributed:
        comm = tl.Comm.from_process_group(None, dev, M, H)
        if ctx.get("shared"):
            comm.set_option("num_ctas", max(2, 148 // W // 2 * 2))
            comm.set_option("timeout_ms", 120000)
    else:
        comm = tl.Comm.single(dev, M, H)
    stream = torch.cuda.current_stream()
    flush = None
    if x.numel() * 2 + w1.numel() * 2 + w2.numel() * 2 <= 126e6:   # small shapes: flush L2 between steps
        flush = torch.empty(128 * 2 ** 20, device="cuda", dtype=torch.int16)

    def step():   # tl_mlp_forward: one fused launch (AG + GEMM1 + SiLU*up, then GEMM2 + RS)
        comm.mlp_forward(x, w1, w2, out, act=act, Z=Z, stream=stream)

    def barrier():
        if distributed:
            dist.barrier()
        torch.cuda.synchronize()

    clocks = Clocks(dev)
    clocks.start()
    nvl = NvlinkCounters(dev)
    time.sleep(0.3)
    for _ in range(args.warmup):
        step()
    barrier()
    fused = comm.get_option("mlp_launches") == 1     # auto mode picked the fused launch for this shape
    mlp_fused_opt = comm.get_option("mlp_fused")

    # ---- timed region: K steps, CUDA events around each layer launch on the launching stream
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(args.steps)]
    barrier()
    nv0 = nvl.read()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    t_start.record(stream)
    for i in range(args.steps):
        if flush is not None:
            flush.fill_(i)
        ev[i][0].record(stream)
        comm.mlp_forward(x, w1, w2, out, act=act, Z=Z, stream=stream)
        ev[i][1].record(stream)
    t_end.record(stream)
    barrier()
    nv1 = nvl.read()
    soak_end = time.perf_counter() + 1.0
    while time.perf_counter() < soak_end:
        for _ in range(4):
            step()
        torch.cuda.synchronize()
    clk = clocks.stop()
    lk = [e[0].elapsed_time(e[1]) for e in ev]
    layer_ms = max_over_ranks(sum(lk) / len(lk))          # the layer's launch(es), mean per step
    if flush is None:
        total_ms = max_over_ranks(t_start.elapsed_time(t_end))
        ms = total_ms / args.steps
    else:   # the L2 flush between steps is not part of the layer
        ms = layer_ms
    st, diag = comm.check()
    # breakdown (context, not the headline): the same layer as two launches, each timed on its own
    comm.set_option("mlp_fused", 0)
    for _ in range(2):
        comm.ag_gemm(x, w1, Z, act=act, stream=stream)
        comm.gemm_rs(Z, w2, out, stream=stream)
    barrier()
    bk = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    for i in range(args.steps):
        if flush is not None:
            flush.fill_(i)
        bk[i][0].record(stream)
        comm.ag_gemm(x, w1, Z, act=act, stream=stream)
        bk[i][1].record(stream)
        comm.gemm_rs(Z, w2, out, stream=stream)
        bk[i][2].record(stream)
    barrier()
    comm.set_option("mlp_fused", mlp_fused_opt)
    k1_ms = max_over_ranks(sum(e[0].elapsed_time(e[1]) for e in bk) / args.steps)
    k2_ms = max_over_ranks(sum(e[1].elapsed_time(e[2]) for e in bk) / args.steps)
    comm.mlp_forward(x, w1, w2, out, act=act, Z=Z, stream=stream)   # `out` from the product path again
    barrier()
    f1, f2 = layer_flops(M, H, I, Wl, gated)
    n_rank_units = 1 if args.rank_shape_of else W
    value = (f1 + f2) * n_rank_units / (ms * 1e-3) / 1e12        # whole job (all ranks), TFLOPS
    per_gpu = value / W
    ach = (f1 + f2) / (layer_ms * 1e-3) / 1e12            # the fused kernel's FLOPs per launch / its time
    v_ag, v_rs = nvlink_bytes(M, H, W) if not args.rank_shape_of else (0, 0)
    # roofline: layer = max((F1+F2)/P_TC, (V_AG+V_RS)/B_NVL); two-phase form beside it
    t_tc = (f1 + f2) / (P_burst * 1e12)
    t_nvl = (v_ag + v_rs) / (B_NVL_MEASURED * 1e9)
    t_layer = max(t_tc, t_nvl)
    t_two = max(f1 / (P_burst * 1e12), v_ag / (B_NVL_MEASURED * 1e9)) + \
        max(f2 / (P_burst * 1e12), v_rs / (B_NVL_MEASURED * 1e9))
    nvl_d = NvlinkCounters.delta(nv0, nv1)
    nvl_line = {"unavailable": nvl.why or "counters not exposed"} if nvl_d is None else {
        "source": nvl_d[0], "tx_bytes_per_step": nvl_d[1] / args.steps, "rx_bytes_per_step": nvl_d[2] / args.steps,
        "algorithmic_bytes_per_dir_per_step": v_ag + v_rs,
        "tx_GBps": nvl_d[1] / (ms * 1e-3 * args.steps) / 1e9, "rx_GBps": nvl_d[2] / (ms * 1e-3 * args.steps) / 1e9,
        "peak_GBps_per_dir": B_NVL_NOMINAL}
    nvl_tx = max_over_ranks(nvl_line.get("tx_bytes_per_step", -1))

    # ---- parity of this run's output against the fp64 oracle: every rank's block is sampled (rows
    # spread over the block + one whole 128-row tile of rank 0), per element and per row
    parity = None
    if distributed and ctx.get("shared"):   # gloo: gather through host memory
        full = torch.empty(M, H, dtype=torch.bfloat16)
        dist.all_gather_into_tensor(full, out.cpu())
    elif distributed:
        full = torch.empty(M, H, device="cuda", dtype=torch.bfloat16)
        dist.all_gather_into_tensor(full, out)
    else:
        full = out
    from oracle import tl_oracle as O
    if rank == 0:
        nb = W if not args.rank_shape_of else 1
        blk = M // nb
        rows = sorted(set(list(range(128)) + [b * blk + (j * 997) % blk for b in range(nb) for j in range(8)]))
        hX, hW1, hW2 = ([TI.to_f64(t) for t in L] for L in host)
        del host
        oracle_rows = lambda rr: O.mlp_forward_rows(hX, hW1, hW2, act, rr)
        ref = oracle_rows(rows)
        got = full.float().cpu().double().numpy()
        parity = check_rows(np.stack([got[i] for i in rows]), np.stack([ref[i] for i in rows]))
        parity["status"] = int(st)
    del full
    barrier()   # rank 0's oracle work is done before any rank launches the next collective layer call

    # ---- end to end through the public API: every step copies its X shard in from pinned host memory
    # and its output back (paper_2503_20313_b200.pipeline.MLPPipeline: H2D of step i+1 and D2H of step
    # i-1 overlap the layer of step i on separate streams)
    e2e = None
    if not args.rank_shape_of:
        from paper_2503_20313_b200.pipeline import MLPPipeline
        pipe = MLPPipeline(comm, w1, w2, act, Mr, H)
        xh = x.cpu()
        hx = [xh.pin_memory(), (xh.float() * -1.0).to(torch.bfloat16).pin_memory()]
        hin = [hx[i % 2] for i in range(args.steps)]
        hout = [torch.empty(Mr, H, dtype=torch.bfloat16).pin_memory() for _ in range(min(args.steps, 4))]
        hout = [hout[i % len(hout)] for i in range(args.steps)]
        pipe.run(hin[:2], hout[:2])
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        pipe.run(hin, hout, e0, e1)
        barrier()
        e2e_ms = max_over_ranks(e0.elapsed_time(e1)) / args.steps
        last = (args.steps - 1) % 2
        comm.mlp_forward(x if last == 0 else hx[1].cuda(), w1, w2, out, act=act, Z=Z)
        torch.cuda.synchronize()
        e2e_match = bool(torch.equal(hout[args.steps - 1], out.cpu()))
        e2e = {"value": round((f1 + f2) * W / (e2e_ms * 1e-3) / 1e12, 2), "unit": "TFLOPS",
               "ms_per_step": round(e2e_ms, 4), "h2d_bytes_per_step": pipe.bytes_in * W,
               "d2h_bytes_per_step": pipe.bytes_out * W,
               "api": "tl_mlp_forward via paper_2503_20313_b200.pipeline.MLPPipeline (pinned host X shard in, "
                      "output shard back, every step on every rank; copies overlap the neighbouring steps' layers)",
               "output_matches_device_run": e2e_match}
        del pipe

    # ---- non-overlapped NCCL + cuBLAS baseline (same inputs, same protocol)
    base = None
    if not args.no_baseline:
        xg = torch.empty(M, H, device="cuda", dtype=torch.bfloat16) if distributed else None
        part = torch.empty(M, H, device="cuda", dtype=torch.bfloat16) if distributed else None
        ob = torch.empty_like(out)
        bev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(args.steps)]

        def base_step(e=None):
            if e:
                e[0].record(stream)
            if distributed:
                dist.all_gather_into_tensor(xg, x)
                src = xg
            else:
                src = x
            y = src @ w1.T
            z = torch.nn.functional.silu(y[:, :Il]) * y[:, Il:] if gated else y
            if distributed:
                torch.matmul(z, w2.T, out=part)
                dist.reduce_scatter_tensor(ob, part)
            else:
                torch.matmul(z, w2.T, out=ob)
            if e:
                e[1].record(stream)

        for _ in range(args.warmup):
            base_step()
        barrier()
        for i in range(args.steps):
            if flush is not None:
                flush.fill_(i)
            base_step(bev[i])
        barrier()
        bms = max_over_ranks(sum(e[0].elapsed_time(e[1]) for e in bev) / args.steps)
        base = {"impl": "nccl+cublas non-overlapped (all_gather_into_tensor, torch.matmul, silu*mul, torch.matmul, "
                        "reduce_scatter_tensor)" if distributed else "cublas (torch.matmul, silu*mul, torch.matmul)",
                "ms_per_step": round(bms, 4), "value": round((f1 + f2) * n_rank_units / (bms * 1e-3) / 1e12, 2),
                "unit": "TFLOPS", "speedup_ours": round(bms / ms, 4)}
        if distributed:
            fullb = torch.empty(M, H, device="cuda", dtype=torch.bfloat16)
            dist.all_gather_into_tensor(fullb, ob)
        else:
            fullb = ob
        if rank == 0:   # the baseline's own error against the same oracle rows
            gb = fullb.float().cpu().double().numpy()
            base["parity_rel_fro"] = O.rel_frobenius(np.stack([gb[i] for i in rows]), np.stack([ref[i] for i in rows]))
        del xg, part, ob, fullb
    barrier()

    # ---- W = 8 ranks emulated on this GPU (full fused protocol, one launch per kernel), N = 1 only
    loop = None
    if not distributed and not args.no_loopback and not args.rank_shape_of and M % 8 == 0 and (M // 8) % 128 == 0:
        loop = loopback_leg(args, M, H, I, act, oracle_rows if rank == 0 else None, stream)

    cpu = None
    if rank == 0 and args.cpu_seconds > 0:
        fpr = (f1 + f2) * n_rank_units / M
        cpu = cpu_baseline_leg(hX, hW1, hW2, act, fpr, M, args.cpu_seconds)
    barrier()
    opts = {k: comm.get_option(k) for k in ("cta_pair", "n_sub", "raster_group", "comm_tile_rows", "ag_binding",
                                            "rs_binding", "rs_order", "ag_mode", "mlp_fused")}
    opts["mlp_launches"] = 1 if fused else 2
    comm.close()
    if rank != 0:
        return None
    line = {
        "metric": METRIC, "value": round(value, 2), "unit": "TFLOPS", "n_gpus": W, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "bf16",
        **({"mode": "TL_BENCH_SHARED_GPU code-path check: all ranks time-share cuda:0, not a measurement"}
           if ctx.get("shared") else {}),
        "data": "synthetic (seeded N(0,1) activations, N(0,1/fan_in) weights, "
                                                  "bf16; random-init weights of the named shape)",
        "config": cfg,
        "options": opts,
        "tflops_per_gpu": round(per_gpu, 2),
        "kernels_ms": {"mlp_fused" if fused else "ag_gemm_act+gemm_rs": round(layer_ms, 4),
                       "unfused_breakdown": {"ag_gemm_act": round(k1_ms, 4), "gemm_rs": round(k2_ms, 4),
                                             "sum": round(k1_ms + k2_ms, 4)}},
        "roofline": {"bound": "tensor" if t_tc >= t_nvl else "nvlink",
                     "kernel": ("tl_mlp_kernel (fused layer: AG + GEMM1 + SiLU*up, then GEMM2 + RS)" if fused else
                                "tl_gemm_kernel x2 (AG-GEMM1 + SiLU*up; GEMM2 + RS)"),
                     "achieved": round(ach, 2),
                     "peak": P_burst, "unit": "TFLOP/s", "frac": round(ach / P_burst, 4),
                     "frac_sustained": round(ach / P_sust, 4), "peak_sustained": P_sust, "peak_source": peak_src,
                     "kernel_roof_ms": round(t_layer * 1e3, 4), "kernel_frac": round(t_layer * 1e3 / layer_ms, 4),
                     "layer_roof_ms": round(t_layer * 1e3, 4), "layer_frac": round(t_layer * 1e3 / ms, 4),
                     "layer_roof_terms_ms": {"tensor": round(t_tc * 1e3, 4), "nvlink": round(t_nvl * 1e3, 4)},
                     "two_phase_roof_ms": round(t_two * 1e3, 4), "two_phase_frac": round(t_two * 1e3 / ms, 4),
                     "nvlink_GBps_per_dir": B_NVL_MEASURED, "nvlink_bytes_per_dir": {"ag": v_ag, "rs": v_rs},
                     "traffic": None, "per_launch_flop": f1 + f2},
        "nvlink_counters": dict(nvl_line, max_tx_bytes_per_step_over_ranks=nvl_tx) if W > 1 else None,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": (1 if fused else 2) * args.steps,
        "clocks": clk,
        "parity": parity,
        "baseline_nccl_cublas": base,
        "loopback_w8": loop,
    }
    traffic_path = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(traffic_path):
        try:
            line["roofline"]["traffic"] = json.load(open(traffic_path)).get(cfg["workload"])
        except Exception:
            pass
    if emit:
        print(json.dumps(line), flush=True)
    return line


def loopback_leg(args, M, H, I, act, oracle_rows, stream):
    """The same layer with 8 ranks emulated on the one GPU: the full AG push / flag / RS push / owner-reduce
    protocol runs, peer stores landing in local HBM (a protocol check and the P:660 overlap ratio)."""
    import numpy as np
    import torch
    import paper_2503_20313_b200 as tl
    import tl_inputs as TI
    from oracle import tl_oracle as O
    LW = 8
    X, G, U, W2f = TI.mlp_full(M, H, I, seed=0, device=torch.device("cuda", torch.cuda.current_device()))
    xs8, w18, w28 = TI.shard_mlp(X, G, U, W2f, LW, act)
    del X, G, U, W2f
    lc = tl.Comm.loopback(LW, torch.cuda.current_device(), M, H)
    o8 = [torch.empty(M // LW, H, device="cuda", dtype=torch.bfloat16) for _ in range(LW)]
    z8 = [torch.empty(M, I // LW, device="cuda", dtype=torch.bfloat16) for _ in range(LW)]
    steps = max(3, min(args.steps, 10))
    f1, f2 = layer_flops(M, H, I, LW, act != tl.ACT_NONE)

    def lb_time(binding, rs_binding=0):
        lc.set_option("ag_binding", binding)
        lc.set_option("rs_binding", rs_binding)
        for _ in range(args.warmup):
            lc.ag_gemm_lb(xs8, w18, z8, act=act)
            lc.gemm_rs_lb(z8, w28, o8)
        torch.cuda.synchronize()
        le = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(steps)]
        for i in range(steps):
            le[i][0].record(stream)
            lc.ag_gemm_lb(xs8, w18, z8, act=act)
            le[i][1].record(stream)
            lc.gemm_rs_lb(z8, w28, o8)
            le[i][2].record(stream)
        torch.cuda.synchronize()
        lst, _ = lc.check()
        l1 = sum(e[0].elapsed_time(e[1]) for e in le) / steps
        l2 = sum(e[1].elapsed_time(e[2]) for e in le) / steps
        return l1, l2, lst

    rows = [0, M // 8 - 1, M // 3, M // 2 + 5, M - 1]
    # the same layer (same seeded full problem), so the oracle rows of the main run apply (sharding invariant)
    ref = oracle_rows(rows) if oracle_rows is not None else None
    loop = {"world": LW, "mode": "loopback (8 ranks on 1 GPU, 18 CTAs each; peer stores -> local HBM; the 8 ranks "
                                 "share one L2, so this is a protocol check, not a perf config)"}

    def ag_ms(mode, n):
        lc.set_option("debug_mode", mode)
        lc.ag_gemm_lb(xs8, w18, z8, act=act)
        torch.cuda.synchronize()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        for _ in range(n):
            lc.ag_gemm_lb(xs8, w18, z8, act=act)
        a1.record(stream)
        torch.cuda.synchronize()
        lc.set_option("debug_mode", 0)
        return a0.elapsed_time(a1) / n
    for binding, name in ((0, "sm"), (1, "copy_engine")):
        lc.set_option("ag_binding", binding)
        runs = [[ag_ms(m, 3) for m in (0, 1, 2)] for _ in range(3)]        # round robin: clock drift hits all
        ov, cp, cm = (sorted(r[m] for r in runs)[1] for m in range(3))
        loop[f"overlap_ratio_ag_{name}"] = {"comp_only_ms": round(cp, 4), "comm_only_ms": round(cm, 4),
                                            "overlap_ms": round(ov, 4),
                                            "ratio": round((cp + cm - ov) / cm, 4) if cm > 0 else None}
        if cm > 0 and cp + cm - ov < 0:
            loop[f"overlap_ratio_ag_{name}"]["note"] = (
                "negative: the fused call is slower than compute-only + copy-only here, because the 8 emulated "
                "ranks' copies (8x one rank's AG bytes) contend with the GEMMs for the one GPU's HBM and L2; "
                "on a real TP-8 box each rank's copies go over NVLink instead")
    lc.check()
    for binding, rsb, name in ((0, 0, "sm"), (1, 0, "copy_engine"), (1, 1, "copy_engine_ag_and_rs")):
        l1, l2, lst = lb_time(binding, rsb)
        d = {"ag_gemm_ms": round(l1, 4), "gemm_rs_ms": round(l2, 4), "ms_per_step": round(l1 + l2, 4),
             "value": round((f1 + f2) * LW / (l1 + l2) / 1e9, 2), "unit": "TFLOPS (whole layer, 1 GPU)",
             "status": int(lst)}
        if ref is not None:
            mr8 = M // LW
            got = np.stack([o8[i // mr8][i % mr8].float().cpu().double().numpy() for i in rows])
            d["parity_rel_fro"] = O.rel_frobenius(got, np.stack([ref[i] for i in rows]))
        loop[f"binding_{name}"] = d
    lc.close()
    return loop


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=sorted(CONFIGS))
    ap.add_argument("--M", type=int, default=None, help="token rows (default: the config's M)")
    ap.add_argument("--act", default="silu_mul", choices=["silu_mul", "none"])
    ap.add_argument("--rank-shape-of", type=int, default=None, dest="rank_shape_of")
    ap.add_argument("--msweep", action="store_true")
    ap.add_argument("--ref-rows", type=int, default=64)
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-loopback", action="store_true")
    ap.add_argument("--no-baseline", action="store_true")
    ap.add_argument("--dry-run", action="store_true")
    ap.add_argument("--workload", default="mlp", choices=["mlp", "moe", "attention"],
                    help="mlp = the north-star TP-MLP layer (default); moe / attention = SURVEY NEXT-3 / NEXT-4 "
                         "(bench_workloads.py), same JSON contract")
    raw = sys.argv[1:] if argv is None else argv
    args = ap.parse_args(raw)
    args.warmup = max(3, args.warmup)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return self_launch(raw, args.gpus)
    if args.rank_shape_of and args.gpus != 1:
        raise SystemExit("--rank-shape-of is a single-GPU mode (N = 1)")
    if args.dry_run:
        return run_dry(args)
    if args.workload != "mlp":
        import bench_workloads as BW
        if args.impl == "reference":
            return BW.run_reference(args)
        return (BW.run_moe if args.workload == "moe" else BW.run_attention)(args, (Clocks, peaks))
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist
    world_env = int(os.environ.get("WORLD_SIZE", "1"))
    distributed = world_env > 1
    # TL_BENCH_SHARED_GPU=1 (code-path check only, never a measurement): every rank on cuda:0 with a share
    # of the SMs, gloo instead of NCCL (which refuses two ranks on one device), no NCCL baseline
    shared = distributed and os.environ.get("TL_BENCH_SHARED_GPU") == "1"
    if shared:
        torch.cuda.set_device(0)
        dist.init_process_group("gloo")
        rank, W = dist.get_rank(), dist.get_world_size()
        args.no_baseline = True
    elif distributed:
        local = int(os.environ.get("LOCAL_RANK", "0"))
        if local >= torch.cuda.device_count():
            raise RuntimeError(f"rank {local} needs cuda:{local}, only {torch.cuda.device_count()} device(s) visible")
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        rank, W = dist.get_rank(), dist.get_world_size()
    else:
        torch.cuda.set_device(0)
        rank, W = 0, 1
    ctx = {"rank": rank, "W": W, "distributed": distributed, "dev": torch.cuda.current_device(), "shared": shared}
    Ms = MSWEEP if args.msweep else [args.M or CONFIGS[args.config]["M"]]
    for M in Ms:
        if args.msweep:
            args.cpu_seconds = min(args.cpu_seconds, 3.0)
        run_layer(args, ctx, M)
    if distributed:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    try:
        rc = main()
        sys.exit(rc if isinstance(rc, int) else 0)
    except Exception as exc:   # still emit one JSON line (rank 0) saying why the run could not complete
        if int(os.environ.get("RANK", "0")) == 0:
            print(json.dumps({"metric": METRIC, "value": None, "unit": "TFLOPS",
                              "n_gpus": int(os.environ.get("WORLD_SIZE", "1")), "error": repr(exc)[:400]}),
                  flush=True)
        raise
