"""Tile timeline of one GEMM launch from the device event trace (option trace_events): when each pair's
MMA warp starts a tile (tile_start) and when its epilogue finishes it (tile_end), to see where a short
kernel loses tensor time (fill, per-tile gaps, tail).

  python tools/tile_timeline.py SHAPE g1|g2 ["opts"]      SHAPE as in tools/ab.py (7b_tp8, 70b_tp8, ...)
"""
import statistics
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2503_20313_b200 as tl  # noqa: E402
from paper_2503_20313_b200.trace import read_events  # noqa: E402

SHAPES = {"7b": (8192, 4096, 11008), "70b": (8192, 8192, 28672), "mix": (16384, 4096, 14336)}


def main():
    shape, op = sys.argv[1], sys.argv[2]
    opts = sys.argv[3] if len(sys.argv) > 3 else ""
    base, _, tp = shape.partition("_tp")
    W = int(tp) if tp else 1
    M, H, I = SHAPES[base]
    il = I // W
    g = torch.Generator(device="cuda").manual_seed(1)
    x = torch.randn(M, H, device="cuda", generator=g).bfloat16()
    w1 = (torch.randn(2 * il, H, device="cuda", generator=g) * H ** -0.5).bfloat16()
    w2 = (torch.randn(H, il, device="cuda", generator=g) * I ** -0.5).bfloat16()
    Z = torch.empty(M, il, device="cuda", dtype=torch.bfloat16)
    out = torch.empty(M, H, device="cuda", dtype=torch.bfloat16)
    c = tl.Comm.single(0, max_M=M, max_H=H)
    for kv in filter(None, opts.split(",")):
        k, v = kv.split("=")
        c.set_option(k, int(v))
    run = (lambda: c.ag_gemm(x, w1, Z, act=tl.ACT_SILU_MUL)) if op == "g1" else (lambda: c.gemm_rs(Z, w2, out))
    for _ in range(5):
        run()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        run()
    b.record()
    torch.cuda.synchronize()
    print(f"untraced: {a.elapsed_time(b) / 10 * 1e3:.1f} us per launch")
    c.set_option("trace_events", 1 << 16)
    run()
    torch.cuda.synchronize()
    c.set_option("trace_events", 1 << 15)   # realloc -> empty
    run()
    torch.cuda.synchronize()
    ev = read_events(c, clocks=True)
    clk = {e["tile"]: e["t_ns"] for e in ev if e["kind"] == "sm_clock"}
    ev = [e for e in ev if e["kind"] != "sm_clock"]
    st = [e for e in ev if e["kind"] == "tile_start"]
    en = [e for e in ev if e["kind"] == "tile_end"]
    t0 = min(e["t_ns"] for e in st)
    n_pairs = (c.get_option("num_ctas") or 148) // 2
    by_pair = {}
    for e in st:
        by_pair.setdefault(e["tile"] % n_pairs, []).append(("s", e["tile"], e["t_ns"] - t0))
    for e in en:
        by_pair.setdefault(e["tile"] % n_pairs, []).append(("e", e["tile"], e["t_ns"] - t0))
    first = [min(t for k, _, t in v if k == "s") for v in by_pair.values()]
    last = [max(t for k, _, t in v if k == "e") for v in by_pair.values()]
    dur = []
    for v in by_pair.values():
        s = sorted(t for k, _, t in v if k == "s")
        dur += [b_ - a_ for a_, b_ in zip(s, s[1:])]
    print(f"items {len(st)} pairs {len(by_pair)}; first tile start (us): min {min(first)/1e3:.1f} med "
          f"{statistics.median(first)/1e3:.1f} max {max(first)/1e3:.1f}")
    print(f"last tile end (us): min {min(last)/1e3:.1f} med {statistics.median(last)/1e3:.1f} max {max(last)/1e3:.1f}")
    if dur:
        print(f"start-to-start per pair (us): min {min(dur)/1e3:.2f} med {statistics.median(dur)/1e3:.2f} "
              f"max {max(dur)/1e3:.2f}")
    # tile periods in SM cycles (clock64 at each MMA tile start) and the implied SM clock
    tstart = {e["tile"]: e["t_ns"] for e in st}
    cyc, mhz = [], []
    for p in by_pair:
        its = sorted(i for k, i, _ in by_pair[p] if k == "s")
        for a_, b_ in zip(its, its[1:]):
            if a_ in clk and b_ in clk:
                cyc.append(clk[b_] - clk[a_])
                mhz.append((clk[b_] - clk[a_]) / max(1, tstart[b_] - tstart[a_]) * 1e3)
    if cyc:
        print(f"tile period (SM cycles): min {min(cyc)} med {statistics.median(cyc)} max {max(cyc)}; "
              f"implied SM clock med {statistics.median(mhz):.0f} MHz")
    for p in sorted(by_pair)[:2]:
        print(p, [(k, i, round(t / 1e3, 1)) for k, i, t in sorted(by_pair[p], key=lambda z: z[2])])


if __name__ == "__main__":
    main()
